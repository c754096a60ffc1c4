#!/bin/bash
# One GPU session: build check, gpu tests, bench, launch list, ncu capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/launch_profile.py 60 llt > gpurun_out/launch_profile.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ncu.csv python tools/ncu_one.py 60 llt 2 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_update\\(" -s 60 -c 4 -o gpurun_out/k_update_full -f python tools/ncu_one.py 60 llt 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
