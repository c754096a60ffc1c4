#!/bin/bash
# ncu --set full of the heaviest k_update launch (non-graph run, table order), 60^3
mkdir -p gpurun_out
N=${1:-60}
python tools/ncu_kupd.py $N info > gpurun_out/kupd_info.json
SKIP=$(python -c "import json; print(json.load(open('gpurun_out/kupd_info.json'))['launch_skip'])")
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_update$" --kernel-name-base function -s $SKIP -c 1 -o gpurun_out/kupd_full -f python tools/ncu_kupd.py $N run > gpurun_out/ncu_kupd.log 2>&1
tail -3 gpurun_out/ncu_kupd.log
