#!/bin/bash
# ncu full captures of the slowest wide diagonal-solve launches (60^3, one graph solve)
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_sv_bdiag" -s ${1:-43} -c 1 -o gpurun_out/sv_bdiag -f python tools/solve_ncu.py 60 > gpurun_out/ncu_sv.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_sv_fdiag" -s ${2:-1} -c 1 -o gpurun_out/sv_fdiag -f python tools/solve_ncu.py 60 >> gpurun_out/ncu_sv.log 2>&1
tail -3 gpurun_out/ncu_sv.log
