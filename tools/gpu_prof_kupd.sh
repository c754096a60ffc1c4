#!/bin/bash
# ncu --set full of the heaviest k_update launch (non-graph run, table order), 60^3
mkdir -p gpurun_out
N=${1:-60}
LEV=${2:-}
TAG=${3:-kupd}
python tools/ncu_kupd.py $N info $LEV > gpurun_out/${TAG}_info.json
SKIP=$(python -c "import json; print(json.load(open('gpurun_out/${TAG}_info.json'))['launch_skip'])")
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_update$" --kernel-name-base function -s $SKIP -c 1 -o gpurun_out/${TAG}_full -f python tools/ncu_kupd.py $N run > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
