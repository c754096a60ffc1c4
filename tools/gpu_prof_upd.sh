#!/bin/bash
# ncu full capture of one large k_update launch (level schedule, 60^3)
mkdir -p gpurun_out
SKIP=${1:-160}
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_update\\(" -s $SKIP -c 1 -o gpurun_out/kupd_full -f python tools/ncu_one.py 60 llt 1 > gpurun_out/ncu_kupd.log 2>&1
tail -3 gpurun_out/ncu_kupd.log
