#!/bin/bash
# ncu capture of the dataflow kernel (source-level stall sampling)
N=${1:-40}
mkdir -p gpurun_out
PS_SCHED=dataflow timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dataflow -s 1 -c 1 -o gpurun_out/df_full_$N -f python tools/ncu_one.py $N llt 2 > gpurun_out/ncu_df_$N.log 2>&1
ls -la gpurun_out
