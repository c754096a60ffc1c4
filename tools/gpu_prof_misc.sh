#!/bin/bash
# ncu --set full of the level-0 narrow-update launch and one diagonal-block launch (60^3)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_update_narrow_w" -c 1 -o gpurun_out/narrow_full -f python tools/ncu_one.py 60 llt 1 > gpurun_out/ncu_misc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_factor_diag_blk" -s 200 -c 1 -o gpurun_out/diag_full -f python tools/ncu_one.py 60 llt 1 >> gpurun_out/ncu_misc.log 2>&1
tail -3 gpurun_out/ncu_misc.log
