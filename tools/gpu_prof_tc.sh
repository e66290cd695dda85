#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'encode_tc|encode_warp' -s 2 -c 2 \
   -o gpurun_out/prof_tc -f python tools/prof_unit.py --reps 2 --attn-batch 0 > gpurun_out/prof_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'encode_tc' -s 1 -c 1 \
   -o gpurun_out/prof_tc256 -f python tools/prof_unit.py --reps 2 --attn-batch 0 --S 256 > gpurun_out/prof_tc256.log 2>&1
echo done
