#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'encode_warp' -s 2 -c 2 \
   -o gpurun_out/prof_enc -f python tools/prof_unit.py --reps 2 --attn-batch 0 > gpurun_out/prof_enc.log 2>&1
echo done
