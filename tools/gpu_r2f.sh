#!/bin/bash
# profiles of the codec kernels at C2 / C3 (round 2 baseline)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'encode_tc|encode_warp|decode_fast' -s 3 -c 3 \
   -o gpurun_out/prof_codec -f python tools/prof_unit.py --reps 2 --attn-batch 0 > gpurun_out/prof_codec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'radix_hist|decode_flag|token_coded' -s 5 -c 5 \
   -o gpurun_out/prof_med3x -f python tools/prof_unit.py --reps 2 --outlier --attn-batch 0 > gpurun_out/prof_med3x.log 2>&1
timeout 300 python tools/decode_bench.py > gpurun_out/decode_bench.log 2>&1
echo done
