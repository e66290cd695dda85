#!/bin/bash
# decode / Med3x kernel captures for the l1tex breakdown
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_fast' -s 3 -c 1 \
   -o gpurun_out/prof_dec -f python tools/prof_unit.py --reps 5 --attn-batch 0 > gpurun_out/prof_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'radix_hist|decode_flag|encode_warp|encode_tc|token_coded|radix_tail' -s 12 -c 12 \
   -o gpurun_out/prof_m3 -f python tools/prof_unit.py --reps 3 --outlier --attn-batch 0 > gpurun_out/prof_m3.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_split.json 2>&1
echo done
