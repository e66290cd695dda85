#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_pair' -s 3 -c 1 \
   -o gpurun_out/prof_attn_pair_n -f python tools/attn_prof.py > gpurun_out/prof_attn_pair_n.log 2>&1
echo done
