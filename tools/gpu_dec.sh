#!/bin/bash
mkdir -p gpurun_out
python tools/decode_bench.py > gpurun_out/decode_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_fast' -s 5 -c 1 \
   -o gpurun_out/prof_dec -f python tools/decode_bench.py > gpurun_out/prof_dec.log 2>&1
echo done
