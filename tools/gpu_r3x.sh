#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:'median_pass' -s 9 -c 3 \
   -o gpurun_out/prof_median_x -f python tools/c3_unit.py 3 > gpurun_out/prof_median_x.log 2>&1
echo done
