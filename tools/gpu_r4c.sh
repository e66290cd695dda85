#!/bin/bash
# r4c: C1 unit launch chain (warm)
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/c1_unit.py > gpurun_out/c1_unit.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 60 -c 30 \
   --csv --log-file gpurun_out/c1_warm_launches.csv python tools/c1_unit.py > gpurun_out/c1_warm.log 2>&1
echo done
