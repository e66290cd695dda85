#!/bin/bash
# r3v: warm-cache launch list of the C3 unit encode chain
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 40 -c 40 --csv --log-file gpurun_out/c3_warm_launches.csv python tools/c3_unit.py 10 > gpurun_out/c3_warm.log 2>&1
echo done
