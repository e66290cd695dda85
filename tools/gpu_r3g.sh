#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 120 python tools/c3_unit.py 20 > gpurun_out/c3_unit.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/c3_unit.py 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > gpurun_out/pytest_r3g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3g.log
echo done
