#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4y.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 1414 > gpurun_out/fuzz_r4y.log 2>&1
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_y2.log 2>&1; done
timeout 300 python tools/c1_unit.py >> gpurun_out/c3_unit_y2.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_y2.json 2> /dev/null
echo done
