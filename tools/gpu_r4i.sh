#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python bench.py --workload c1 --no-attn --no-cpu > gpurun_out/bench_c1_i.json 2> gpurun_out/bench_c1_i.err
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4i.log
echo done
