#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or attn or paged" > gpurun_out/pytest_r4p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4p.log
timeout 1200 python bench.py --no-cpu --no-e2e > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err
echo done
