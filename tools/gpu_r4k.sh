#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or attn or paged or med3x" > gpurun_out/pytest_r4k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4k.log
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_attention_k.log 2>&1
timeout 300 python tools/m3dec_time.py > gpurun_out/m3dec_k.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err
echo done
