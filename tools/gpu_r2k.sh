#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_err.log 2>&1
timeout 900 python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py tests/test_gpu_attention_shapes.py -q -p no:cacheprovider > gpurun_out/pytest_med3x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_med3x.log
timeout 120 python tools/enc_timing.py > gpurun_out/enc_timing.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_occ.json 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_occ.json 2>&1
echo done
