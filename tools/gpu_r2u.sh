#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/m3dec_check.py > gpurun_out/m3dec_check.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_u.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_u.log
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_u.json 2> gpurun_out/bench_c2_u.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_u.json 2> gpurun_out/bench_c3_u.err
timeout 300 python tools/attn_cmp.py > gpurun_out/attn_cmp.log 2>&1
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_err.log 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention and not prefill or token_ranges or golden and s64" > gpurun_out/racecheck_mma.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_mma.log
echo done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_med3x_serving.py -x -q -p no:cacheprovider -k "1032 or 2048" > gpurun_out/racecheck_med3x.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_med3x.log
