#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/m3dec_check.py > gpurun_out/m3dec_check.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py tests/test_gpu_fuzz.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider > gpurun_out/pytest_t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t.log
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_t.json 2> gpurun_out/bench_c2_t.err
timeout 400 python bench.py --no-attn --no-cpu --no-e2e --workload c5 --steps 2 > gpurun_out/bench_c5_t.json 2> gpurun_out/bench_c5_t.err
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention and not prefill" > gpurun_out/racecheck_mma.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_mma.log
echo done
