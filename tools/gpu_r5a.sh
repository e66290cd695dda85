#!/bin/bash
# r5a: second median pass compacts by the first pass's recorded bin indices
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py -q -x -p no:cacheprovider > gpurun_out/pytest_r5a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r5a.log
timeout 900 python tools/fuzz_parity.py --cases 2000 --seed 5150 > gpurun_out/fuzz_r5a.log 2>&1
rm -f gpurun_out/c3_r5a.log
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_r5a.log 2>&1; done
timeout 300 python tools/c1_unit.py >> gpurun_out/c3_r5a.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_r5a.json 2> /dev/null
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit or per_head" > gpurun_out/memcheck_r5a.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_r5a.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit" > gpurun_out/racecheck_r5a.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_r5a.log
echo done
