#!/bin/bash
# r4h: sample bracket merged into the first median pass
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4h.log
timeout 900 python tools/fuzz_parity.py --cases 1500 --seed 4711 > gpurun_out/fuzz_r4h.log 2>&1
timeout 300 python tools/c1_unit.py > gpurun_out/c1_unit_h.log 2>&1
timeout 300 python tools/c3_unit.py 40 > gpurun_out/c3_unit_h.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_h.json 2> gpurun_out/bench_c1_h.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_h.json 2> gpurun_out/bench_c3_h.err
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit" > gpurun_out/racecheck_r4h.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_r4h.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit or per_head" > gpurun_out/memcheck_r4h.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_r4h.log
echo done
