#!/bin/bash
# r4a: two-pass median + race fix validation
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r4a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4a.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 888 > gpurun_out/fuzz_r4a.log 2>&1
timeout 300 python tools/c3_unit.py 40 > gpurun_out/c3_unit_r4a.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_r4a.json 2> gpurun_out/bench_c3_r4a.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_r4a.json 2> gpurun_out/bench_c1_r4a.err
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit" \
  > gpurun_out/sanitize_racecheck_median.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck_median.log
echo done
