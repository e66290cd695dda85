#!/bin/bash
# r3s: fused vs separate Med3x prep, C3 unit timing (+ C2 prep dsqrt fix)
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c3_unit or golden or outlier" > gpurun_out/pytest_r3s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3s.log
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_s_fused.log 2>&1; done
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_s.json 2> gpurun_out/bench_c3_s.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_s.json 2> gpurun_out/bench_c2_s.err
HQMQ_NVCC_EXTRA="-DHQMQ_FUSED_PREP=0" python -m paper_2605_27646_b200.build --force > gpurun_out/build2.log 2>&1
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_s_sep.log 2>&1; done
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_s2.json 2> gpurun_out/bench_c3_s2.err
echo done
