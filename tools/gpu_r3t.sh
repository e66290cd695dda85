#!/bin/bash
# r3t: sampled-bracket Med3x median
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adversarial or c3_unit or golden or outlier or per_head or vs_oracle" > gpurun_out/pytest_r3t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3t.log
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3t_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3t_all.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 321 > gpurun_out/fuzz_r3t.log 2>&1
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_t.log 2>&1; done
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_t.json 2> gpurun_out/bench_c3_t.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_t.json 2> gpurun_out/bench_c1_t.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'median' -s 8 -c 4 \
   -o gpurun_out/prof_median_t -f python tools/c3_unit.py 3 > gpurun_out/prof_median_t.log 2>&1
echo done
