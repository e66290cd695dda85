#!/bin/bash
# r3o: decode error-word fix (flagged chunks' skipped code slots), C3/C1 re-bench
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c3_unit or token_ranges" > gpurun_out/pytest_r3o_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3o_k.log
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_o.json 2> gpurun_out/bench_c3_o.err
timeout 300 python bench.py --no-cpu --workload c1 > gpurun_out/bench_c1_o.json 2> gpurun_out/bench_c1_o.err
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3o.log
echo done
