#!/bin/bash
# Round-2 closing refresh (r02j): bench lines of the final code (default C2,
# c1 / c3 / c5, reference arm), GPU tests, smoke, parity fuzz.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_j.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_j.log
timeout 1200 python bench.py > gpurun_out/bench_j.log 2> gpurun_out/bench_j.err
for wl in c1 c3 c5; do
  timeout 900 python bench.py --workload $wl --no-attn --no-cpu --steps 3 > gpurun_out/bench_j_$wl.log 2> gpurun_out/bench_j_$wl.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_j_ref.log 2>&1
timeout 1200 python tools/fuzz_parity.py --cases 2000 --seed 9001 > gpurun_out/fuzz_parity_j.log 2>&1
echo done
