#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 120 python tools/c3_unit.py 20 > gpurun_out/c3_unit.log 2>&1
timeout 600 python tools/fuzz_parity.py --cases 300 > gpurun_out/fuzz_parity.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --workload c3 > gpurun_out/bench_c3_r3d.json 2> gpurun_out/bench_c3_r3d.err
timeout 300 python bench.py --no-attn --no-cpu --workload c1 > gpurun_out/bench_c1_r3d.json 2> gpurun_out/bench_c1_r3d.err
echo done
