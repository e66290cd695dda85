#!/bin/bash
# r4f: NVML clock sampler in bench.py
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r4f.json 2> gpurun_out/bench_r4f.err
timeout 300 python bench.py --workload c1 --no-attn --no-cpu > gpurun_out/bench_c1_r4f.json 2> gpurun_out/bench_c1_r4f.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r4f.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r4f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4f.log
echo done
