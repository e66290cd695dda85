#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_i.log 2> gpurun_out/bench_i.err
timeout 900 python bench.py --workload c5 --no-attn --no-cpu --steps 3 > gpurun_out/bench_i_c5.log 2> gpurun_out/bench_i_c5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_i.log 2>&1
echo done
