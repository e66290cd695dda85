#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/prefill_err.py > gpurun_out/prefill_err.log 2>&1
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
echo done
