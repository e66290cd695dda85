#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r4l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4l.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r4l.log 2>&1
timeout 900 python tools/fuzz_parity.py --cases 800 --seed 2718 > gpurun_out/fuzz_r4l.log 2>&1
timeout 300 python tools/c3_unit.py 40 > gpurun_out/c3_unit_l.log 2>&1
echo done
