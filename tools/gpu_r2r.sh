#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/split_diag.py 8 > gpurun_out/split_pdl.log 2>&1
HQMQ_NVCC_EXTRA="-DHQMQ_NO_PDL" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
timeout 300 python tools/split_diag.py 8 > gpurun_out/split_nopdl.log 2>&1
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
echo done
