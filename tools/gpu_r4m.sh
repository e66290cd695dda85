#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python tools/attn_cmp.py > gpurun_out/attn_cmp_m.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or attn or paged" > gpurun_out/pytest_r4m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4m.log
echo done
