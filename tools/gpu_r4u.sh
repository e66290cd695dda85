#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
timeout 900 python tools/fuzz_parity.py --cases 1500 --seed 777 > gpurun_out/fuzz_final.log 2>&1
timeout 900 python tools/fuzz_attention.py --cases 150 --seed 777 > gpurun_out/fuzz_attn_final.log 2>&1
echo done
