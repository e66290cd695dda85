#!/bin/bash
# long randomized parity runs on the final library
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python tools/fuzz_parity.py --cases 6000 --seed 20261017 > gpurun_out/fuzz_parity_long.log 2>&1
timeout 2400 python tools/fuzz_attention.py --cases 300 --seed 20261017 > gpurun_out/fuzz_attention_long.log 2>&1
echo done
