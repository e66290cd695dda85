#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python tools/fuzz_parity.py --cases 2000 --seed 2026 > gpurun_out/fuzz_parity.log 2>&1
echo done
