#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > /dev/null 2>&1
timeout 120 python tools/enc_timing.py > gpurun_out/enc_timing.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_write tools/ubench_write.cu && (timeout 120 /tmp/ubench_write 256; timeout 120 /tmp/ubench_write 2048) > gpurun_out/ubench_write.log 2>&1
echo done
