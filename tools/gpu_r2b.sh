#!/bin/bash
# round 2: GPU test suite + write-bandwidth microbenchmark
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_write tools/ubench_write.cu && (timeout 120 /tmp/ubench_write 256; timeout 120 /tmp/ubench_write 2048) > gpurun_out/ubench_write.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
