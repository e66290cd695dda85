#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_err.log 2>&1
timeout 900 python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py tests/test_gpu_attention_shapes.py -q -p no:cacheprovider > gpurun_out/pytest_med3x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_med3x.log
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_occ.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,launch__waves_per_multiprocessor,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'decode_fast' -s 3 -c 2 python tools/prof_unit.py --reps 5 --attn-batch 0 > gpurun_out/ncu_dec_occ.log 2>&1
echo done
