#!/bin/bash
# r3z: Med3x decode, predicated staged payload fix-up
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
for i in 1 2 3; do timeout 300 python tools/m3dec_time.py >> gpurun_out/m3dec_time_z.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider -k "c3_unit or token_ranges or outlier or med3x or golden or adversarial" > gpurun_out/pytest_r3z.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3z.log
timeout 600 python tools/fuzz_parity.py --cases 400 --seed 77 > gpurun_out/fuzz_r3z.log 2>&1
echo done
