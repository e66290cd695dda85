#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/pcie_bw.py > gpurun_out/pcie.log 2>&1
echo done
