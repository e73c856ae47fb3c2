#!/bin/bash
mkdir -p gpurun_out
RUNS=12 VR_TIMING=1 timeout 400 python tools/solve_timing.py > gpurun_out/solve_timing2.jsonl 2> gpurun_out/solve_timing2.err
timeout 120 python tools/pcie_probe.py > gpurun_out/pcie.json 2>&1
N=256 timeout 300 python tools/cufft_compare.py > gpurun_out/cufft256.jsonl 2>&1
N=512 timeout 300 python tools/cufft_compare.py > gpurun_out/cufft512.jsonl 2>&1
echo done
