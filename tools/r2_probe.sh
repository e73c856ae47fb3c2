#!/bin/bash
# round-2 probe: gather lab (variants + ncu of the L1 gather and the staged gather) and the
# config-3 solve phase timing. Run from the repo root on the GPU box.
set -x
mkdir -p gpurun_out
python tools/gather_lab_inputs.py 256 backward > gpurun_out/lab_inputs.log 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v tools/gather_lab.cu -o /tmp/gather_lab > gpurun_out/lab_build.log 2>&1
timeout 300 /tmp/gather_lab 256 > gpurun_out/lab.jsonl 2> gpurun_out/lab.err
VR_TIMING=1 timeout 300 python tools/solve_timing.py > gpurun_out/solve_timing.jsonl 2> gpurun_out/solve_timing.err
timeout 600 ncu --set full --import-source on -k regex:k_gather_A -c 1 -o gpurun_out/lab_A -f /tmp/gather_lab 256 > gpurun_out/ncu_lab_A.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_gather_D -c 1 -o gpurun_out/lab_D -f /tmp/gather_lab 256 > gpurun_out/ncu_lab_D.log 2>&1
echo done
