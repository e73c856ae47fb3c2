#!/bin/bash
# gather lab only (inputs + variants); optional ncu of one variant: $1 = kernel regex
mkdir -p gpurun_out
python tools/gather_lab_inputs.py 256 backward > gpurun_out/lab_inputs.log 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v tools/gather_lab.cu -o /tmp/gather_lab > gpurun_out/lab_build.log 2>&1
timeout 300 /tmp/gather_lab 256 > gpurun_out/lab.jsonl 2> gpurun_out/lab.err
if [ -n "$1" ]; then
  timeout 600 ncu --set full --import-source on -k "regex:$1" -c 1 -o gpurun_out/lab_ncu -f /tmp/gather_lab 256 > gpurun_out/ncu_lab.log 2>&1
fi
echo done
