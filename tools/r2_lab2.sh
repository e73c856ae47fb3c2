#!/bin/bash
# gather lab 2 (several lanes per point); optional ncu: $1 = kernel regex, $2 = launches to capture
mkdir -p gpurun_out
python tools/gather_lab_inputs.py 256 backward > gpurun_out/lab2_inputs.log 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v tools/gather_lab2.cu -o /tmp/gather_lab2 > gpurun_out/lab2_build.log 2>&1
timeout 300 env ${LAB_T:+LAB_T=1} /tmp/gather_lab2 256 > gpurun_out/lab2.jsonl 2> gpurun_out/lab2.err
if [ -n "$1" ]; then
  timeout 900 ncu --set full --import-source on -k "regex:$1" -c ${2:-1} -o gpurun_out/lab2_ncu -f /tmp/gather_lab2 256 /tmp/lab_X.bin /tmp/lab_f.bin ncu > gpurun_out/ncu_lab2.log 2>&1
fi
cat gpurun_out/lab2.jsonl
echo done
