#!/bin/bash
# round-2b evidence, bench part (one GPU): smoke, bench (ours + reference arm), the one-rank NCCL
# run of the multi-GPU path, the ncu launch list and a compact ncu --set full capture
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2b_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_bench_ref.json 2> gpurun_out/r2b_bench_ref.err
VR_DIST_SINGLE_RANK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 1 --steps 10 --warmup 3 --force-slabs --slab-two-level > gpurun_out/r2b_forced_slabs_256.json 2> gpurun_out/r2b_forced_slabs_256.err
Q="--no-solve --no-fp32 --no-config2 --no-config4 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py --steps 2 --warmup 3 $Q > gpurun_out/r2b_launch_cmd.json 2> gpurun_out/r2b_launch_cmd.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 $Q > gpurun_out/r2b_ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_incstate_step|k_adjoint_step|k_accumulate|k_fft_axis|k_c2r_rows|k_r2c_rows" --launch-skip 40 -c 6 -o gpurun_out/r2b_matvec_full -f python bench.py --steps 2 --warmup 3 $Q > gpurun_out/r2b_ncu_full.log 2>&1
ls -la gpurun_out
echo done
