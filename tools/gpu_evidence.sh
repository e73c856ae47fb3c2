# round evidence: bench line, reference arm, ncu launch list of the same command, one ncu --set full
# capture of the dominant kernel (each ncu pass only after its own command ran clean without ncu)
set -x
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo bench=$? >> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-solve --no-cpu-baseline --no-config4"
timeout 600 $CMD > gpurun_out/launch_cmd.json 2> gpurun_out/launch_cmd.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_incstate_step|k_adjoint_step|k_accumulate" \
   -s 12 -c 3 -o gpurun_out/ncu_top -f $CMD > gpurun_out/ncu_top.log 2>&1
echo done >> gpurun_out/bench_final.err
