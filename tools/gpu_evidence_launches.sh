CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-solve --no-cpu-baseline --no-config4 --no-config2 --no-fp32"
timeout 600 $CMD > gpurun_out/launch_cmd.json 2> gpurun_out/launch_cmd.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_incstate_step|k_adjoint_step|k_accumulate" \
   -s 12 -c 3 -o gpurun_out/ncu_top -f $CMD > gpurun_out/ncu_top.log 2>&1
echo done > gpurun_out/ev2.done
