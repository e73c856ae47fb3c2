#!/bin/bash
# one-rank NCCL slab path: timed ms per matvec for the four overlap settings
# (VR_OVERLAP: reg-term FFT + transposes on the side stream; VR_OVERLAP_HALO: interior planes
# while the halo exchange is in flight)
export VR_DIST_SINGLE_RANK=1
for n in 256 512; do
 for reg in 0 1; do for halo in 0 1; do
  VR_OVERLAP=$reg VR_OVERLAP_HALO=$halo python bench.py --force-slabs --n $n --steps 5 --warmup 3 --no-solve --no-e2e --no-cpu-baseline 2>>gpurun_out/overlap_matrix.err | grep '^{"metric"' | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(json.dumps({'n': $n, 'overlap_reg': $reg, 'overlap_halo': $halo, 'ms_per_matvec': d['ms_per_step'], 'serial_compute_ms': d['comm']['compute_ms_per_matvec'], 'serial_comm_ms': d['comm']['total_ms_per_matvec']}))"
 done; done
done
