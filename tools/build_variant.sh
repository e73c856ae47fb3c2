#!/bin/bash
# build_variant.sh NAME "EXTRA NVCC FLAGS": compile libveloreg_gpu.so with extra
# -D switches into variants/NAME/ (tuning experiments; select with VR_LIB=...).
set -e
NAME=$1; shift
EXTRA="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_1808_04487_b200
OUT=$ROOT/variants/$NAME
mkdir -p "$OUT"
FLAGS="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$ROOT/include -I$PKG/csrc --expt-relaxed-constexpr $EXTRA"
pids=()
for s in blas1 fft fft_axis fft_axis_fused spectral sl objective objective_f32 twolevel postprocess dist capi; do
  /usr/local/cuda/bin/nvcc $FLAGS -c "$PKG/csrc/$s.cu" -o "$OUT/$s.o" -Xptxas -v 2> "$OUT/$s.log" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libveloreg_gpu.so" "$OUT"/*.o -lcudart
echo "built $OUT/libveloreg_gpu.so"
