# GPU sweep: GPU tests (unless SKIP_TESTS), then config-3 matvec timings of the default
# build and of every variants/*/libveloreg_gpu.so (tools/build_variant.sh)
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
: > gpurun_out/vb.jsonl
timeout 300 python tools/variant_bench.py >> gpurun_out/vb.jsonl 2>>gpurun_out/vb.err
for v in variants/*/; do VR_LIB=$v/libveloreg_gpu.so timeout 300 python tools/variant_bench.py >> gpurun_out/vb.jsonl 2>>gpurun_out/vb.err; done
