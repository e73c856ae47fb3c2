# GPU sweep: parity of both gather paths, then matvec timings of the default build and variants/*
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_smem.log 2>&1; echo rc=$? >> gpurun_out/gputests_smem.log
[ -n "$SKIP_TESTS" ] || VR_GATHER=global timeout 600 python -m pytest tests -m gpu -x -q -k "transport or objective or golden" > gpurun_out/gputests_global.log 2>&1; echo rc=$? >> gpurun_out/gputests_global.log
: > gpurun_out/vb.jsonl
VR_GATHER=global timeout 300 python tools/variant_bench.py >> gpurun_out/vb.jsonl 2>>gpurun_out/vb.err
timeout 300 python tools/variant_bench.py >> gpurun_out/vb.jsonl 2>>gpurun_out/vb.err
for v in variants/*/; do VR_LIB=$v/libveloreg_gpu.so timeout 300 python tools/variant_bench.py >> gpurun_out/vb.jsonl 2>>gpurun_out/vb.err; done
