# FFT pass variants: cuFFT comparison numbers + config-3 matvec per variant (256^3) and 512^3 passes
: > gpurun_out/fft_sweep.jsonl
for lib in paper_1808_04487_b200/libveloreg_gpu.so variants/*/libveloreg_gpu.so; do
  for n in 256 512; do
    VR_LIB=$lib N=$n timeout 300 python tools/cufft_compare.py | sed "s|^{|{\"lib\": \"$lib\", |" >> gpurun_out/fft_sweep.jsonl 2>>gpurun_out/fft_sweep.err
  done
  VR_LIB=$lib STEPS=20 timeout 300 python tools/variant_bench.py >> gpurun_out/fft_sweep.jsonl 2>>gpurun_out/fft_sweep.err
done
