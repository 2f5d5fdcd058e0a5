for t in base cold creg; do
  if [ $t = base ]; then lib=paper_2308_10960_b200/libhcmx_gpu.so; else lib=variants/libhcmx_gpu_$t.so; fi
  HCMX_GPU_LIB=$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_compress|k_unpack" -c 4 -o gpurun_out/codec_$t python tools/prof_codec_one.py > gpurun_out/ncu_codec_$t.log 2>&1; echo $t=$?
done
