#!/bin/bash
# A/B of library variants on the config-2 codec microbench (bench.codec_microbench:
# L2 flushed before every call, median of CUDA-event times) -- profiling aid:
#   tools/ab_codec.sh REPS tag1 tag2 ...
reps=$1; shift
for r in $(seq $reps); do
  for t in base "$@"; do
    if [ $t = base ]; then lib=paper_2308_10960_b200/libhcmx_gpu.so; else lib=variants/libhcmx_gpu_$t.so; fi
    echo "== $t"
    HCMX_GPU_LIB=$lib python -c "
import json, bench
r = bench.codec_microbench()
print(' '.join(f\"{k}: c {v['compress_gbs']} ({v['compress_frac']}) d {v['decompress_gbs']} ({v['decompress_frac']})\" for k, v in r.items() if isinstance(v, dict)))
"
  done
done
