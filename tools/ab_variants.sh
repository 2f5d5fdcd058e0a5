#!/bin/bash
# A/B of library variants (variants/libhcmx_gpu_<tag>.so, built with
# HCMX_BUILD_TAG=<tag> HCMX_NVCC_DEFS=...) on one cached matrix (profiling aid):
#   tools/ab_variants.sh CONFIG REPS tag1 tag2 ...
cfg=$1; reps=$2; shift 2
cache=${HCMX_AB_CACHE_DIR:-/dev/shm}/hmat_c${cfg}.pkl
python tools/prof_hmat.py --config $cfg --iters 5 --cache $cache --yref ${HCMX_AB_CACHE_DIR:-/dev/shm}/yref_c${cfg}.npy 2>&1 | tail -2
for r in $(seq $reps); do
  for t in base "$@"; do
    if [ $t = base ]; then lib=paper_2308_10960_b200/libhcmx_gpu.so; else lib=variants/libhcmx_gpu_$t.so; fi
    echo "== $t"
    HCMX_GPU_LIB=$lib python tools/prof_hmat.py --config $cfg --iters 50 --cache $cache --yref ${HCMX_AB_CACHE_DIR:-/dev/shm}/yref_c${cfg}.npy 2>&1 | tail -1
  done
done
