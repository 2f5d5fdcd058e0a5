#!/bin/bash
# A/B of library variants on the 4-RHS arena of a cached config (profiling aid):
#   tools/ab_rhs4.sh CONFIG REPS tag1 tag2 ...
cfg=$1; reps=$2; shift 2
cache=${HCMX_AB_CACHE_DIR:-/dev/shm}/hmat_c${cfg}.pkl
python tools/prof_hmat.py --config $cfg --iters 3 --cache $cache 2>&1 | tail -1
for r in $(seq $reps); do
  for t in base "$@"; do
    if [ $t = base ]; then lib=paper_2308_10960_b200/libhcmx_gpu.so; else lib=variants/libhcmx_gpu_$t.so; fi
    echo "== $t"
    HCMX_GPU_LIB=$lib python tools/prof_hmat.py --config $cfg --iters 10 --rhs4 --cache $cache 2>&1 | tail -1
  done
done
