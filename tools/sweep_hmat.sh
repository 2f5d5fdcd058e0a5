#!/bin/bash
# build-parameter sweep of the matvec kernels on one config (profiling aid):
#   tools/sweep_hmat.sh "-DHCMX_NWA=8" "-DHCMX_NWA=12" ...
# the compressed matrix is cached in /tmp between variants
cfg=${CFG:-3}
for defs in "$@"; do
  HCMX_NVCC_DEFS="$defs" python -m paper_2308_10960_b200.build -f > /dev/null || { echo "build failed: $defs"; continue; }
  echo "== $defs"
  python tools/prof_hmat.py --config $cfg --iters 50 --cache /tmp/hmat_c$cfg.pkl 2>&1 | tail -1
done
python -m paper_2308_10960_b200.build -f > /dev/null
