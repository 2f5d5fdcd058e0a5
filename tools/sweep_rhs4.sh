#!/bin/bash
# build-parameter sweep of the 4-RHS arena on the cached config-3 matrix (profiling aid)
for defs in "$@"; do
  HCMX_NVCC_DEFS="$defs" python -m paper_2308_10960_b200.build -f > /dev/null || { echo "build failed: $defs"; continue; }
  echo "== $defs"; python tools/prof_hmat.py --config 3 --iters 10 --cache /tmp/hmat_c3.pkl --rhs4 2>&1 | grep rhs4
done
python -m paper_2308_10960_b200.build -f > /dev/null
