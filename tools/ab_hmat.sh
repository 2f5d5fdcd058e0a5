#!/bin/bash
# A/B of two hmat.cu versions on the cached config-3 matrix (profiling aid):
#   tools/ab_hmat.sh OLD.cu   (compares against the working tree)
old=$1
cp paper_2308_10960_b200/csrc/hmat.cu /tmp/hmat_new.cu
for v in new old new old; do
  if [ $v = old ]; then cp $old paper_2308_10960_b200/csrc/hmat.cu; else cp /tmp/hmat_new.cu paper_2308_10960_b200/csrc/hmat.cu; fi
  python -m paper_2308_10960_b200.build -f > /dev/null 2>&1 || echo "build failed $v"
  echo "== $v"; python tools/prof_hmat.py --config 3 --iters 50 --cache /tmp/hmat_c3.pkl 2>&1 | tail -1
done
cp /tmp/hmat_new.cu paper_2308_10960_b200/csrc/hmat.cu
python -m paper_2308_10960_b200.build -f > /dev/null
