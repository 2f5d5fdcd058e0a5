HCMX_PROF_BUILD=1 python -m paper_2308_10960_b200.build -f > /dev/null
for dbg in 0 1; do
  echo "== HCMX_DEBUG=$dbg"
  HCMX_PROF=1 HCMX_DEBUG=$dbg python tools/prof_hmat.py --config 3 --iters 3 --cache /tmp/hmat_c3.pkl 2>&1 | grep -E "prof|phase" | tail -6
done
python -m paper_2308_10960_b200.build -f > /dev/null
HCMX_BUILD_STATS=1 python tools/prof_hmat.py --config 3 --iters 3 --cache /tmp/hmat_c3.pkl 2>&1 | grep -v "^n=" | tail -30
