HCMX_PROF_BUILD=1 python -m paper_2308_10960_b200.build -f > /dev/null
for dbg in 0 1 2; do
  echo "== HCMX_DEBUG=$dbg"
  HCMX_PROF=1 HCMX_DEBUG=$dbg python tools/prof_hmat.py --config 3 --iters 3 --cache /tmp/hmat_c3.pkl 2>&1 | grep -E "prof|phaseA" | tail -5
done
