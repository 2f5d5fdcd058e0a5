for defs in "-DHCMX_AGROUP_MULTI=1" "-DHCMX_AGROUP_MULTI=2" "-DHCMX_AGROUP_MULTI=4"; do
  HCMX_NVCC_DEFS="$defs" python -m paper_2308_10960_b200.build -f > /dev/null
  echo "== $defs"; HCMX_BUILD_STATS=1 python tools/prof_hmat.py --config 3 --iters 10 --cache /tmp/hmat_c3.pkl --rhs4 2>&1 | grep -E "build A|rhs4" | tail -2
done
