timeout 1500 tools/ab_variants.sh 3 2 nwb10 nwb6 2>&1 | grep -E "==|GB/s"
