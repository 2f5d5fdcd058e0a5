timeout 1500 tools/ab_variants.sh 3 2 b2s44 b4s18 2>&1 | grep -E "==|GB/s"
