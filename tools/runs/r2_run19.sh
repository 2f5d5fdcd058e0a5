timeout 1500 tools/ab_variants.sh 3 2 a1w16 a1w12 a1w20 2>&1 | grep -E "==|GB/s"
