timeout 1500 tools/ab_variants.sh 3 2 b2s44 b2s46 b2s40 ab2 2>&1 | grep -E "==|GB/s"
