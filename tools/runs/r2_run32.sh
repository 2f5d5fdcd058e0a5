timeout 1500 tools/ab_variants.sh 3 2 a1big a1big12 2>&1 | grep -E "==|GB/s"
