timeout 1500 tools/ab_variants.sh 3 2 bi16 bi12 bg64 2>&1 | grep -E "==|GB/s"
