timeout 1500 tools/ab_variants.sh 3 2 ac6 ac5 2>&1 | grep -E "==|GB/s"
