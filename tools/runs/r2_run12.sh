timeout 1500 tools/ab_variants.sh 3 2 a4s19 a4s16 a5s14 w40 nwa10 2>&1 | grep -E "==|GB/s"
