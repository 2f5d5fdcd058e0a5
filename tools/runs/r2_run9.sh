timeout 1500 tools/ab_variants.sh 3 2 b3s14 b3s12 w50 w0 a3 b12w 2>&1 | grep -E "==|GB/s|mismatch|err"
