timeout 1500 tools/ab_variants.sh 3 2 ph1k ph10k ph0 2>&1 | grep -E "==|GB/s"
