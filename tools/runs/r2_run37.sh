timeout 1500 tools/ab_variants.sh 3 2 old 2>&1 | grep -E "==|GB/s"
HCMX_AB_CACHE_DIR=/tmp timeout 2400 tools/ab_variants.sh 4 1 old 2>&1 | grep -E "==|GB/s"
