HCMX_AB_CACHE_DIR=/tmp timeout 2400 tools/ab_variants.sh 4 2 b2s46 2>&1 | grep -E "==|GB/s"
