HCMX_AB_CACHE_DIR=/tmp timeout 2400 tools/ab_rhs4.sh 4 1 ag4 ag8 2>&1 | grep -E "==|rhs4"
