set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t10.log 2>&1; echo tests=$?; tail -5 gpurun_out/t10.log
timeout 900 tools/ab_variants.sh 3 2 old 2>&1 | grep -E "==|GB/s"
