set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t8.log 2>&1; echo tests=$?; tail -3 gpurun_out/t8.log
timeout 900 tools/ab_codec.sh 1
