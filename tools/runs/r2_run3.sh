set -x
timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py -x -q > gpurun_out/t3.log 2>&1; echo tests=$?; tail -3 gpurun_out/t3.log
timeout 900 tools/ab_codec.sh 2 u3 u2
