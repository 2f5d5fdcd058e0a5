set -x
timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py -x -q > gpurun_out/t5.log 2>&1; echo tests=$?; tail -3 gpurun_out/t5.log
timeout 900 tools/ab_codec.sh 2 creg t4 t16
