set -x
timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py tests/test_truncate_gpu.py tests/test_formats.py -x -q > gpurun_out/t31.log 2>&1; echo tests=$?; tail -3 gpurun_out/t31.log
timeout 900 tools/ab_codec.sh 2 ureg
