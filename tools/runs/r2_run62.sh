timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py tests/test_capi.py tests/test_truncate_gpu.py -m gpu -x -q > gpurun_out/t62.log 2>&1; echo tests=$?; tail -3 gpurun_out/t62.log
bash tools/ab_codec.sh 3 b2 2>&1 | grep -v "^{" | cut -c1-400
