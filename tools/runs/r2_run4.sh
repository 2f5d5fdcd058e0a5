set -x
timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py tests/test_hmat_gpu.py -x -q -k "codec or compress or aplr or golden or storage" > gpurun_out/t4.log 2>&1; echo tests=$?; tail -3 gpurun_out/t4.log
timeout 900 tools/ab_codec.sh 2 creg
