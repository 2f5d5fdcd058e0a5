set -x
timeout 900 python -m pytest tests/test_complex.py -x -q > gpurun_out/t15.log 2>&1; echo tests=$?; tail -15 gpurun_out/t15.log
timeout 900 python tools/prof_c5.py 32768 > gpurun_out/c5_32k.log 2>&1; tail -3 gpurun_out/c5_32k.log
