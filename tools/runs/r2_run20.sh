set -x
timeout 900 python -m pytest tests/test_hmat_gpu.py tests/test_complex.py -x -q > gpurun_out/t20.log 2>&1; echo tests=$?; tail -5 gpurun_out/t20.log
timeout 2400 python tools/prof_c5.py > gpurun_out/c5_full8.log 2>&1; tail -2 gpurun_out/c5_full8.log
