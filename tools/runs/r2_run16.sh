set -x
timeout 900 python -m pytest tests/test_complex.py -x -q > gpurun_out/t16.log 2>&1; echo tests=$?; tail -3 gpurun_out/t16.log
timeout 2400 python tools/prof_c5.py > gpurun_out/c5_full.log 2>&1; tail -3 gpurun_out/c5_full.log
