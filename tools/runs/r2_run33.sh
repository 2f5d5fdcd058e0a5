timeout 900 python -m pytest tests/test_hmat_gpu.py tests/test_complex.py -x -q -k "transposed or schemes" > gpurun_out/t33.log 2>&1; echo tests=$?; tail -15 gpurun_out/t33.log
