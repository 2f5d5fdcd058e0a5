timeout 900 python -m pytest tests/test_hmat_gpu.py tests/test_parity_bench.py -m gpu -x -q > gpurun_out/t48.log 2>&1; echo tests=$?; tail -3 gpurun_out/t48.log
bash tools/ab_variants.sh 3 2 nopf 2>&1 | grep -v "^{" 
bash tools/ab_variants.sh 4 2 nopf 2>&1 | grep -v "^{"
