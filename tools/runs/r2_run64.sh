timeout 900 python -m pytest tests/test_hmat_gpu.py tests/test_parity_bench.py tests/test_complex.py -m gpu -x -q > gpurun_out/t64.log 2>&1; echo tests=$?; tail -3 gpurun_out/t64.log
HCMX_BUILD_STATS=1 python tools/prof_hmat.py --config 3 --iters 2 2>&1 | grep "build" | head -4
bash tools/ab_variants.sh 3 2 lo sg32 sg30 2>&1 | grep -v "^{" | cut -c1-260
bash tools/ab_variants.sh 4 1 lo sg32 sg30 2>&1 | grep -v "^{" | cut -c1-260
