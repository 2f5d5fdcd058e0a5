timeout 900 python -m pytest tests/test_hmat_gpu.py tests/test_parity_bench.py tests/test_complex.py -m gpu -x -q > gpurun_out/t42.log 2>&1; echo tests=$?; tail -3 gpurun_out/t42.log
bash tools/ab_variants.sh 3 2 bpf0 u4 2>&1 | grep -v "^{" 
bash tools/ab_variants.sh 4 2 bpf0 2>&1 | grep -v "^{"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_phase" -c 2 -f -o gpurun_out/r2_phase_full_c3_v42 \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /dev/shm/hmat_c3.pkl > gpurun_out/ncu_full42.log 2>&1; echo full=$?
