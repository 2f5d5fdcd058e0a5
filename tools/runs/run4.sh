timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_r2b.log 2>&1; tail -3 gpurun_out/tests_r2b.log
tools/ab_variants.sh 3 2 prev > gpurun_out/ab4.log 2>&1; cat gpurun_out/ab4.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -o gpurun_out/phase_r2a \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > gpurun_out/ncu_r2a.log 2>&1; echo full=$?
timeout 900 python tools/probe_asm.py 4 262144 > gpurun_out/probe_asm4b.log 2>&1; cat gpurun_out/probe_asm4b.log
