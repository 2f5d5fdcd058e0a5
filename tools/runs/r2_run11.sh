python tools/prof_hmat.py --config 3 --iters 5 --cache /tmp/hmat_c3.pkl 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_phase" -c 2 -o gpurun_out/r2_phase_full_c3b \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > gpurun_out/ncu_full_c3b.log 2>&1; echo full=$?
