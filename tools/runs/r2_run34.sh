python tools/prof_hmat.py --config 4 --iters 3 --cache /tmp/hmat_c4.pkl 2>&1 | tail -1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_phase_b" -c 1 -o gpurun_out/r2_phase_b_c4_2slot \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /tmp/hmat_c4.pkl > /dev/null 2>&1; echo full=$?
