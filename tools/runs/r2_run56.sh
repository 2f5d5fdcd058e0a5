python tools/prof_hmat.py --config 4 --iters 3 --cache /dev/shm/hmat_c4.pkl 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_phase_a" -c 1 -f -o gpurun_out/r2_phase_a_c4_v56 \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /dev/shm/hmat_c4.pkl > gpurun_out/ncu_full56.log 2>&1; echo full=$?
