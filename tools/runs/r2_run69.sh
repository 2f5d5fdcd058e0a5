python tools/prof_hmat.py --config 4 --iters 3 --cache /dev/shm/hmat_c4.pkl 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -f -o gpurun_out/r2_phase_full_c4_v69 \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /dev/shm/hmat_c4.pkl > gpurun_out/ncu_full69.log 2>&1; echo full=$?
timeout 1500 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 600 --csv --log-file gpurun_out/launches69.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-complex > gpurun_out/ncu_launch69.log 2>&1; echo launches=$?
timeout 900 python bench.py --gpus 1 --config 3 --steps 20 --warmup 5 --no-complex > gpurun_out/bench69_c3.json 2> gpurun_out/bench69_c3.err; echo bench3=$?
