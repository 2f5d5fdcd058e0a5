set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t50.log 2>&1; echo tests=$?; tail -3 gpurun_out/t50.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke50.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke50.log
timeout 1200 python bench.py > gpurun_out/bench50.json 2> gpurun_out/bench50.err; echo bench=$?; head -c 2500 gpurun_out/bench50.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref50.json 2> gpurun_out/ref50.err; echo ref=$?; cat gpurun_out/ref50.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:^k_ -c 3000 --csv --log-file gpurun_out/launches50.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench50.log 2>&1; echo launches=$?
python tools/prof_hmat.py --config 4 --iters 3 --cache /dev/shm/hmat_c4.pkl 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -f -o gpurun_out/r2_phase_full_c4_v50 \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /dev/shm/hmat_c4.pkl > gpurun_out/ncu_full50.log 2>&1; echo full=$?
