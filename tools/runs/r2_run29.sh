set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t29.log 2>&1; echo tests=$?; tail -2 gpurun_out/t29.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?; tail -2 gpurun_out/bench_final.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo ref=$?; cat gpurun_out/ref_final.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 600 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-complex > gpurun_out/ncu_launch_final.log 2>&1; echo launches=$?
