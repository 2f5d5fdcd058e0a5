set -x
timeout 1800 python bench.py > gpurun_out/bench_c4b.json 2> gpurun_out/bench_c4b.err; echo bench=$?; cat gpurun_out/bench_c4b.json; tail -3 gpurun_out/bench_c4b.err
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo ref=$?; cat gpurun_out/ref_c4.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 400 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-rhs4 > gpurun_out/ncu_launch_c4.log 2>&1; echo launches=$?
