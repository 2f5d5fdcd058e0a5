set -x
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench51.json 2> gpurun_out/bench51.err; echo bench=$?; head -c 1800 gpurun_out/bench51.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 600 --csv --log-file gpurun_out/launches51.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-complex > gpurun_out/ncu_launch51.log 2>&1; echo launches=$?
tail -3 gpurun_out/ncu_launch51.log
