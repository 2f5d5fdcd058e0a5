set -x
timeout 1500 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 600 --csv --log-file gpurun_out/launches52.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-complex > gpurun_out/ncu_launch52.log 2>&1; echo launches=$?
tail -3 gpurun_out/ncu_launch52.log; wc -l gpurun_out/launches52.csv
