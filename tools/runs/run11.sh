timeout 1500 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench=$?; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_" -c 4000 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-codec --no-rhs4 > gpurun_out/ncu_launch_c4.log 2>&1; echo launches=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_phase|k_reduce" -c 3 --csv --log-file gpurun_out/dram_c4.csv \
    python tools/prof_config.py 4 1 > gpurun_out/ncu_dram_c4.log 2>&1; echo dram=$?
tools/ab_variants.sh 3 2 sa18n4 sa18n4i4 sa13n5i4 i6 > gpurun_out/ab11.log 2>&1; cat gpurun_out/ab11.log
timeout 1500 python tools/prof_c5.py > gpurun_out/prof_c5.log 2>&1; tail -3 gpurun_out/prof_c5.log
