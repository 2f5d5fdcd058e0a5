rm -f /tmp/yref_c3.npy /dev/shm/hmat_c3.pkl
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests_r2d.log 2>&1; tail -4 gpurun_out/tests_r2d.log
tools/ab_variants.sh 3 2 prev > gpurun_out/ab9.log 2>&1; cat gpurun_out/ab9.log
HCMX_BUILD_STATS=1 timeout 2000 python tools/prof_config.py 4 2 4 8 > gpurun_out/prof_c4c.log 2>&1; grep -v "^\[assemble\]\|^\[build" gpurun_out/prof_c4c.log | tail -24
