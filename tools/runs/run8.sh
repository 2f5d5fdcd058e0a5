tools/ab_variants.sh 3 2 a16x6 a12x6 a24x6 a16x6i4 > gpurun_out/ab8.log 2>&1; cat gpurun_out/ab8.log
HCMX_BUILD_STATS=1 timeout 2000 python tools/prof_config.py 4 8 > gpurun_out/prof_c4b.log 2>&1; grep -v "^\[assemble\]\|^\[build" gpurun_out/prof_c4b.log | tail -20
