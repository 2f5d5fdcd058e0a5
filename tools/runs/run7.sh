HCMX_BUILD_STATS=1 HCMX_VERBOSE=1 timeout 2000 python tools/prof_config.py 4 2 4 8 > gpurun_out/prof_c4.log 2>&1; grep -v "^\[assemble\]" gpurun_out/prof_c4.log | tail -30
