tools/ab_variants.sh 3 2 nwb4 nwb6 nwb12 bi16k ns4 > gpurun_out/ab3.log 2>&1; cat gpurun_out/ab3.log
timeout 1500 python tools/probe_asm.py 4 > gpurun_out/probe_asm4.log 2>&1; cat gpurun_out/probe_asm4.log
