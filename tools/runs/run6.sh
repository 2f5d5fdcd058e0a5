python tools/probe_cpu.py > gpurun_out/probe_cpu.log 2>&1; cat gpurun_out/probe_cpu.log
tools/ab_variants.sh 3 2 c3 c3b c2s2 > gpurun_out/ab6.log 2>&1; cat gpurun_out/ab6.log
timeout 1500 python tools/probe_c4.py 4 > gpurun_out/probe_c4b.log 2>&1; tail -12 gpurun_out/probe_c4b.log
