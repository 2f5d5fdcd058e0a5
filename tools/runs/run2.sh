python tools/probe_svd2.py > gpurun_out/probe_svd2.log 2>&1; cat gpurun_out/probe_svd2.log
tools/ab_variants.sh 3 2 nwb4 nwb6 nwb8 nwb10 nwb8bi nwa6 nwa4 > gpurun_out/ab2.log 2>&1; cat gpurun_out/ab2.log
