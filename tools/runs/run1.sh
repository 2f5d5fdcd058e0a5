set -x
python -m pytest tests -m gpu -x -q > gpurun_out/tests_r2a.log 2>&1; tail -5 gpurun_out/tests_r2a.log
python tools/probe_svd.py > gpurun_out/probe_svd.log 2>&1; cat gpurun_out/probe_svd.log
tools/ab_variants.sh 3 2 nwa12 nwa12u2 u2 nwb8 nwa10u2 nwa14 nwa16u2 > gpurun_out/ab1.log 2>&1; cat gpurun_out/ab1.log
