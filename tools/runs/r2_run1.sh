set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_r2a.log 2>&1; echo tests=$?; tail -5 gpurun_out/tests_r2a.log
timeout 1800 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench=$?; cat gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
