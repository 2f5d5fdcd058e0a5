timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t40.log 2>&1; echo tests=$?; tail -3 gpurun_out/t40.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke40.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke40.log
timeout 900 python bench.py > gpurun_out/bench40.json 2> gpurun_out/bench40.err; echo bench=$?; head -c 1500 gpurun_out/bench40.json
