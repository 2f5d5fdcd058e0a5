timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t38.log 2>&1; echo tests=$?; tail -2 gpurun_out/t38.log
