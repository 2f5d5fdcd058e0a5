set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t24.log 2>&1; echo tests=$?; tail -3 gpurun_out/t24.log
python tools/prof_hmat.py --config 3 --iters 20 --rhs4 --cache /tmp/hmat_c3.pkl 2>&1 | tail -2
