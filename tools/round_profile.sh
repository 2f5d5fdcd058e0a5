#!/bin/bash
# Round-end evidence on one GPU (profiling aid): gpu tests, the bench line,
# the reference arm, the ncu launch list of the bench command and one
# `--set full` capture of the phase kernels.  Outputs under gpurun_out/.
set -x
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -2 gpurun_out/tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:^k_ -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo launches=$?
python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -o gpurun_out/phase_full \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > gpurun_out/ncu_full.log 2>&1; echo full=$?
