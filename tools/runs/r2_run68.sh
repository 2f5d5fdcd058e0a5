timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t68.log 2>&1; echo tests=$?; tail -2 gpurun_out/t68.log
python tools/prof_hmat.py --config 3 --iters 50 --cache /dev/shm/hmat_c3.pkl --yref /dev/shm/yref_c3.npy 2>&1 | tail -1
python tools/prof_hmat.py --config 4 --iters 5 --cache /dev/shm/hmat_c4.pkl --yref /dev/shm/yref_c4.npy 2>&1 | tail -1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench68.json 2> gpurun_out/bench68.err; echo bench=$?; head -c 600 gpurun_out/bench68.json
