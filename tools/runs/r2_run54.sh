set -x
date +%s
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench54.json 2> gpurun_out/bench54.err; echo bench=$?; head -c 1400 gpurun_out/bench54.json
date +%s
