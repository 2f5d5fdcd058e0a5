timeout 900 python bench.py --gpus 1 --config 3 --steps 20 --warmup 5 --no-complex > gpurun_out/bench60_c3.json 2> gpurun_out/bench60_c3.err; echo bench=$?; head -c 1500 gpurun_out/bench60_c3.json
