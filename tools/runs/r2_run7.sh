set -x
timeout 600 python -m pytest tests/test_codec_gpu.py tests/test_aplr_gpu.py -x -q > gpurun_out/t7.log 2>&1; echo tests=$?; tail -3 gpurun_out/t7.log
timeout 900 tools/ab_codec.sh 1 t16 t4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_compress" -c 1 -o gpurun_out/codec_tma2 python tools/prof_codec_one.py > /dev/null 2>&1; echo ncu=$?
