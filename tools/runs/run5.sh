python tools/debug_codec_dev.py > gpurun_out/dbg_codec.log 2>&1; cat gpurun_out/dbg_codec.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/tests_r2c.log 2>&1; tail -8 gpurun_out/tests_r2c.log
tools/ab_variants.sh 3 2 prev > gpurun_out/ab5.log 2>&1; cat gpurun_out/ab5.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -o gpurun_out/phase_r2a \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > gpurun_out/ncu_r2a.log 2>&1; echo full=$?
timeout 1500 python tools/probe_asm.py 4 > gpurun_out/probe_asm4c.log 2>&1; cat gpurun_out/probe_asm4c.log
