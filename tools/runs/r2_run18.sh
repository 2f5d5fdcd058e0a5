# config-4 evidence after the interleaved arena: per-rank partition emulation,
# DRAM traffic per phase kernel, one --set full capture of the phase kernels
timeout 1500 python tools/prof_config.py 4 2 4 8 > gpurun_out/part_c4b.log 2>&1; grep -E "^N=|build_config|hmat_create" gpurun_out/part_c4b.log
python tools/prof_hmat.py --config 4 --iters 3 --cache /tmp/hmat_c4.pkl 2>&1 | tail -1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum --clock-control none -k regex:"k_phase|k_reduce" -c 3 --csv --log-file gpurun_out/dram_c4b.csv \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /tmp/hmat_c4.pkl > /dev/null 2>&1; echo dram=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_phase" -c 2 -o gpurun_out/r2_phase_full_c4 \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /tmp/hmat_c4.pkl > /dev/null 2>&1; echo full=$?
