# profiling pass: config-3 full ncu capture of the phase kernels (source-level),
# config-4 DRAM traffic per phase kernel, staging-only (HCMX_DEBUG=1) timing,
# config-4 per-rank partition emulation
set -x
python tools/prof_hmat.py --config 3 --iters 5 --cache /tmp/hmat_c3.pkl 2>&1 | tail -3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_phase|k_reduce" -c 3 -o gpurun_out/r2_phase_full_c3 \
    python tools/prof_hmat.py --config 3 --iters 1 --cache /tmp/hmat_c3.pkl > gpurun_out/ncu_full_c3.log 2>&1; echo full=$?
python tools/prof_hmat.py --config 4 --iters 5 --cache /tmp/hmat_c4.pkl 2>&1 | tail -3
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_phase|k_reduce" -c 3 --csv --log-file gpurun_out/dram_c4.csv \
    python tools/prof_hmat.py --config 4 --iters 1 --cache /tmp/hmat_c4.pkl > gpurun_out/ncu_dram_c4.log 2>&1; echo dram=$?
HCMX_PROF_BUILD=1 python -m paper_2308_10960_b200.build -f > /dev/null
for dbg in 0 1; do
  echo "== HCMX_DEBUG=$dbg"
  HCMX_PROF=1 HCMX_DEBUG=$dbg python tools/prof_hmat.py --config 4 --iters 3 --cache /tmp/hmat_c4.pkl 2>&1 | grep -E "prof|phase" | tail -6
done
python -m paper_2308_10960_b200.build -f > /dev/null
timeout 900 python tools/prof_config.py 4 2 4 8 > gpurun_out/part_c4.log 2>&1; tail -20 gpurun_out/part_c4.log
