set -x
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_hmat_gpu.py -m gpu -x -q -k "golden_hmatrix or rank_zero or alpha_zero" > gpurun_out/san_$tool.log 2>&1; echo $tool=$?
grep -c "ERROR SUMMARY\|Race reported\|RACECHECK SUMMARY" gpurun_out/san_$tool.log; grep "SUMMARY" gpurun_out/san_$tool.log | tail -3; tail -2 gpurun_out/san_$tool.log
done
