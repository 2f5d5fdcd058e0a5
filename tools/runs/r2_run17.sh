set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 2400 python bench.py --steps 20 --no-codec --no-rhs4 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err; echo bench=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_t.json')); print(d['value'], d['ms_per_step'], d['parity'], d['complex'])"; tail -3 gpurun_out/bench_t.err
