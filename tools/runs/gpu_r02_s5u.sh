# session 5, call u: proxy fence also in the GEMM core and the 64 x 64-tile phase B consumers: GPU suite, smoke, bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02h_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in c5 c3 c2; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/r02h_bench_$c.json 2> gpurun_out/r02h_bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02h_bench_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],2), d['roofline']['kernel'], round(d['roofline']['frac'],3))"; done
