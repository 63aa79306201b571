# session 6, call a: final confirmation of HEAD in the driver's order: GPU suite, smoke, default bench (C5, CPU leg), reference arm, secondary configs
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02i_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02i_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/r02i_bench_c5.json 2> gpurun_out/r02i_bench_c5.err; echo "default bench rc=$? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02i_bench_ref.json 2> gpurun_out/r02i_bench_ref.err; echo "reference arm rc=$? wall $(( $(date +%s) - t0 )) s"
for c in c4 c3 c2 c1; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/r02i_bench_$c.json 2> gpurun_out/r02i_bench_$c.err; done
for c in c5 c4 c3 c2 c1; do python -c "
import json; d=json.load(open('gpurun_out/r02i_bench_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],2), d['roofline']['kernel'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],4), d['clocks']['reasons'])"; done
python -c "
import json; d=json.load(open('gpurun_out/r02i_bench_ref.json')); print('ref', d['value'], d['steps'], d['timing']['wall_s'])"
