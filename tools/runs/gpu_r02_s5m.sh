# session 5, call m: GEMM core with the half-warp conflict-free k order: GPU suite + C5 / C2 / C4 bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/s5m_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5m_gputests.log
timeout 300 python tools/sketch_engines.py c5 0 2>&1 | tail -1 | cut -c1-400
for c in c5 c2 c3; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/s5m_bench_$c.json 2> gpurun_out/s5m_bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/s5m_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['class_ms_per_step'].get('dmma_gemm'))"; done
