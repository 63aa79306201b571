# session 5, call l: measurement set r02g (all configs + reference arm + GPU suite + smoke + C5 launch list)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02g_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02g_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02g_smoke.log 2>&1; tail -1 gpurun_out/r02g_smoke.log
for c in c5 c4 c3 c2 c1; do ( time timeout 900 python bench.py --config $c > gpurun_out/r02g_bench_$c.json 2> gpurun_out/r02g_bench_$c.err ) 2>&1 | grep real; done
( time timeout 900 python bench.py --impl reference > gpurun_out/r02g_bench_ref.json 2> gpurun_out/r02g_bench_ref.err ) 2>&1 | grep real
python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r02g_plain.json 2> gpurun_out/r02g_plain.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02g_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r02g_ncu.log 2>&1; echo "ncu rc=$?"
wc -l gpurun_out/r02g_launches_c5.csv
python tools/parity_report.py > gpurun_out/r02g_parity_table.json 2> gpurun_out/r02g_parity.err; echo "parity rc=$?"
