mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
for c in c2 c1 c3 c4 c5; do timeout 900 python bench.py --config $c > gpurun_out/r01f_bench_$c.json 2> gpurun_out/r01f_bench_$c.err; done
timeout 900 python bench.py --impl reference > gpurun_out/r01f_bench_ref.json 2> gpurun_out/r01f_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01f_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
