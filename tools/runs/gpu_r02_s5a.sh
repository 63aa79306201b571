# session 5, call a: state check of HEAD (phase A on the GEMM core): GPU suite, smoke, C5 bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s5a_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s5a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5a_smoke.log 2>&1; tail -1 gpurun_out/s5a_smoke.log
( time timeout 1200 python bench.py > gpurun_out/s5a_bench_c5.json 2> gpurun_out/s5a_bench_c5.err ) 2>&1 | grep real
( time timeout 900 python bench.py --impl reference > gpurun_out/s5a_bench_ref.json 2> gpurun_out/s5a_bench_ref.err ) 2>&1 | grep real
for c in c5 c4; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1; done
