mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/v2i_gputests.log 2>&1; echo "tests rc=$? $(( $(date +%s)-start ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2i_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/v2i_c5.json 2> gpurun_out/v2i_c5.err; echo "bench rc=$? $(( $(date +%s)-start ))s"
tail -3 gpurun_out/v2i_gputests.log; cut -c1-600 gpurun_out/v2i_c5.json
