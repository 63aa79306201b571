mkdir -p gpurun_out
start=$(date +%s)
timeout 1200 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/y_gputests.log 2>&1; echo "tests rc=$? $(( $(date +%s)-start ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/y_c5.json 2> gpurun_out/y_c5.err; echo "bench rc=$? $(( $(date +%s)-start ))s"
