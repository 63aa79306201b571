mkdir -p gpurun_out
start=$(date +%s)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --durations=30 > gpurun_out/v2a_gputests.log 2>&1; echo "tests rc=$? $(( $(date +%s)-start ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/v2a_c5.json 2> gpurun_out/v2a_c5.err; echo "bench rc=$? $(( $(date +%s)-start ))s"
tail -3 gpurun_out/v2a_gputests.log; cat gpurun_out/v2a_c5.json
