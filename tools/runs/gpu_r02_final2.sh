mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/f2_gputests.log 2>&1; echo "tests rc=$? $(( $(date +%s)-start ))s"; tail -2 gpurun_out/f2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/f2_bench_c5.json 2> gpurun_out/f2_bench_c5.err; echo "bench c5 rc=$? $(( $(date +%s)-start ))s"
for c in c4 c3; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/f2_bench_$c.json 2> gpurun_out/f2_bench_$c.err; echo "bench $c rc=$?"; done
python - <<'PY'
import json
for c in ["c5","c4","c3"]:
    try:
        d=json.load(open(f"gpurun_out/f2_bench_{c}.json"))
        r=d.get("roofline",{}); print(c, d.get("value"), d.get("ms_per_step"), r.get("kernel"), r.get("frac"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("reasons"))
        print("  ", {k: v[0] for k, v in r.get("class_ms_per_step", {}).items()})
    except Exception as e: print(c, "err", e)
PY
