mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/v2t_gputests.log 2>&1; echo "tests rc=$? $(( $(date +%s)-start ))s"; tail -2 gpurun_out/v2t_gputests.log
timeout 1200 python bench.py > gpurun_out/v2t_c5.json 2> gpurun_out/v2t_c5.err; echo "bench c5 rc=$? $(( $(date +%s)-start ))s"
for c in c4 c3; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/v2t_$c.json 2> gpurun_out/v2t_$c.err; echo "bench $c rc=$?"; done
python - <<'PY'
import json
for c in ["c5","c4","c3"]:
    try:
        d=json.load(open(f"gpurun_out/v2t_{c}.json"))
        r=d["roofline"]; print(c, d["value"], d["ms_per_step"], r["kernel"], round(r["frac"],3), d["e2e"]["value"], d["clocks"]["reasons"])
    except Exception as e: print(c, "err", e)
PY
