mkdir -p gpurun_out
start=$(date +%s)
for c in c5 c4 c3 c2 c1; do timeout 1200 python bench.py --config $c $( [ $c != c5 ] && echo --no-cpu ) > gpurun_out/f1_bench_$c.json 2> gpurun_out/f1_bench_$c.err; echo "bench $c rc=$? $(( $(date +%s)-start ))s"; done
timeout 1200 python bench.py --impl reference > gpurun_out/f1_bench_ref.json 2> gpurun_out/f1_bench_ref.err; echo "ref rc=$? $(( $(date +%s)-start ))s"
python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/f1_plain_c5.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 6000 --csv --log-file gpurun_out/f1_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/f1_ncu_launch.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import json
for c in ["c5","c4","c3","c2","c1","ref"]:
    try:
        d=json.load(open(f"gpurun_out/f1_bench_{c}.json"))
        r=d.get("roofline",{}); print(c, d.get("value"), d.get("ms_per_step"), r.get("kernel"), r.get("frac"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("reasons"))
    except Exception as e: print(c, "err", e)
PY
