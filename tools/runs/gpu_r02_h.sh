python tools/matvec_one.py c5 1 > gpurun_out/mv5.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"phbg|phb2|pha_all" -c 3 --csv --log-file gpurun_out/mv5_launches.csv python tools/matvec_one.py c5 1 > /dev/null 2>&1
cat gpurun_out/mv5.log
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/mv5_launches.csv")))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
for r in rows[hi+1:]:
    print(r[h.index("Kernel Name")][:30], r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
python tools/matvec_one.py c3 3; python tools/matvec_one.py c4 3
