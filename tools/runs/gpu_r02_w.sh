timeout 600 python -m pytest tests/test_gpu_comm.py -q -x --timeout 300 2>&1 | tail -3
python tools/sketch_one.py c5 > gpurun_out/sk5.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"dgemm|formj|gemm_reduce" -c 8 --csv --log-file gpurun_out/r02_gemm_c5_traffic.csv python tools/sketch_one.py c5 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r02_gemm_c5_traffic.csv")))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
for r in rows[hi+1:]:
    print(r[h.index("Kernel Name")][:50], r[h.index("Metric Name")], r[h.index("Metric Unit")], r[h.index("Metric Value")])
PY
