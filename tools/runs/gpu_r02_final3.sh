mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/f3_plain.json 2> gpurun_out/f3_plain.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/f3_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/f3_ncu.log 2>&1; echo "ncu rc=$?"
wc -l gpurun_out/f3_launches_c5.csv
