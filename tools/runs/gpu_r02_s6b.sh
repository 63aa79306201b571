# session 6, call b: C5 launch list of the default bench command and the parity table at HEAD (r02i)
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r02i_plain.json 2> gpurun_out/r02i_plain.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02i_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r02i_ncu.log 2>&1; echo "ncu rc=$?"
wc -l gpurun_out/r02i_launches_c5.csv
python tools/parity_report.py > gpurun_out/r02i_parity_table.json 2> gpurun_out/r02i_parity.err; echo "parity rc=$?"
