timeout 2400 python tools/parity_report.py > gpurun_out/r02_parity_table.json 2> gpurun_out/parity.err; echo rc=$?
tail -3 gpurun_out/parity.err
