python tools/matvec_one.py c5 1 > gpurun_out/mv5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"phag" -c 1 -o gpurun_out/r02_phag_c5 python tools/matvec_one.py c5 1 > gpurun_out/ncu_phag.log 2>&1
tail -1 gpurun_out/ncu_phag.log
