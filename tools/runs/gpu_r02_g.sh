python tools/matvec_one.py c5 1 > gpurun_out/mv5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"phbg" -c 1 -o gpurun_out/r02_phbg_c5 python tools/matvec_one.py c5 1 > gpurun_out/ncu_phbg.log 2>&1
tail -3 gpurun_out/ncu_phbg.log
