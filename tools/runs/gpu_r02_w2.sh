# ncu of the phase-A kernels at C5 (GEMM-core wide layers + thin layers) after a clean run
python tools/matvec_one.py c5 1 > gpurun_out/w2_mv.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"phag|pha_all|reduce_pha" -c 3 -o gpurun_out/r02_phag2_c5 python tools/matvec_one.py c5 1 > gpurun_out/w2_ncu.log 2>&1
tail -3 gpurun_out/w2_ncu.log
python tools/matvec_one.py c4 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"phag|pha_all" -c 2 -o gpurun_out/r02_phag2_c4 python tools/matvec_one.py c4 1 > gpurun_out/w2_ncu4.log 2>&1
tail -3 gpurun_out/w2_ncu4.log
