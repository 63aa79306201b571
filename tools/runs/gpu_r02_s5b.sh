# session 5, call b: DMMA/DFMA pipe-sharing probe; ncu full capture of the C5 matvec kernels on the GEMM core
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_mix tools/probe/fp64_mix.cu && /tmp/fp64_mix | tee gpurun_out/s5b_fp64_mix.txt
python tools/matvec_one.py c5 1 > gpurun_out/s5b_mv_plain.log 2>&1; cat gpurun_out/s5b_mv_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"phag_kernel|phbg_kernel|phb2_kernel|pha_all" -c 5 -o gpurun_out/s5b_phabg_c5 \
    python tools/matvec_one.py c5 1 > gpurun_out/s5b_ncu.log 2>&1 || echo "ncu rc=$?"
ncu -i gpurun_out/s5b_phabg_c5.ncu-rep --page raw --csv > gpurun_out/s5b_phabg_c5_raw.csv 2>/dev/null
ls -la gpurun_out | tail -8
