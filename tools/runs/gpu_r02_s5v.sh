# session 5, call v: ncu --set full at C4 (the matvec / sketch microbench config): matvec kernels and the INT8 sketch kernels
mkdir -p gpurun_out
python tools/matvec_one.py c4 1 > gpurun_out/s5v_mv_plain.log 2>&1; tail -1 gpurun_out/s5v_mv_plain.log
timeout 1200 ncu --set full --clock-control none -k regex:"phag_kernel|phbg_kernel|phb2_thin|pha_all" -c 8 -o gpurun_out/s5v_matvec_c4 \
    python tools/matvec_one.py c4 1 > gpurun_out/s5v_ncu1.log 2>&1 || echo "ncu rc=$?"
ncu -i gpurun_out/s5v_matvec_c4.ncu-rep --page raw --csv > gpurun_out/s5v_matvec_c4_raw.csv 2>/dev/null
python tools/sketch_one.py c4 > gpurun_out/s5v_sk_plain.log 2>&1; tail -1 gpurun_out/s5v_sk_plain.log
timeout 1800 ncu --set full --clock-control none -k regex:"oz_i8gemm2|oz_rows_blocked|oz_crt_kernel|formj_kernel" -c 10 -o gpurun_out/s5v_sketch_c4 \
    python tools/sketch_one.py c4 > gpurun_out/s5v_ncu2.log 2>&1 || echo "ncu rc=$?"
ncu -i gpurun_out/s5v_sketch_c4.ncu-rep --page raw --csv > gpurun_out/s5v_sketch_c4_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep; wc -l gpurun_out/s5v_*_raw.csv
