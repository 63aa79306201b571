# session 5, call t: ncu --set full of the C5 PCG iteration's vector / preconditioner / thin-layer kernels
mkdir -p gpurun_out
python tools/pcg_one.py c5 3 > gpurun_out/s5t_plain.log 2>&1; cat gpurun_out/s5t_plain.log | tail -2
timeout 2400 ncu --set full --clock-control none -k regex:"utv_kernel|uc_kernel|pcg_ad_kernel|pcg_update_kernel|pcg_dir_pack_kernel|reduce_pha_cols_kernel|out_phase_b_kernel|phb2_thin_kernel|pha_all_kernel" \
    -o gpurun_out/s5t_pcg_c5 python tools/pcg_one.py c5 3 > gpurun_out/s5t_ncu.log 2>&1 || echo "ncu rc=$?"
ncu -i gpurun_out/s5t_pcg_c5.ncu-rep --page raw --csv > gpurun_out/s5t_pcg_c5_raw.csv 2>/dev/null; wc -l gpurun_out/s5t_pcg_c5_raw.csv
