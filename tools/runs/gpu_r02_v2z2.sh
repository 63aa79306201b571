mkdir -p gpurun_out
python tools/pha_classes.py c5 > gpurun_out/v2z_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_i8gemm2|oz_crt_dot" -c 2 -o gpurun_out/v2z_pha python tools/pha_classes.py c5 > gpurun_out/v2z_ncu.log 2>&1; echo "ncu rc=$?"
