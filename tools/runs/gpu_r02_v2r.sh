mkdir -p gpurun_out
python tools/sketch_engines.py c5 1 > gpurun_out/v2r_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"oz_i8gemm" -c 2 -o gpurun_out/v2r_gemm python tools/sketch_engines.py c5 1 > gpurun_out/v2r_ncu.log 2>&1; echo "ncu rc=$?"
