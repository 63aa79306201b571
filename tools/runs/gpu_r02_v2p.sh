mkdir -p gpurun_out
python tools/sketch_engines.py c3 1 > gpurun_out/v2p_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_rows_kernel|oz_cols_t" -c 4 -o gpurun_out/v2p_oz python tools/sketch_engines.py c3 1 > gpurun_out/v2p_ncu.log 2>&1; echo "ncu rc=$?"
