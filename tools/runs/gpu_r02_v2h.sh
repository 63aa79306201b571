mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x -k "not c5 and not c4" > gpurun_out/v2h_oz.log 2>&1; echo "oz rc=$?"; tail -2 gpurun_out/v2h_oz.log
python tools/sketch_engines.py c3 1 > gpurun_out/v2h_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_rows_kernel|oz_cols_t" -c 4 -o gpurun_out/v2h_oz python tools/sketch_engines.py c3 1 > gpurun_out/v2h_ncu.log 2>&1; echo "ncu rc=$?"
tail -1 gpurun_out/v2h_plain.log
