mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x -k "not c5" > gpurun_out/v2d_oz.log 2>&1; echo "oz rc=$?"; tail -3 gpurun_out/v2d_oz.log
python tools/sketch_engines.py c3 1 > gpurun_out/v2d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:oz_ -c 8 -o gpurun_out/v2d_oz python tools/sketch_engines.py c3 1 > gpurun_out/v2d_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/v2d_ncu.log
