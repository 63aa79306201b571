mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/v2g_oz.log 2>&1; echo "oz rc=$?"; tail -3 gpurun_out/v2g_oz.log
timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -2
timeout 300 python tools/sketch_engines.py c4 1 2>&1 | tail -2
timeout 600 python tools/sketch_engines.py c5 1 2>&1 | tail -2
