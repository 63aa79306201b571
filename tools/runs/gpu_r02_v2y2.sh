timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/v2y_oz.log 2>&1; echo "oz rc=$?"; tail -3 gpurun_out/v2y_oz.log
timeout 300 python tools/pha_classes.py c5 2>&1 | tail -1
timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1
