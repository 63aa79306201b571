timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/v2q_oz.log 2>&1; echo "oz rc=$?"; tail -4 gpurun_out/v2q_oz.log
timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1
timeout 600 python tools/sketch_engines.py c5 1 2>&1 | tail -1
