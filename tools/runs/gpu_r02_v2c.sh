mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x -k "not c5" > gpurun_out/v2c_oz.log 2>&1; echo "oz rc=$?"; tail -5 gpurun_out/v2c_oz.log
timeout 300 python tools/sketch_engines.py c2 1,0 2>&1 | tail -3
timeout 300 python tools/sketch_engines.py c3 1,0 2>&1 | tail -3
timeout 600 python tools/sketch_engines.py c5 1 2>&1 | tail -3
