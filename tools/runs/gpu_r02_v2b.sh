mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x -k "not full_size and not oracle" > gpurun_out/v2b_oz.log 2>&1; echo "oz unit rc=$?"; tail -30 gpurun_out/v2b_oz.log
timeout 300 python tools/sketch_engines.py c2 1,0 2>&1 | tail -5
timeout 600 python tools/sketch_engines.py c5 1,0 2>&1 | tail -5
