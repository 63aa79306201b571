timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_properties.py tests/test_gpu_comm.py -q -x > gpurun_out/v3e.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/v3e.log
timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1
timeout 300 python tools/sketch_engines.py c4 1 2>&1 | tail -1
