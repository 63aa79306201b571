timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x -k "phase_a or pcg_with" > gpurun_out/v2x_oz.log 2>&1; echo "oz pha rc=$?"; tail -3 gpurun_out/v2x_oz.log
timeout 300 python tools/pha_classes.py c5 2>&1 | tail -1
timeout 300 python tools/pha_classes.py c5 pha_gemm=0 2>&1 | tail -1
