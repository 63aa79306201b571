mkdir -p gpurun_out
timeout 120 ./tools/probe/i8gemm > gpurun_out/z_i8.log 2>&1; echo "i8 rc=$?"; cat gpurun_out/z_i8.log
timeout 600 python -m pytest tests/test_gpu_comm.py -q -x 2>&1 | tail -3
