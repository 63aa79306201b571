mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_small_svd.py -q -x --timeout 240 -k "cholesky" 2>&1 | tail -60 > gpurun_out/t_chol.txt
cat gpurun_out/t_chol.txt
