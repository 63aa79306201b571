set -x
free -g | head -2; nproc
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 240 2>&1 | tail -15 > gpurun_out/t_gemm.txt
cat gpurun_out/t_gemm.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -40 > gpurun_out/t_gpu.txt
cat gpurun_out/t_gpu.txt
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/b_c2.txt 2> gpurun_out/b_c2.err
tail -3 gpurun_out/b_c2.err; cat gpurun_out/b_c2.txt | head -c 3000
