timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -3
python tools/sketch_one.py c2; python tools/sketch_one.py c1; python tools/sketch_one.py c3
timeout 600 python bench.py --config c2 --no-cpu --steps 10 > gpurun_out/b_c2.txt 2> gpurun_out/b_c2.err; echo rc=$?
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/b_c3.txt 2> gpurun_out/b_c3.err; echo rc=$?
