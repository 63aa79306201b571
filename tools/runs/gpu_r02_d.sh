mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/b_c5.txt 2> gpurun_out/b_c5.err; echo rc=$?
tail -5 gpurun_out/b_c5.err
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/b_c3.txt 2> gpurun_out/b_c3.err; echo rc=$?
tail -3 gpurun_out/b_c3.err
