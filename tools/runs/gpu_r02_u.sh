mkdir -p gpurun_out
python tools/matvec_one.py c5 3
timeout 1500 python bench.py > gpurun_out/b_c5.txt 2> gpurun_out/b_c5.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/b_ref.txt 2> gpurun_out/b_ref.err; echo rc=$?
timeout 600 python bench.py --config c4 --no-cpu > gpurun_out/b_c4.txt 2> gpurun_out/b_c4.err; echo rc=$?
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/b_c3.txt 2> gpurun_out/b_c3.err; echo rc=$?
timeout 600 python bench.py --config c2 --no-cpu --steps 10 > gpurun_out/b_c2.txt 2> gpurun_out/b_c2.err; echo rc=$?
timeout 600 python bench.py --config c1 --no-cpu --steps 10 > gpurun_out/b_c1.txt 2> gpurun_out/b_c1.err; echo rc=$?
