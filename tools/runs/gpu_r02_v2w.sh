timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x -k "phase_a or pcg_with" > gpurun_out/v2w_oz.log 2>&1; echo "oz pha rc=$?"; tail -15 gpurun_out/v2w_oz.log
for c in c5 c4; do timeout 300 python tools/matvec_one.py $c 3 2>&1 | tail -1; timeout 300 python tools/matvec_one.py $c 3 pha_gemm=0 2>&1 | tail -1; done
