# routes: GEMM-core phase A (pha_gemm) x precontracted output layer (out_pre); tests + matvec timings
timeout 900 python -m pytest tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -3
for c in c5 c4 c3; do
  for pg in 0 1; do for op in 0 1; do python tools/matvec_one.py $c 3 pha_gemm=$pg out_pre=$op; done; done
done
python tools/matvec_one.py c2 3; python tools/matvec_one.py c2 3 out_pre=1
python tools/matvec_one.py c5 1 pha_gemm=1 out_pre=1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 12 --csv python tools/matvec_one.py c5 1 pha_gemm=1 out_pre=1 > gpurun_out/w5_launch.csv 2>&1
grep -E "phag|pha_all|out_|reduce|phb" gpurun_out/w5_launch.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-150
