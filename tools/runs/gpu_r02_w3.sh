# phase A GEMM core: L2 prefetch of the D tile / next item's Zin (PF), ring depth 7
for v in libngd_b200 _var_pf0 _var_ns7 _var_ns7a4; do
  for c in c5 c4; do NGD_LIB_PATH=paper_2505_11638_b200/$v.so python tools/matvec_one.py $c 3 pha_gemm=1 | sed "s/^/$v /"; done
done
python tools/matvec_one.py c5 3 pha_gemm=0
timeout 600 python -m pytest tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -2
