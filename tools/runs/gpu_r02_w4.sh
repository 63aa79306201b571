# phase A GEMM core variants: D from global memory (DG), D prefetch, ring depth 7
for v in libngd_b200 _var_dg _var_dgpf _var_ns7 _var_dgns7; do
  for c in c5 c4; do NGD_LIB_PATH=paper_2505_11638_b200/$v.so python tools/matvec_one.py $c 3 pha_gemm=1 | sed "s/^/$v /"; done
done
for v in _var_dg _var_dgns7; do NGD_LIB_PATH=paper_2505_11638_b200/$v.so timeout 600 python -m pytest tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -1; done
