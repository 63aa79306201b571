# phase A on the GEMM core (ngd_phag.cu): correctness on the wide-layer tile plans, then C5 / C4 matvec A/B
set -x
timeout 900 python -m pytest tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -5
for c in c5 c4; do
  python tools/matvec_one.py $c 3 pha_gemm=1
  python tools/matvec_one.py $c 3 pha_gemm=0
  NGD_LIB_PATH=paper_2505_11638_b200/_var_a5.so python tools/matvec_one.py $c 3 pha_gemm=1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 2>&1 | tail -3
