for v in "" paper_2505_11638_b200/_var_jet2.so; do
  echo "== variant ${v:-default (3 stages)}"
  for c in c5 c4 c3 c2; do NGD_LIB_PATH=${v:-paper_2505_11638_b200/libngd_b200.so} python tools/matvec_one.py $c 3; done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_phase_b.py -q -x --timeout 300 2>&1 | tail -2
