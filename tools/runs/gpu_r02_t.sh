for c in c5 c4 c3 c2; do python tools/matvec_one.py $c 3; done
timeout 600 python -m pytest tests/test_gpu_phase_b.py tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
