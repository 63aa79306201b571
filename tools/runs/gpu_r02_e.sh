timeout 300 python -m pytest tests/test_gpu_phase_b.py -q -x --timeout 200 2>&1 | tail -5
python tools/matvec_one.py c5 1; python tools/matvec_one.py c4 2; python tools/matvec_one.py c3 3; python tools/matvec_one.py c2 3
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8
