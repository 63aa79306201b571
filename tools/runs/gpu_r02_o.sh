timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "nd_1k or c4_1k or c1_loss" 2>&1 | tail -2
python tools/sketch_one.py c5; python tools/sketch_one.py c3; python tools/sketch_one.py c2
