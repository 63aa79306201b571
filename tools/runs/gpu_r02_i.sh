timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_problems.py -q -x --timeout 300 -k "sketch or spectrum or c1_loss or nd_1k or c4_1k or problem" 2>&1 | tail -4
python tools/sketch_one.py c5; python tools/sketch_one.py c3; python tools/sketch_one.py c2
