for v in c256 c512; do echo "== $v"; NGD_LIB_PATH=/root/repo/_variants/v_$v.so timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1; done
NGD_LIB_PATH=/root/repo/_variants/v_c512.so timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x -k "not c5" 2>&1 | tail -2
