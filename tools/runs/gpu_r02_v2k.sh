for v in NO_STORE NO_COMPUTE; do NGD_LIB_PATH=/root/repo/_variants/v_$v.so timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1; done
timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1
