for v in 1 2 8; do echo T$v; NGD_LIB_PATH=/root/repo/_variants/v_T$v.so timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1; done
timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1
