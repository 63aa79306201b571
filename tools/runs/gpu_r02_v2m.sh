for v in ONE_PLANE NO_STORE; do echo $v; NGD_LIB_PATH=/root/repo/_variants/v_$v.so timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1; done
timeout 300 python tools/sketch_engines.py c3 1 2>&1 | tail -1
