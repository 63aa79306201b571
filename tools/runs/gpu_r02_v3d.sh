for v in j16 j24; do echo "== $v"; NGD_LIB_PATH=/root/repo/_variants/v_$v.so timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1; done
