echo "== fakek"; NGD_LIB_PATH=/root/repo/_variants/v_fakek.so timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1
echo "== base"; timeout 300 python tools/sketch_engines.py c5 1 2>&1 | tail -1
