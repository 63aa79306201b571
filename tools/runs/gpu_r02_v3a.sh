for v in NOSTORE NOMATH; do echo "== $v"; NGD_LIB_PATH=/root/repo/_variants/v_$v.so timeout 300 python tools/pha_classes.py c5 2>&1 | tail -2; done
