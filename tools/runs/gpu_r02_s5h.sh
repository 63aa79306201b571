for v in _var_afence _var_adsync _var_ans4; do
  export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so
  echo "== $v"; timeout 600 python tools/ws_stress.py plain 100 2>&1 | tail -2 | cut -c1-400
  timeout 300 python tools/pha_classes.py c5 2>&1 | tail -1
done
