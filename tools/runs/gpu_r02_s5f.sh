for v in "" _var_aonly _var_bonly _var_ws0; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  echo "== ${v:-default}"; timeout 300 python tools/ws_stress.py plain 12 2>&1 | tail -2
done
unset NGD_LIB_PATH
timeout 300 python tools/ws_stress.py nopdl 12 2>&1 | tail -2
