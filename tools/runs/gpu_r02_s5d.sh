# session 5, call d: which warp-specialised kernel breaks the C5 symmetry check (race hunt)
for v in "" _var_ws0 _var_aonly _var_bonly; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  echo "== ${v:-default}"; timeout 300 python tools/ws_check.py c5 4 2>&1 | tail -3
  timeout 300 python -m pytest tests/test_gpu_properties.py -q -x -k "full_size and c5" 2>&1 | tail -1
done
