for v in "" _var_gk0; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  echo "== ${v:-default}"; timeout 300 python tools/c2_traj_probe.py 2>&1 | tail -8 | cut -c1-700
done
export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/_var_w128.so
for o in "" pha_gemm=0; do timeout 300 python tools/pha_classes.py c3 $o 2>&1 | tail -1; done
unset NGD_LIB_PATH
timeout 300 python tools/pha_classes.py c3 2>&1 | tail -1
