# session 5, call i: producer-warpgroup phase A / B with the proxy fence and the half-warp conflict-free k order
mkdir -p gpurun_out
for v in "" _var_kord0; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  for c in c5 c4; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1 | sed "s/^/[${v:-default}] /"; done
done
unset NGD_LIB_PATH
timeout 900 python tools/ws_stress.py plain 400 2>&1 | tail -2 | cut -c1-600
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s5i_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s5i_gputests.log
