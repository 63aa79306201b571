# session 5, call c: warp-specialised phase A / phase B (producer warpgroup + setmaxnreg) vs the single-role form
mkdir -p gpurun_out
for v in "" _var_ws0 _var_kord1; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  for c in c5 c4; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1 | sed "s/^/[${v:-default}] /"; done
done
unset NGD_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_phase_b.py tests/test_gpu_properties.py tests/test_gpu_parity.py -q -x > gpurun_out/s5c_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5c_tests.log
NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/_var_kord1.so timeout 600 python -m pytest tests/test_gpu_phase_b.py -q -x > gpurun_out/s5c_tests_kord1.log 2>&1; echo "kord1 tests rc=$?"; tail -1 gpurun_out/s5c_tests_kord1.log
