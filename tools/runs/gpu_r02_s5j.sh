# session 5, call j: half-warp conflict-free fragment k order {0,10,5,15} (default) vs the first order
mkdir -p gpurun_out
for v in "" _var_kord0; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  for c in c5 c4; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1 | sed "s/^/[${v:-default}] /"; done
done
unset NGD_LIB_PATH
timeout 900 python tools/ws_stress.py plain 150 2>&1 | tail -2 | cut -c1-600
timeout 1500 python -m pytest tests/test_gpu_phase_b.py tests/test_gpu_properties.py tests/test_gpu_parity.py -x -q > gpurun_out/s5j_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5j_tests.log
python tools/matvec_one.py c5 1 > gpurun_out/s5j_mv_plain.log 2>&1; cat gpurun_out/s5j_mv_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"phag_kernel|phbg_kernel" -c 2 -o gpurun_out/s5j_phabg_c5 \
    python tools/matvec_one.py c5 1 > gpurun_out/s5j_ncu.log 2>&1 || echo "ncu rc=$?"
ncu -i gpurun_out/s5j_phabg_c5.ncu-rep --page raw --csv > gpurun_out/s5j_phabg_c5_raw.csv 2>/dev/null
