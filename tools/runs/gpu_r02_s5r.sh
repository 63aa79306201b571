# session 5, call r: phase B GEMM core with 16 DMMA warps (32 x 32 warp tiles, 112 registers) vs 8 (64 x 32, 232)
for v in "" _var_b16; do
  if [ -n "$v" ]; then export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/$v.so; else unset NGD_LIB_PATH; fi
  for c in c5 c4; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1 | sed "s/^/[${v:-default}] /"; done
done
export NGD_LIB_PATH=/root/repo/paper_2505_11638_b200/_var_b16.so
timeout 600 python -m pytest tests/test_gpu_phase_b.py -q -x 2>&1 | tail -1
timeout 600 python tools/ws_stress.py plain 60 2>&1 | tail -2 | cut -c1-300
