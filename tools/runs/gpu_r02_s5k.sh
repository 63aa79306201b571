# session 5, call k: sampled column-maxima pass of the INT8 sketch (oz_max_blocks 1024 vs 0 = every block); C4 phase A on the GEMM core
mkdir -p gpurun_out
for c in c5 c4; do
  timeout 900 python tools/sketch_engines.py $c 1,0 2>&1 | tail -3 | cut -c1-900
done
python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, bench
import paper_2505_11638_b200 as ngd
from paper_2505_11638_b200 import _lib
for cfg in ("c5", "c4"):
    prob, quad, theta0, _ = bench.make_problem(ngd, cfg)
    ell = bench.CONFIGS[cfg][4]
    gop = ngd.GramianOperator.from_problem(prob, theta0, quad)
    torch.manual_seed(1)
    V = torch.randn((ell, gop.dim), dtype=torch.float64, device="cuda")
    Y = {}
    for mb in (0, 1024):
        _lib.set_option("oz_max_blocks", mb)
        with _lib.option("sketch_gemm", 1):
            y = torch.empty_like(V); gop.matmat_colmajor(V, y); torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); gop.matmat_colmajor(V, y); e.record(); e.synchronize()
            Y[mb] = y.clone(); print(cfg, "oz_max_blocks", mb, f"{s.elapsed_time(e):.1f} ms")
    d = (torch.linalg.norm(Y[1024] - Y[0], dim=1) / torch.linalg.norm(Y[0], dim=1)).max().item()
    print(cfg, "sampled vs full maxima: max column deviation", d)
    del gop, V, Y
PY
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/s5k_ozaki.log 2>&1; echo "ozaki tests rc=$?"; tail -2 gpurun_out/s5k_ozaki.log
timeout 300 python tools/pha_classes.py c4 pha_gemm=1 2>&1 | tail -1
timeout 300 python tools/pha_classes.py c4 2>&1 | tail -1
