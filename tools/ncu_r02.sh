# r02 ncu evidence at C5 (one GPU): launch list of one bench step, full captures of the sketch GEMM
# and of phase A / phase B.  Each command runs once plain (must exit 0) before its ncu run.
set -e
mkdir -p gpurun_out
python tools/sketch_one.py c5 > gpurun_out/sk_plain.log 2>&1
cat gpurun_out/sk_plain.log
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -c 2 -o gpurun_out/r02_gemm_c5 \
    python tools/sketch_one.py c5 > gpurun_out/ncu_gemm.log 2>&1 || echo "ncu gemm rc=$?"
python tools/matvec_one.py c5 1 > gpurun_out/mv_plain.log 2>&1
cat gpurun_out/mv_plain.log
ncu --set full --clock-control none --import-source on -k regex:"pha_all|phb2" -c 2 -o gpurun_out/r02_phab_c5 \
    python tools/matvec_one.py c5 1 > gpurun_out/ncu_phab.log 2>&1 || echo "ncu phab rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/b1_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_launches_c5.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1 || echo "ncu launches rc=$?"
ls -la gpurun_out
