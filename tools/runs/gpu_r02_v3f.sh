timeout 900 python -m pytest tests/test_gpu_phase_b.py tests/test_gpu_properties.py tests/test_gpu_parity.py -q -x > gpurun_out/v3f.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/v3f.log
for c in c5 c4 c1; do timeout 300 python tools/pha_classes.py $c 2>&1 | tail -1; done
