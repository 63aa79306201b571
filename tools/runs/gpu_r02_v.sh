for c in c2 c3 c1; do python tools/pcg_periter.py $c pcg_fused=0 pcg_fused=1; done
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_comm.py -q -x --timeout 300 -k "pcg or c1_nystrom or c2_factor or trajectory or comm" 2>&1 | tail -5
