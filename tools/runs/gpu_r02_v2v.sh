mkdir -p gpurun_out
python tools/sketch_engines.py c5 1 > gpurun_out/v2v_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"oz_" -c 12 -o gpurun_out/v2v_sketch python tools/sketch_engines.py c5 1 > gpurun_out/v2v_ncu.log 2>&1; echo "ncu rc=$?"
