python tools/sketch_one.py c5 > gpurun_out/sk5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:formj -c 1 -o gpurun_out/r02_formj_c5 python tools/sketch_one.py c5 > gpurun_out/ncu_formj.log 2>&1
tail -2 gpurun_out/ncu_formj.log
