timeout 600 ncu --set full --import-source on --clock-control none -k regex:fold_axis3 -s 1 -c 1 -o gpurun_out/fa3b python tools/prof_sharded.py 2 > gpurun_out/ncu_fa3.log 2>&1
