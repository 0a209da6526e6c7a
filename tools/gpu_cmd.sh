export VSR_NO_GRAPH=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/cfg4_launches.csv python tools/prof_cfg4.py 2 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
