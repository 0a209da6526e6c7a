mkdir -p gpurun_out
python tools/prof_cfg4.py 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python tools/prof_cfg4.py 2 > gpurun_out/ncu.log 2>&1
echo rc=$? >> gpurun_out/ncu.log
