mkdir -p gpurun_out
python tools/prof_step.py tiklat > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spatial_march" -s 1 -c 1 -o gpurun_out/march2 python tools/prof_step.py tiklat > gpurun_out/ncu.log 2>&1
echo rc=$? >> gpurun_out/ncu.log
