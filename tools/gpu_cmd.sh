mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.csv 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo rc=$? >> gpurun_out/r02_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_ref.err; echo rc=$? >> gpurun_out/r02_ref.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 --no-sharded > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 --no-sharded > gpurun_out/ncu.log 2>&1
echo rc=$? >> gpurun_out/ncu.log
