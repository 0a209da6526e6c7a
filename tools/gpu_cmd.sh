mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fp32.py -q -x > gpurun_out/t_fp32.log 2>&1; echo rc=$? >> gpurun_out/t_fp32.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-config4 --no-cpu --no-sharded --no-fft-path > gpurun_out/bench_nb4.json 2> gpurun_out/bench.err
