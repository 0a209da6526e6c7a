mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_fp32.py tests/test_full_configs.py -q -x -k "tikhonov or golden or env_variants or config" > gpurun_out/t_march.log 2>&1; echo rc=$? >> gpurun_out/t_march.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-config4 --no-cpu --no-sharded --no-fft-path --no-tv > gpurun_out/bench_march.json 2> gpurun_out/bench.err
