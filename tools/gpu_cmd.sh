mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dist.py tests/test_fp32.py -q -x -k "admm_tv or slab or fft or tv_" > gpurun_out/t_inv.log 2>&1; echo rc=$? >> gpurun_out/t_inv.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sharded --no-fft-path > gpurun_out/bench_inv.json 2> gpurun_out/bench.err
