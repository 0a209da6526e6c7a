mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fp32.py tests/test_dist.py -q -m gpu -x -k "tv or TV or stencil or slab" > gpurun_out/t1.log 2>&1; echo rc=$? >> gpurun_out/t1.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sharded --no-fft-path > gpurun_out/b1.log 2>&1; echo rc=$? >> gpurun_out/b1.log
