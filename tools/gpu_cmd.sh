mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fp32.py -q -s > gpurun_out/t_fp32.log 2>&1; echo rc=$? >> gpurun_out/t_fp32.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "admm_tv or tv_" > gpurun_out/t_tv.log 2>&1; echo rc=$? >> gpurun_out/t_tv.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-config4 --no-cpu --no-sharded --no-fft-path > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
