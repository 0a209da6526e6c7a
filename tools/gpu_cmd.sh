mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp32.py -q -s > gpurun_out/t_fp32.log 2>&1; echo rc=$? >> gpurun_out/t_fp32.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tikhonov" > gpurun_out/t_tik.log 2>&1; echo rc=$? >> gpurun_out/t_tik.log
