timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "admm_tv_vs_oracle" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
