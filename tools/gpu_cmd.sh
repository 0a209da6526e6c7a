mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp32.py tests/test_acceptance.py -q -s > gpurun_out/t_fp32.log 2>&1; echo rc=$? >> gpurun_out/t_fp32.log
timeout 600 python tools/diag_fp32.py > gpurun_out/diag.log 2>&1
