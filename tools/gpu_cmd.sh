mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_cli.py tests/test_acceptance.py -q -s > gpurun_out/t_cli.log 2>&1; echo rc=$? >> gpurun_out/t_cli.log
