mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_cli.py -q -s -k acceptance > gpurun_out/t_acc.log 2>&1; echo rc=$? >> gpurun_out/t_acc.log
