mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_cpp_mirror.py tests/test_cli.py -q -m gpu > gpurun_out/t_cpp.log 2>&1; echo rc=$? >> gpurun_out/t_cpp.log
