timeout 900 python -m pytest tests/test_degrade.py tests/test_cpp_mirror.py tests/test_volio.py -x -q > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
