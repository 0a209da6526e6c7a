timeout 900 python -m pytest tests/test_volio.py tests/test_capi_abi.py tests/test_cpp_mirror.py -x -q > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
