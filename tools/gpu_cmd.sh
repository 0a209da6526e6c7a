timeout 900 python -m pytest tests/test_degrade.py -x -q > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
