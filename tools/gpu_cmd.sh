timeout 900 python -m pytest tests/test_dist.py tests/test_full_configs.py -x -q -k "slab or config" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
