timeout 1200 python -m pytest tests/test_full_configs.py -x -q -k "reference_binary" --durations=5 > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
