free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 1200 python -m pytest tests/test_full_configs.py -x -q --durations=10 > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
