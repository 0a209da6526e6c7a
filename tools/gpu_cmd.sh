SECONDS=0
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01i_gputests.log 2>&1; echo "rc=$? t=$SECONDS" >> gpurun_out/r01i_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r01i_smoke.log
timeout 900 python bench.py > gpurun_out/r01i_bench.json 2> gpurun_out/r01i_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01i_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 > gpurun_out/ncu_l.log 2>&1
