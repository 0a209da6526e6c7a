timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_full_configs.py -x -q -k "tv or admm or objective or env" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
VSR_NO_GRAPH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "admm_tv" >> gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
rm -f gpurun_out/b3.txt
for v in "" ""; do
env $v timeout 600 python bench.py --no-cpu --no-fft-path --no-config4 --steps 10 > gpurun_out/b3.json 2> gpurun_out/b3.err
python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('$v', d['tv']['ms_per_iter'], d['tv']['objective_last'])" >> gpurun_out/b3.txt
done
