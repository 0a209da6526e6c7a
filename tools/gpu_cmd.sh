timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -x -q -k "spatial or env_variants or rfft or half or config1 or config4" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
timeout 900 python bench.py --no-cpu --no-fft-path --no-tv > gpurun_out/b9.json 2> gpurun_out/b9.err
python -c "
import json;d=json.loads(open('gpurun_out/b9.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['config4']['tikhonov_ms'])" > gpurun_out/b9.txt
