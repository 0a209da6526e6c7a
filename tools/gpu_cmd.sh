timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 900 python bench.py --no-cpu > gpurun_out/b9.json 2> gpurun_out/b9.err
python -c "
import json;d=json.loads(open('gpurun_out/b9.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['tv']['ms_per_iter'], d['config4']['tikhonov_ms'], d['config4']['tv_ms_per_iter'], d['fft3_vs_cufft'])" > gpurun_out/b9.txt
