timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 600 python bench.py --no-cpu --no-fft-path > gpurun_out/b3.json 2> gpurun_out/b3.err
python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['tv']['ms_per_iter'], {k:round(v['avg_us'],1) for k,v in d['tv']['stages'].items()})" > gpurun_out/b3.txt
