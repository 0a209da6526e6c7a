SECONDS=0; timeout 900 python bench.py --no-cpu > gpurun_out/b5.json 2> gpurun_out/b5.err
python -c "
import json;d=json.loads(open('gpurun_out/b5.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['tv']['ms_per_iter']); print(d.get('config4'))" > gpurun_out/b5.txt
echo "elapsed $SECONDS s" >> gpurun_out/b5.txt
