VSR_SLAB_UNFUSED=1 timeout 900 python -m pytest tests/test_dist.py -x -q -k "gpu" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
for v in "" "VSR_SLAB_UNFUSED=1"; do
env $v timeout 600 python bench.py --sharded --no-cpu --no-fft-path --no-config4 --no-tv --steps 10 > gpurun_out/b6.json 2> gpurun_out/b6.err
python -c "
import json;d=json.loads(open('gpurun_out/b6.json').read().strip().splitlines()[-1]);print(d['sharded']['ms_per_iter'])" >> gpurun_out/b6.txt
done
