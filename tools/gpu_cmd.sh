timeout 900 python -m pytest tests/test_dist.py tests/test_capi_abi.py -x -q > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
timeout 600 python bench.py --sharded --no-cpu --no-fft-path --no-config4 --no-tv --steps 10 > gpurun_out/b6.json 2> gpurun_out/b6.err
python -c "
import json;d=json.loads(open('gpurun_out/b6.json').read().strip().splitlines()[-1]);print(d['sharded'])" > gpurun_out/b6.txt
