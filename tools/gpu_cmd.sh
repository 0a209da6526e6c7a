timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "admm_tv" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
rm -f gpurun_out/b10.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-config4 --no-fft-path --steps 20 > gpurun_out/b9.json 2> gpurun_out/b9.err
python -c "
import json;d=json.loads(open('gpurun_out/b9.json').read().strip().splitlines()[-1]);print(d['tv']['ms_per_iter'], {k:round(v['avg_us'],1) for k,v in d['tv']['stages'].items()})" >> gpurun_out/b10.txt
done
