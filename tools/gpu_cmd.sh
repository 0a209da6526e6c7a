nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi2.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-config4 --no-fft-path --steps 20 > gpurun_out/b9.json 2> gpurun_out/b9.err
python -c "
import json;d=json.loads(open('gpurun_out/b9.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['tv']['ms_per_iter'], d['clocks'], {k:round(v['avg_us'],1) for k,v in d['tv']['stages'].items()})" >> gpurun_out/b10.txt
done
