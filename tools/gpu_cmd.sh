timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "spatial or env_variants or rfft" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
rm -f gpurun_out/b2.log
for v in "" ""; do
  env $v timeout 300 python bench.py --no-tv --no-cpu --no-fft-path --no-config4 --steps 30 --warmup 5 2>>gpurun_out/b2.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:round(v['avg_us'],1) for k,v in d['stages'].items()})" >> gpurun_out/b2.log
done
