timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "spatial or env_variants" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
VSR_MARCH_YX=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -x -q -k "spatial or config1 or config4" >> gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
rm -f gpurun_out/b2.log
for v in "" "VSR_MARCH_YX=1" "" "VSR_MARCH_YX=1"; do
  echo "== $v" >> gpurun_out/b2.log
  env $v timeout 300 python bench.py --no-tv --no-cpu --no-fft-path --no-config4 --steps 30 --warmup 5 2>>gpurun_out/b2.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages']['spatial_expand']['avg_us'])" >> gpurun_out/b2.log
done
