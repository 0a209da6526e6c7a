timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "spatial or env_variants" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
for v in "" "VSR_MARCH_ZC=16" "VSR_MARCH_ZC=24" "VSR_MARCH_ZC=43"; do
  echo "== $v" >> gpurun_out/b2.log
  env $v timeout 300 python bench.py --no-tv --no-cpu --no-fft-path --steps 20 --warmup 5 2>>gpurun_out/b2.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages']['spatial_expand']['avg_us'], d['roofline']['frac'])" >> gpurun_out/b2.log
done
export VSR_NO_GRAPH=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spatial_march -s 1 -c 1 -o gpurun_out/march7 python tools/prof_step.py tiklat > gpurun_out/ncu_march.log 2>&1
