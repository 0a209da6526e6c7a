#!/bin/bash
# A/B of one environment knob on the same box: tools/ab_env.sh VAR "bench flags" (runs default, VAR=1, default, VAR=1)
var=$1; shift
for rep in 1 2; do for val in "" 1; do
  if [ -z "$val" ]; then env -u $var python bench.py "$@" > gpurun_out/ab.json 2> gpurun_out/ab.err; else env $var=$val python bench.py "$@" > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  echo "== $var=${val:-unset} rep $rep"; python tools/bench_summary.py gpurun_out/ab.json | grep -E "cfg4|ms/iter|tik ms"
done; done
