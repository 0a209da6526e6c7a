#!/bin/bash
# Same-box A/B of one environment knob: tools/ab_env.sh VAR "val1 val2 ..." [bench flags]
# ("-" as a value = unset).  Two rounds, interleaved, to see the box's own noise.
var=$1; vals=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2; do for val in $vals; do
  if [ "$val" = "-" ]; then env -u $var python bench.py "$@" > gpurun_out/ab.json 2> gpurun_out/ab.err
  else env $var=$val python bench.py "$@" > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  echo "== $var=$val rep $rep"; python tools/bench_summary.py gpurun_out/ab.json | grep -E "cfg4|ms/iter|tik ms|fft_|fold|r2c|c2r"
done; done
