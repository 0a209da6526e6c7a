#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines, ncu launch list, ncu --set full captures.
# usage: tools/collect_profiles.sh <tag>   -> gpurun_out/<tag>_*  (kept under gpurun's 64 MiB return limit:
# the --set full captures carry no source; add --import-source on for a stall-by-line session)
tag=${1:-rXX}; o=gpurun_out; mkdir -p $o
python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $o/${tag}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 --no-sharded > $o/${tag}_launches.log 2>&1
ncu --set full --clock-control none -k regex:"spatial_march|rows_kernel|lr_sandwich|fft_pass_kernel<128" -c 12 \
    -o $o/${tag}_tik -f python tools/prof_step.py tiklat 3 > $o/${tag}_ncu_tik.log 2>&1
ncu --set full --clock-control none -k regex:"rpair|tv_stencil_fast|fft_pass|tv_sandwich|tv_finalize" -s 14 -c 7 \
    -o $o/${tag}_tv -f python tools/prof_step.py tv 5 > $o/${tag}_ncu_tv.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rpair|tv_stencil_fast|fft_pass|fft_wide|tv_sandwich|tv_finalize" --csv --log-file $o/${tag}_cfg4_launches.csv \
    python tools/prof_cfg4.py 2 > $o/${tag}_cfg4.log 2>&1
ls -la $o | grep $tag
