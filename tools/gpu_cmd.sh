mkdir -p gpurun_out
for e in 0 1 2 4 5 7; do VSR_PIPE_EXP=$e timeout 600 python bench.py --steps 10 --warmup 3 --no-config4 --no-cpu --no-sharded --no-fft-path > gpurun_out/bench_e$e.json 2> gpurun_out/bench_e$e.err; done
