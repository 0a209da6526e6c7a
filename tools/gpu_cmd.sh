export VSR_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none -k regex:"fold_axis1|tv_stencil_fast|rpair_fwd|rpair_inv|fft_pass" -s 6 -c 6 -o gpurun_out/r01h_tv python tools/prof_step.py tv > gpurun_out/ncu_tv.log 2>&1
tail -2 gpurun_out/ncu_tv.log
