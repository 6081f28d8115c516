# Full ncu captures of the short-filter kernels at 32 and 64 taps.
cd /root/repo; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fir_short|k_fir_tapreg" -s 3 -c 1 \
  -o gpurun_out/prof/full_short32 python bench.py --config short32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fir_short|k_fir_tapreg" -s 3 -c 1 \
  -o gpurun_out/prof/full_short64 python bench.py --config short64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof | grep short
