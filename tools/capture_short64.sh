cd /root/repo; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fir_short -s 3 -c 1 \
  -f -o gpurun_out/prof/full_short64 python bench.py --config short64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_short64.log 2>&1
