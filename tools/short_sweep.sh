# short-filter sweep (bench lines) + the short-filter parity tests
cd /root/repo; mkdir -p gpurun_out/prof; : > gpurun_out/short_sweep.txt
for c in short8 short16 short32 short64 short128; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', round(d['ms_per_step'],4), r['bound'], round(r['frac'],3), d['kernel'])" >> gpurun_out/short_sweep.txt
done
timeout 900 python -m pytest -q -m gpu tests/test_short_gpu.py 2>&1 | tail -2 >> gpurun_out/short_sweep.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fir_short|k_fir_tapreg" -s 3 -c 1 \
  -f -o gpurun_out/prof/full_short32 python bench.py --config short32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_short32.log 2>&1
