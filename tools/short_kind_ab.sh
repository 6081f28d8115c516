# A/B of the short-filter kernels: SC_SHORT_KIND=1 (tap-stationary, taps in
# registers) vs 0 (register window <= 32 taps, smem kernel above)
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/short_kind_ab.txt; : > $out
line() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['ms_per_step'],4), r['bound'], round(r['frac'],3), d['kernel'])"; }
for rep in 1 2; do
  for c in ${CFGS:-short8 short16 short32 short64}; do
    for k in ${KINDS:-0 1}; do
      SC_SHORT_KIND=$k timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | line "$c kind=$k" >> $out
    done
  done
done
