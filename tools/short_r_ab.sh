# A/B of the register-window short-filter kernel: outputs per thread (SC_SHORT_R)
# for Nh <= 32 and the register/smem cut-over (SC_SHORT_REG_MAXNH) for 33..64 taps
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/short_r_ab.txt; : > $out
line() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['ms_per_step'],4), r['bound'], round(r['frac'],3), d['kernel'])"; }
for rep in 1 2; do
  for c in short8 short16 short32; do
    for r in 8 16; do
      SC_SHORT_R=$r timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | line "$c R=$r" >> $out
    done
  done
  for m in 32 64; do
    SC_SHORT_REG_MAXNH=$m timeout 300 python bench.py --config short64 --no-cpu-baseline --no-e2e 2>/dev/null | line "short64 regmax=$m" >> $out
  done
done
