# A/B two library builds on the FFMA2 CUDA-core FIR (--mode ffma): tools/ab_ffma.sh A.so B.so
cd /root/repo; out=gpurun_out/ab_ffma.txt; : > $out
for rep in 1 2; do for lib in $1 $2; do for c in cfg5 cfg4; do
  SC_B200_LIB=$PWD/$lib timeout 600 python bench.py --config $c --mode ffma --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', '$c', round(d['ms_per_step'],3), round(d['pct_fp32_fma_peak'],1), d['clocks']['sm_mhz'])" >> $out
done; done; done
