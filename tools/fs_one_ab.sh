# one-stage fused-split units (short32/short128): this build vs the build before the
# 4-accumulator ring (paper_2401_01607_b200/_lib/ab/lib_old.so)
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/fs_one_ab.txt; : > $out
for rep in 1 2 3; do
for lib in default old; do
  for cfg in short32 short128 short256; do
    if [ $lib = default ]; then unset SC_B200_LIB; else export SC_B200_LIB=$PWD/paper_2401_01607_b200/_lib/ab/lib_$lib.so; fi
    timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', '$cfg', round(d['ms_per_step'],4), 'frac', round(r['frac'],3))" >> $out
  done
done
done
unset SC_B200_LIB
sort -s -k2,2 -k1,1 $out
