# multi-stage fused-split kernel: epilogue / converter warp counts (A/B builds
# under paper_2401_01607_b200/_lib/ab, -DFS_NEPI_MULTI / -DFS_NCONV_MULTI)
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/fs_warps_ab.txt; : > $out
for rep in 1 2; do
for lib in default e8c4 e8c8 e4c8; do
  for cfg in short512 short768 short1024 short2048; do
    if [ $lib = default ]; then unset SC_B200_LIB; else export SC_B200_LIB=$PWD/paper_2401_01607_b200/_lib/ab/lib_$lib.so; fi
    timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', '$cfg', round(d['ms_per_step'],4), 'frac', round(r['frac'],3))" >> $out
  done
done
done
unset SC_B200_LIB
cat $out
