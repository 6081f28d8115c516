# fused-split multi-stage kernel: step times at medium filters + CTA 0's unit timeline
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/fs_probe2.txt; : > $out
for cfg in short512 short768 short1024 short1536 short2048 short4096 short8192; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), r.get('kernel','')[:24])" >> $out
done
for c in short512 short1024; do echo $c >> $out; SC_FS_TRACE=1 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "fs\] unit" | head -12 | tail -6 >> $out; done
cat $out
