# medium filters (2^26 samples): step time per config under the default
# dispatch, 2-shift drains on the image path (SC_TC_WIDE_SSH=2) and the image
# path forced (SC_TC_FUSED=0)
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/medium_ssh.txt; : > $out
run() {  # label env... -- config
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$label', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), r.get('kernel','')[:40])" >> $out
}
for cfg in short384 short512 short768 short1024 short1536 short2048 short4096; do
  run default X=1
  run wide_ssh2 SC_TC_WIDE_SSH=2
  run image SC_TC_FUSED=0
done
