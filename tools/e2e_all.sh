cd /root/repo; mkdir -p gpurun_out
for c in cfg1 cfg2 mstream short8 short128; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>gpurun_out/e2e_$c.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['value'],1), d['e2e'])"
done > gpurun_out/e2e.txt 2>&1
timeout 600 python bench.py --config mstream --mode ordered --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mstream-ordered', round(d['ms_per_step'],4), round(d['value'],1), d['e2e'])" >> gpurun_out/e2e.txt 2>&1
