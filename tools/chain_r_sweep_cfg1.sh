cd /root/repo; mkdir -p gpurun_out; : > gpurun_out/r_sweep.txt
for rep in 1 2; do
for r in 0 1 2 4 8; do
  if [ $r = 0 ]; then unset SC_CHAIN_R; else export SC_CHAIN_R=$r; fi
  for tb in 32 128; do
    SC_CHAIN_TB=$tb timeout 300 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg1 R=$r tb=$tb', round(d['ms_per_step'],4))" >> gpurun_out/r_sweep.txt 2>&1
  done
done
done
