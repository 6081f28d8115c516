cd /root/repo; mkdir -p gpurun_out; : > gpurun_out/r_check.txt
for rep in 1 2; do
  for c in cfg1; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c default', round(d['ms_per_step'],4))" >> gpurun_out/r_check.txt
  done
  for r in 0 4 8; do
    if [ $r = 0 ]; then unset SC_CHAIN_R; else export SC_CHAIN_R=$r; fi
    timeout 300 python bench.py --config cfg2 --mode ordered --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg2-ordered R=$r', round(d['ms_per_step'],4))" >> gpurun_out/r_check.txt
  done
  unset SC_CHAIN_R
done
timeout 600 python -m paper_2401_01607_b200 bench --ir-sweep 200000:400000:200000 --input noise:10 --reps 1 --csv gpurun_out/rt_default.csv > /dev/null 2>&1
echo "rt default $(tail -2 gpurun_out/rt_default.csv | cut -d, -f1,4 | tr '\n' ' ')" >> gpurun_out/r_check.txt
timeout 900 python -m pytest -q -m gpu tests/ 2>&1 | tail -2 >> gpurun_out/r_check.txt
