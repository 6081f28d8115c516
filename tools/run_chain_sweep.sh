# Ordered-chain experiment: GPU tests, then cfg1/cfg2/mstream at every R.
cd /root/repo
python -m pytest tests -m gpu -x -q > gpurun_out/chain_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/chain_tests.log
: > gpurun_out/chain_bench.log
for c in ${CONFIGS:-cfg1 cfg2 mstream}; do
  for r in ${RS:-0 1 2 4 8}; do
    if [ $r = 0 ]; then unset SC_CHAIN_R; else export SC_CHAIN_R=$r; fi
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c R=$r', round(d['ms_per_step'],4), [round(v,4) for v in d['step_ms_rank0']])" >> gpurun_out/chain_bench.log 2>&1
  done
done
unset SC_CHAIN_R
