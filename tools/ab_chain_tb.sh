#!/bin/bash
# A/B of the ordered chain's CTA width (SC_CHAIN_TB=32 vs 128) on the ordered
# workloads, plus the ordered parity tests under the narrow CTA.
set -u
mkdir -p gpurun_out
out=gpurun_out/ab_chain_tb.txt
: > $out
for tb in 128 32 128 32; do
  for cfg in mstream cfg2 cfg1; do
    SC_CHAIN_TB=$tb python bench.py --config $cfg --mode ordered --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tb=$tb', '$cfg', d['ms_per_step'], d['value'])" >> $out 2>&1
  done
done
for tb in 128 32 128 32; do
  echo "c05 tb=$tb" >> $out
  SC_CHAIN_TB=$tb timeout 300 python -m pytest -x -q -m gpu tests/test_acceptance_gpu.py -k c05 2>&1 | grep -E "passed|failed|r_squared|LinearFit" | tail -3 >> $out
done
SC_CHAIN_TB=32 timeout 1200 python -m pytest -q -m gpu tests/ 2>&1 | tail -5 >> $out
