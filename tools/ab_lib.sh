#!/bin/bash
# A/B two builds of the library (SC_B200_LIB) on the ordered workloads:
#   tools/ab_lib.sh A.so B.so [configs...]
set -u
A=$1; B=$2; shift 2
cfgs=${*:-mstream cfg2 cfg1}
mkdir -p gpurun_out
out=gpurun_out/ab_lib.txt
: > $out
for rep in 1 2; do
  for lib in $A $B; do
    for cfg in $cfgs; do
      SC_B200_LIB=$PWD/$lib python bench.py --config $cfg --mode ordered --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$cfg', d['ms_per_step'], d['value'])" >> $out 2>&1
    done
  done
done
SC_B200_LIB=$PWD/$B timeout 1200 python -m pytest -q -m gpu tests/ 2>&1 | tail -3 >> $out
