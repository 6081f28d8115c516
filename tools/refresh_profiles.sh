# Re-measure the bench lines kept under profiles/ (no profiler attached).
cd /root/repo
mkdir -p gpurun_out/prof
for c in ${CONFIGS:-cfg5 cfg1 cfg2 cfg3 cfg4 mstream}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err
  echo "$c rc=$?"
done
