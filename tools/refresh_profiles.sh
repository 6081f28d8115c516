# Re-measure the bench lines and launch lists kept under profiles/ (bench
# lines without any profiler attached; ncu runs separately afterwards).
cd /root/repo
mkdir -p gpurun_out/prof
for c in ${CONFIGS:-cfg5 cfg1 cfg2 cfg3 cfg4 mstream}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err
  echo "$c rc=$?"
done
if [ -n "${ORDERED_MSTREAM:-}" ]; then
  timeout 900 python bench.py --config mstream --mode ordered --no-cpu-baseline > gpurun_out/prof/bench_mstream_ordered.json 2>/dev/null
fi
for c in ${LAUNCH_LISTS:-}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
for c in ${FULL_CHAIN:-}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_chain_w -s 3 -c 1 \
    -o gpurun_out/prof/full_${c}_k_chain_w python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
