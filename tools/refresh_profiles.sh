# Re-measure the bench lines kept under profiles/ (no profiler attached).
cd /root/repo
mkdir -p gpurun_out/prof
for c in ${CONFIGS:-cfg5 cfg1 cfg2 cfg3 cfg4 mstream}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err
  echo "$c rc=$?"
done
for c in ${ORDERED:-}; do
  timeout 900 python bench.py --config $c --mode ordered --no-cpu-baseline > gpurun_out/prof/bench_${c}_ordered.json 2>/dev/null
done
for c in ${SHORTS:-}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/prof/bench_$c.json 2>/dev/null
done
if [ -n "${WS2:-}" ]; then
  SC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-cpu-baseline \
    > gpurun_out/prof/bench_ws2.json 2> gpurun_out/prof/bench_ws2.err
  echo "ws2 rc=$?"
fi
for c in ${LAUNCH_LISTS:-}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
