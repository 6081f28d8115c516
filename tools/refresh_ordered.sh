# Refresh the ordered-chain evidence: the paper's real-time-limit sweep
# (float64, bit-exact), the ordered bench lines, and the chain's launch list.
cd /root/repo
mkdir -p gpurun_out/prof
timeout 900 python -m paper_2401_01607_b200 bench --ir-sweep 3600000:4400000:400000 --input noise:10 --reps 1 \
  --csv gpurun_out/prof/realtime_limit_f64.csv > gpurun_out/prof/realtime_limit_f64.log 2>&1
for c in mstream cfg2; do
  timeout 900 python bench.py --config $c --mode ordered --no-cpu-baseline > gpurun_out/prof/bench_${c}_ordered.json 2>/dev/null
done
for c in cfg1 cfg2; do
  timeout 900 python bench.py --config $c > gpurun_out/prof/bench_$c.json 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_mstream_ordered.csv \
  python bench.py --config mstream --mode ordered --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_chain_w -s 3 -c 1 \
  -o gpurun_out/prof/full_mstream_k_chain_w python bench.py --config mstream --mode ordered --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof
