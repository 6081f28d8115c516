# Ordered-chain evidence: float64 big-launch sweep (A/B of two library builds
# when given), the ordered bench lines, and one full ncu capture of k_chain_w
# (mstream ordered).   tools/capture_chain.sh [A.so B.so]
cd /root/repo
mkdir -p gpurun_out/prof
for lib in "$@"; do
  n=$(basename $lib .so)
  SC_B200_LIB=$PWD/$lib timeout 600 python -m paper_2401_01607_b200 bench --ir-sweep 200000:400000:200000 \
    --input noise:10 --reps 1 --csv gpurun_out/prof/rt_$n.csv > gpurun_out/prof/rt_$n.log 2>&1
done
for c in mstream cfg2; do
  timeout 900 python bench.py --config $c --mode ordered --no-cpu-baseline > gpurun_out/prof/bench_${c}_ordered.json 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_mstream_ordered.csv \
  python bench.py --config mstream --mode ordered --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_chain_w -s 3 -c 1 \
  -o gpurun_out/prof/full_mstream_k_chain_w python bench.py --config mstream --mode ordered --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof
