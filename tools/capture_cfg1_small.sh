# ncu capture of cfg1's kernel (k_chain_small, strict float64) from the bench
# command itself, plus its launch list.
cd /root/repo; mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_chain_small -s 5 -c 1 \
  -f -o gpurun_out/prof/cfg1_k_chain_small python bench.py --config cfg1 --steps 2 --warmup 5 \
  --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_cfg1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
