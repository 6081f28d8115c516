# Launch list of one cfg5 step and one full ncu capture of k_tc_fir (cfg5).
cd /root/repo
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_cfg5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_tc_fir -s 3 -c 1 \
  -o gpurun_out/prof/full_cfg5_k_tc_fir python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_fir_short -s 3 -c 1 \
  -o gpurun_out/prof/full_short8 python bench.py --config short8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof
