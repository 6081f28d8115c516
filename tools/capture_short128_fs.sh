# ncu capture of the fused-split tensor-core kernel at short128 (2^26 x 128
# taps) from the bench command, plus the step's launch list.
cd /root/repo; mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc_fir_fs -s 3 -c 1 \
  -f -o gpurun_out/prof/short128_k_tc_fir_fs python bench.py --config short128 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_short128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_short128.csv python bench.py --config short128 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
SC_FS_TRACE=1 python bench.py --config short128 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 \
  | grep "fs\] unit" | head -28 > gpurun_out/prof/short128_fs_unit_timeline.txt
