# ncu capture of the multi-stage fused-split tensor-core kernel at short1024
# (2^26 x 1,024 taps) from the bench command, plus the step's launch list.
cd /root/repo; mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc_fir_fs -s 3 -c 1 \
  -f -o gpurun_out/prof/short1024_k_tc_fir_fs python bench.py --config short1024 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_short1024.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_short1024.csv python bench.py --config short1024 --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
