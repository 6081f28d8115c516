# A/B of shift splits for small tensor-core launches (cfg2 FAST), + TC/engine tests
cd /root/repo; mkdir -p gpurun_out; : > gpurun_out/tc_split.txt
for rep in 1 2; do for v in 0 1; do
  SC_TC_SMALL_SPLIT=$v timeout 300 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg2 small_split=$v', round(d['ms_per_step'],4))" >> gpurun_out/tc_split.txt
done; done
timeout 900 python -m pytest -q -m gpu tests/test_tc_gpu.py tests/test_engine_fast_gpu.py tests/test_engine_host_gpu.py tests/test_multichannel_gpu.py 2>&1 | tail -2 >> gpurun_out/tc_split.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg2_launches_split.csv \
    python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
