cd /root/repo; mkdir -p gpurun_out
python -m pytest tests/test_tc_gpu.py tests/test_engine_gpu.py tests/test_short_gpu.py -q -x > gpurun_out/s3b_tests.log 2>&1; echo rc=$? >> gpurun_out/s3b_tests.log
for c in short1024 short1536 short2048 short4096 cfg4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s3b_bench_$c.json 2>/dev/null
done
timeout 300 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3b_bench_cfg5.json 2>/dev/null
