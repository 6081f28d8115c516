# session-3 probes: kernel label test, medium-filter bench lines, a two-rank
# bench on one GPU (gloo: functional check of the spawn/shard/max-over-ranks
# path, not a scaling number), cfg3 e2e vs pipeline chunk count, raw pinned copy rates
cd /root/repo; mkdir -p gpurun_out
python -m pytest tests/test_tc_gpu.py -q -x -k "last_kernel" > gpurun_out/s3_tests.log 2>&1; echo rc=$? >> gpurun_out/s3_tests.log
for c in short256 short512 short1024; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s3_bench_$c.json 2>/dev/null; done
SC_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench_ws2_gloo_1gpu.json 2> gpurun_out/s3_bench_ws2.err
python - > gpurun_out/s3_copy_rates.txt 2>&1 <<'PY'
import torch, time
for n in (2_880_000, 2_976_000, 57_600_000):
    h = torch.empty(n, dtype=torch.float32, pin_memory=True); d = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(10): fn()
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
        print(f"{name} n={n} {dt*1e3:.3f} ms {4*n/dt/1e9:.1f} GB/s")
PY
: > gpurun_out/s3_pipe_chunks.txt
for k in 0 1 2 3 4 6 8; do
  SC_PIPE_CHUNKS=$k timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg3 chunks=$k dev', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))" >> gpurun_out/s3_pipe_chunks.txt
done
