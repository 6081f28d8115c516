# e2e of cfg3 at several pipeline chunk counts (SC_PIPE_CHUNKS)
cd /root/repo; mkdir -p gpurun_out; : > gpurun_out/pipe_chunks.txt
for rep in 1 2; do
for k in 0 2 3 4 6; do
  SC_PIPE_CHUNKS=$k timeout 300 python bench.py --config cfg3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg3 chunks=$k dev', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))" >> gpurun_out/pipe_chunks.txt
done
done
