# What the driver runs at round end, in order: GPU tests, smoke, the
# reference arm, the default bench line.
cd /root/repo; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/re_tests.log 2>&1; echo "tests rc=$?" > gpurun_out/re_summary.txt
tail -2 gpurun_out/re_tests.log >> gpurun_out/re_summary.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re_summary.txt
timeout 900 python bench.py --impl reference > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo "ref rc=$?" >> gpurun_out/re_summary.txt
timeout 900 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?" >> gpurun_out/re_summary.txt
