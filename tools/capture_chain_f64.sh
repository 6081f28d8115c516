# ncu capture of the float64 ordered chain on a large launch: 10 s of noise
# through an 8.8 M-tap IR (the real-time-limit sweep's cell).
cd /root/repo; mkdir -p gpurun_out/prof
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_chain_w -s 1 -c 1 \
  -f -o gpurun_out/prof/full_f64_rt_k_chain_w python -m paper_2401_01607_b200 bench --ir-sweep 200000:200000:1 \
  --input noise:10 --reps 1 > gpurun_out/ncu_f64.log 2>&1
