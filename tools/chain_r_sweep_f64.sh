# float64 chain: outputs-per-thread R on a large launch (10 s stream through
# 8.8 M / 17.6 M-tap IRs) -- R=4 is pick_r's choice there.
cd /root/repo; mkdir -p gpurun_out; : > gpurun_out/r_sweep_f64.txt
for r in 4 8 2; do
  SC_CHAIN_R=$r timeout 600 python -m paper_2401_01607_b200 bench --ir-sweep 200000:400000:200000 --input noise:10 \
    --reps 1 --csv gpurun_out/rt_R$r.csv > /dev/null 2>&1
  echo "R=$r $(tail -2 gpurun_out/rt_R$r.csv | cut -d, -f1,4 | tr '\n' ' ')" >> gpurun_out/r_sweep_f64.txt
done
