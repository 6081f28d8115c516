# medium filters (2^26 samples): fused-split path extended beyond 8 padded
# shifts (SC_FS_MAX_S8) vs the default dispatch; then an accuracy check of the
# extended path against the CPU oracle (spot windows)
cd /root/repo; mkdir -p gpurun_out; out=gpurun_out/fs_max.txt; : > $out
run() {  # label env... (config in $cfg)
  local label=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$label', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), r.get('kernel','')[:24])" >> $out
}
for cfg in short768 short1024 short1536 short2048 short3072 short4096 short8192; do
  run default X=1
  run fs_max72 SC_FS_MAX_S8=72
done
cat $out
SC_FS_MAX_S8=72 timeout 600 python - <<'PY' >> $out 2>&1
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2401_01607_b200 import configs
from paper_2401_01607_b200.core import Signal, scatter_convolve
for ne, nh in [(1 << 25, 1024), (1 << 25, 1100), (1 << 25, 2048), (40_000_003, 4096), (1 << 25, 8191)]:
    rng = np.random.default_rng(nh)
    x = rng.uniform(-1, 1, ne).astype(np.float32)
    h = (rng.standard_normal(nh) * np.exp(-np.arange(nh) / (nh / 5))).astype(np.float32)
    y = np.asarray(scatter_convolve(Signal(x), Signal(h), mode="tc").concatenated().samples)
    tol = configs.tolerance(x, h, "f32")
    nout = ne + nh - 1
    st = [0, nout - 4096] + [int(s) for s in np.random.default_rng(1).integers(0, nout - 4096, 6)]
    err = max(float(np.max(np.abs(y[s:s + 4096].astype(np.float64) - O.scatter_window(x, h, s, s + 4096)))) for s in st)
    print("acc", ne, nh, "err/tol", round(err / tol, 4), "finite", bool(np.isfinite(y).all()))
PY
tail -6 $out
