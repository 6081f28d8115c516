"""Host-stream pipeline probe: raw pinned copy rates (H2D, D2H, both at once)
for the mstream input size, then mstream's host-stream e2e at several run
counts (SC_HOST_PIPE_CHUNKS).  Prints one line per measurement."""
import os
import subprocess
import sys
import time

import torch


def rate(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return dt * 1e3, nbytes / dt / 1e9


def main():
    n = 64 * 480_000
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d2 = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    print("h2d ms %.3f GB/s %.1f" % rate(lambda: d.copy_(h, non_blocking=True), 4 * n))
    print("d2h ms %.3f GB/s %.1f" % rate(lambda: h2.copy_(d2, non_blocking=True), 4 * n))
    print("both ms %.3f GB/s %.1f (aggregate)" % rate(both, 8 * n))
    for chunks in sys.argv[1:] or ["1", "2", "4", "7", "12", "16"]:
        env = dict(os.environ, SC_HOST_PIPE_CHUNKS=chunks)
        out = subprocess.run([sys.executable, "bench.py", "--config", "mstream", "--no-cpu-baseline"], env=env,
                             capture_output=True, text=True).stdout.strip().splitlines()[-1]
        import json

        e = json.loads(out)["e2e"]
        print(f"mstream chunks={chunks} e2e ms {e['ms_per_step']:.3f} value {e['value']:.1f}")


if __name__ == "__main__":
    main()
