"""HBM bandwidth of plain streaming kernels at the stage kernel's read:write mixes.

The stage kernel moves 1 read : 1 write (first RK stage) and 2 reads : 1 write
(stages 2-4).  MEASURED_PEAKS.json's hbm_gbs is a 1:1 copy.  This measures,
with torch's own vectorised elementwise kernels on arrays far larger than L2:
  copy   c = a              1:1
  add    c = a + b          2:1
  add3   d = a + b + c      3:1 (two passes: reported per pass)
  sum    a.sum()            read only
Time with CUDA events, best of N.  Usage: python profiles/hbm_mix.py [GiB]
"""

import json
import sys

import torch


def best_ms(fn, reps=8):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
    n = int(gib * (1 << 30) / 8)
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    nb = n * 8
    out = {"array_gib": gib}
    ms = best_ms(lambda: c.copy_(a))
    out["copy_1r1w_gbs"] = 2 * nb / ms / 1e6
    ms = best_ms(lambda: torch.add(a, b, out=c))
    out["add_2r1w_gbs"] = 3 * nb / ms / 1e6
    ms = best_ms(lambda: a.sum())
    out["sum_read_only_gbs"] = nb / ms / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
