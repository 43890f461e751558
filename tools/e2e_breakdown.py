"""Where the e2e step's extra time goes (bench.py e2e vs value): CUDA-event
times of each piece of solve_multi on a pinned host block, C2 workload.
    python tools/e2e_breakdown.py [C2]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    from paper_1701_02324_b200 import workloads as W
    w = W.CONFIGS[name]
    run = bench.SingleRunner(w, 0)
    f = run.factorize()
    torch.cuda.synchronize()
    t = torch
    ev = lambda: t.cuda.Event(enable_timing=True)
    for rep in range(4):
        e = [ev() for _ in range(8)]
        h0 = time.perf_counter()
        e[0].record()
        b = run.Bh.to(device="cuda", non_blocking=True)
        e[1].record()
        B = b[f.tree.device_perm()]
        e[2].record()
        Bt = B.t().contiguous()
        e[3].record()
        from paper_1701_02324_b200.solver import solve_device
        X = solve_device(f, Bt)
        e[4].record()
        out = t.empty_like(X)
        out[:, f.tree.device_perm()] = X
        Xn = out.t().contiguous()
        e[5].record()
        xh = t.empty(Xn.shape, dtype=t.float64, pin_memory=True)
        e[6].record()
        xh.copy_(Xn, non_blocking=True)
        e[7].record()
        t.cuda.current_stream().synchronize()
        h1 = time.perf_counter()
        parts = [e[i].elapsed_time(e[i + 1]) for i in range(7)]
        print(f"host {1e3 * (h1 - h0):.3f} ms; h2d {parts[0]:.3f} gather {parts[1]:.3f} transpose {parts[2]:.3f} "
              f"solve {parts[3]:.3f} scatter+T {parts[4]:.3f} pin-alloc {parts[5]:.3f} d2h {parts[6]:.3f}")
    # the factorize itself: host time vs device time
    for rep in range(3):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        s, e1 = ev(), ev()
        s.record()
        f2 = run.factorize()
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        print(f"factorize: host returns {1e3 * (h1 - h0):.3f} ms, drained {1e3 * (h2 - h0):.3f} ms, "
              f"device {s.elapsed_time(e1):.3f} ms")
        del f2


if __name__ == "__main__":
    main()
