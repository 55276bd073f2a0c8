"""Timing probe of the descent kernels at C3: descent ms vs T (prologue vs per-step cost) for a kernel choice.

    python tools/tcp_probe.py [kernel=4] [n_starts=131072]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_13576_b200 import maple
    from synth import c3
    kernel = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    inst = c3()
    maple.load()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    ctx.set_descent_kernel(kernel)
    print("kernel", ctx.descent_kernel, "N", N)
    for T in (1, 2, 20, 100, 200):
        ms = []
        for rep in range(3):
            ds = ctx.extract(N, T, inst.lr, inst.seed)
            torch.cuda.synchronize()
            ms.append(ctx.timings()["descent"])
            ds.free()
        print(f"T={T:4d} descent ms {np.median(ms):9.3f}  per-step {np.median(ms) / T:8.4f}")


if __name__ == "__main__":
    main()
