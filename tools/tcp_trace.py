"""Per-step timeline of the CTA-pair descent kernel (maple_debug_trace): one C3 extraction, then the first pair's
%globaltimer stamps printed relative to the step's first stamp.
Slots: MMA 0 wait-A, 1 A-ready, 2 fwd issued+committed, 3 S-ready, 4 bwd committed; epilogue (thread 0)
5 wait-G, 6 G-done, 7 sign done + S arrive, 8 harvest done / wait-M, 9 M-done, 10 Adam done, 11 H-done,
12 harvest test done, 13 after the partials barrier, 14 after the slot barrier."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_13576_b200 import maple
    from synth import c3
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    inst = c3()
    maple.load()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    ctx.extract(N, 20, inst.lr, inst.seed)
    ctx.debug_trace(True)
    ctx.extract(N, 20, inst.lr, inst.seed)
    torch.cuda.synchronize()
    tr = ctx.debug_trace(False).astype(np.int64)
    names = ["mma:waitA", "mma:A", "mma:fwd", "mma:S", "mma:bwd", "epi:waitG", "epi:G", "epi:sign", "epi:waitM",
             "epi:M", "epi:adam", "epi:H", "epi:htest", "epi:bar1", "epi:bar2"]
    for t in (5, 6, 7):
        base = tr[:, t, :15]
        t0 = base[base > 0].min()
        for cta in range(2):
            row = tr[cta, t, :15]
            print(f"step {t} cta {cta}: " + "  ".join(f"{names[k]} {(row[k] - t0) / 1e3:6.2f}"
                                                     for k in (0, 1, 2, 3, 4, 5, 6, 7, 11, 12, 13, 14, 8, 9, 10)
                                                     if row[k]))
    for cta in range(2):
        steps = tr[cta, 2:15, 6]
        print(f"cta {cta} step period (us):", np.round(np.diff(steps) / 1e3, 2))

if __name__ == "__main__":
    main()
