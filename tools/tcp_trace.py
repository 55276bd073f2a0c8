"""Per-step timeline of the CTA-pair descent kernel (maple_debug_trace): one C3 extraction, then the first pair's
%globaltimer stamps printed relative to the step's first stamp.
Slots: MMA 0 wait-A, 1 A-ready, 2 fwd issued+committed, 3 S-ready, 4 bwd committed; epilogue (thread 0)
5 wait-G, 6 G-done, 7 sign done + S arrive, 8 harvest done / wait-M, 9 M-done, 10 Adam done."""
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
             "epi:M", "epi:adam", "epi:H"]
    for cta in range(2):
        for t in (5, 6, 7):
            row = tr[cta, t, :12]
            t0 = row[row > 0].min() if np.any(row > 0) else 0
            print(f"cta {cta} step {t}: " + "  ".join(f"{names[k]} {(row[k] - t0) / 1e3:6.2f}" for k in range(11) if row[k]))
        steps = tr[cta, 2:15, 6]
        print(f"cta {cta} step period (us):", np.round(np.diff(steps) / 1e3, 2))


if __name__ == "__main__":
    main()
