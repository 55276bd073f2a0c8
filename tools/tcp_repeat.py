"""Repeat the small-T parity check of the CTA-pair kernel (flakiness probe): prints the pass fraction per run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import extraction as OX
    from oracle import lattice as OL
    from paper_2412_13576_b200 import maple
    from synth import c3
    inst = c3()
    maple.load()
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    N, T = 300, 1
    ref = None
    for k in range(reps):
        ctx = maple.Context(inst.A, inst.l, inst.u)
        ctx.set_descent_kernel(4)
        Z, Z0 = ctx.debug_descent(N, 0, N, T, inst.lr, 11)
        if ref is None:
            _, z0 = OX.sample_starts(inst.l, inst.u, OL.pinv(ctx.B), 11, np.arange(N))
            ref = OX.descend(z0, ctx.B, T, inst.lr)
            z0ref = z0
        rel = np.abs(Z.astype(np.float64) - ref) / np.maximum(1.0, np.abs(ref))
        bad = np.flatnonzero(~np.all(rel <= 1e-4, axis=1))
        print(k, "bad starts", bad[:10].tolist(), "z0 maxerr", float(np.max(np.abs(Z0 - z0ref))),
              "maxrel", float(rel.max()))
        ctx.close()


if __name__ == "__main__":
    main()
