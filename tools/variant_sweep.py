"""optimizer / harvest variants and λ1, λ2 sweeps (readings #24-#25; Eq. 3 P:383 with the
paper's λ1 = 0.85, λ2 = 1 at P:447). On C2a, whose Graver basis is known in closed form (225 canonical
directions: e_i - e_j inside each of the 5 groups of 10), every setting reports the ⊑-minimal set size, its
recall of the closed form, the pool size, the descent time and the best augmented objective from the bench's
100 incumbents. GPU box only.

Usage: python tools/variant_sweep.py [out.json] [n_starts]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import c2a, feasible_points  # noqa: E402


def closed_form(k=5, s=10):
    out = set()
    for r in range(k):
        for i in range(s):
            for j in range(i + 1, s):
                v = [0] * (k * s)
                v[r * s + i], v[r * s + j] = 1, -1
                out.add(tuple(v))
    return out


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/variant_sweep.json"
    n_starts = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    inst = c2a()
    X0 = feasible_points(inst, 100, seed=99)
    G = closed_form()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    settings = []
    for opt in ("adam", "gd", "signgd"):
        for fin in (False, True):
            settings.append({"optimizer": opt, "harvest_final": fin, "lambda1": 0.85, "lambda2": 1.0})
    for l1 in (0.0, 0.25, 0.5, 1.0, 2.0):
        for l2 in (0.0, 1.0, 4.0):
            settings.append({"optimizer": "adam", "harvest_final": False, "lambda1": l1, "lambda2": l2})
    rows = []
    for st in settings:
        ctx.set_params(lambda1=st["lambda1"], lambda2=st["lambda2"])
        ctx.set_descent_variant(st["optimizer"], st["harvest_final"])
        ctx.extract(n_starts, inst.steps, inst.lr, inst.seed).free()   # warm
        t0 = time.perf_counter()
        ds = ctx.extract(n_starts, inst.steps, inst.lr, inst.seed)
        wall = time.perf_counter() - t0
        tm = ctx.timings()
        S = {tuple(int(v) for v in r) for r in ds.rows().tolist()}
        _, fb, _, _ = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
        rows.append(dict(st, minimal=len(S), recall=len(S & G) / len(G), non_graver=len(S - G),
                         pool=int(ds.pool_size() if callable(ds.pool_size) else ds.pool_size), descent_ms=tm["descent"], extract_ms=tm["extract_total"],
                         extract_wall_ms=wall * 1e3, f_best=fb))
        print(json.dumps(rows[-1]), flush=True)
        ds.free()
    ctx.close()
    with open(out_path, "w") as f:
        json.dump({"workload": "C2a", "n_starts": n_starts, "steps": inst.steps, "lr": inst.lr, "seed": inst.seed,
                   "closed_form_size": len(G), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
