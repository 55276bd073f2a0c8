"""does the ⊑ filter cost augmentation quality? The paper keeps every in-box B⌈z⌋
 and calls exact minimality impractical; the north star filters. Same extraction (same
starts, same candidates), two direction sets — the ⊑-minimal set and the paper's unfiltered pool — and the same
incumbents; compare the best objective per instance. GPU box only.

Usage: python tools/unfiltered_study.py [out.json]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import c4_batch, config, feasible_points  # noqa: E402


def one(inst, n_starts, incumbents=100):
    ctx = maple.Context(inst.A, inst.l, inst.u)
    X0 = feasible_points(inst, incumbents, seed=99)
    out = {"workload": inst.name, "n": inst.n, "n_starts": n_starts}
    for filt in (True, False):
        ctx.set_params(filter_minimal=filt)
        t0 = time.perf_counter()
        ds = ctx.extract(n_starts, inst.steps, inst.lr, inst.seed)
        t1 = time.perf_counter()
        xb, fb, _, iters = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
        t2 = time.perf_counter()
        key = "filtered" if filt else "unfiltered"
        out[key] = {"directions": ds.size, "f_best": fb, "extract_s": t1 - t0, "augment_s": t2 - t1,
                    "mean_iters": float(np.mean(iters))}
        ds.free()
    ctx.close()
    return out


def c4(n_inst=1000, incumbents=256):
    base, insts = c4_batch(n_inst, incumbents)
    ctx = maple.Context(base.A, base.l, base.u)
    Qs, cs, bs, X0s = zip(*insts)
    res = {}
    for filt in (True, False):
        ctx.set_params(filter_minimal=filt)
        ds = ctx.extract(base.n_starts, base.steps, base.lr, base.seed)
        t0 = time.perf_counter()
        _, fb = ctx.augment_many(ds, Qs, cs, [0.0] * n_inst, bs, np.stack(X0s))
        res["filtered" if filt else "unfiltered"] = (ds.size, fb, time.perf_counter() - t0)
        ds.free()
    ctx.close()
    (kf, ff, tf), (ku, fu, tu) = res["filtered"], res["unfiltered"]
    return {"workload": f"C4 ({n_inst} instances x {incumbents} incumbents)",
            "filtered": {"directions": kf, "augment_s": tf}, "unfiltered": {"directions": ku, "augment_s": tu},
            "instances_unfiltered_better": int(np.sum(fu < ff)), "instances_filtered_better": int(np.sum(ff < fu)),
            "instances_equal": int(np.sum(ff == fu)), "mean_f_filtered": float(ff.mean()),
            "mean_f_unfiltered": float(fu.mean())}


def main():
    rows = [one(config("C2a"), 65536), one(config("C2b"), 65536), one(config("C3"), 16384), c4(100, 32)]
    for r in rows:
        print(json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
