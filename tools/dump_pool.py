"""Dump the unfiltered exact pool of a workload (C2b by default) to gpurun_out/pool_<name>.npz for host-side
study of the ⊑ filter's pair structure (tools/filter_stats.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2412_13576_b200 import maple
    from synth import config
    name = sys.argv[1] if len(sys.argv) > 1 else "C2b"
    inst = config(name)
    maple.load()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    ctx.set_params(filter_minimal=False)
    ds = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed)
    rows = ds.rows()
    ctx.set_params(filter_minimal=True)
    ds2 = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed)
    kept = ds2.rows()
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed(f"gpurun_out/pool_{name}.npz", pool=rows.astype(np.int8), kept=kept.astype(np.int8),
                        u=inst.u, l=inst.l)
    print(name, "pool", rows.shape, "kept", kept.shape, "timings", ctx.timings())


if __name__ == "__main__":
    main()
