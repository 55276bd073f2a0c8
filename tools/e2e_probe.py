"""Host wall-clock breakdown of one end-to-end solve through the public API (create, extract, D2H, augment,
close), repeated; used to locate host-side overhead in bench.py's e2e number. GPU box only."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import config, feasible_points  # noqa: E402


def main(name="C2a", reps=6):
    inst = config(name)
    X0 = feasible_points(inst, 100, seed=99)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    for r in range(reps):
        t = [time.perf_counter()]
        c = maple.Context(inst.A, inst.l, inst.u)
        t.append(time.perf_counter())
        c.set_stream(stream.cuda_stream)
        d = c.extract(inst.n_starts if name != "C3" else 65536, inst.steps, inst.lr, inst.seed)
        t.append(time.perf_counter())
        rows = d.rows()
        t.append(time.perf_counter())
        c.augment(d, inst.Q, inst.c, inst.c0, inst.b, X0)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        d.free()
        c.close()
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        dt = np.diff(t) * 1e3
        print(f"{name} rep {r}: create {dt[0]:.2f} extract {dt[1]:.2f} rows {dt[2]:.2f} augment {dt[3]:.2f} "
              f"close {dt[4]:.2f} ms  (rows {rows.shape[0]})", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C2a"]))
