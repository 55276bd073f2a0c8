"""A/B timing of libmaple builds on one workload (same box, interleaved runs): python tools/ab_descent.py
[--workload C2a] [--reps 3] LIB.so [LIB.so ...]. Each library runs in its own process (the binding keeps one
loaded library per process); prints the mean device time of each extraction phase."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, workload, iters, n_starts=0):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2412_13576_b200 import maple
    from synth import config
    maple.load(lib)
    inst = config(workload)
    ctx = maple.Context(inst.A, inst.l, inst.u, device=0)
    N = n_starts or inst.n_starts
    for _ in range(3):
        ctx.extract(N, inst.steps, inst.lr, inst.seed)
    acc = {}
    for _ in range(iters):
        ctx.extract(N, inst.steps, inst.lr, inst.seed)
        for k, v in ctx.timings().items():
            acc.setdefault(k, []).append(v)
    print(json.dumps({k: float(np.mean(v)) for k, v in acc.items()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--workload", default="C2a")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--n-starts", type=int, default=0)
    a = ap.parse_args()
    if a.child:
        child(a.libs[0], a.workload, a.iters, a.n_starts)
        return
    for r in range(a.reps):
        for lib in a.libs:
            out = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--iters",
                                  str(a.iters), "--n-starts", str(a.n_starts), lib], capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"rep {r} {os.path.basename(lib)}: {line}", flush=True)


if __name__ == "__main__":
    main()
