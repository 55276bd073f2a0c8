"""A/B timing of the Eq. 4 feasible-start generator (maple_feasible_starts) between libmaple builds, each in its own
process: python tools/eq4_ab.py [--workload C3] [--reps 2] LIB.so [LIB.so ...]. Prints the mean wall time of one
call (1,024 starts, T = 1,000, lr 0.05: the bench's incumbent generator) and the number of feasible points."""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, workload, iters):
    sys.path.insert(0, ROOT)
    from paper_2412_13576_b200 import maple
    from synth import config
    maple.load(lib)
    inst = config(workload)
    ctx = maple.Context(inst.A, inst.l, inst.u, device=0)
    for _ in range(3):
        pts, _ = ctx.feasible_starts(inst.b, 1024, 1000, 0.05, seed=17)
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        pts, _ = ctx.feasible_starts(inst.b, 1024, 1000, 0.05, seed=17)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"ms": 1e3 * sum(ts) / len(ts), "points": int(len(pts)), "checksum": int(abs(pts).sum())}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.libs[0], a.workload, a.iters)
        return
    for r in range(a.reps):
        for lib in a.libs:
            out = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--iters",
                                  str(a.iters), lib], capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"{a.workload} rep {r} {os.path.basename(lib)}: {line}", flush=True)


if __name__ == "__main__":
    main()
