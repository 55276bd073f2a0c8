"""One extraction of a workload (default C2b, configs[1]'s filter-heavy variant) after a warm-up, for launch-list
profiling. Usage: python tools/c2b_once.py [reps] [workload] [filter_algo]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2412_13576_b200 import maple
    from synth import config
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    inst = config(sys.argv[2] if len(sys.argv) > 2 else "C2b")
    maple.load()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    if len(sys.argv) > 3:
        ctx.set_filter_algorithm(int(sys.argv[3]))
    for _ in range(reps):
        ds = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed)
        print("rows", ds.size, ctx.timings())


if __name__ == "__main__":
    main()
