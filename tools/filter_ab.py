"""A/B of the ⊑ filter's pair enumerations (maple_set_filter_algorithm 1/2/3) at full size: filter time and
bit-identical kept sets. Usage: python tools/filter_ab.py [C2b C3 C2a ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2412_13576_b200 import maple
    from synth import config
    maple.load()
    for name in sys.argv[1:] or ["C2b", "C3", "C2a"]:
        inst = config(name)
        ctx = maple.Context(inst.A, inst.l, inst.u)
        ref = None
        for algo in (2, 3, 2, 3):
            ctx.set_filter_algorithm(algo)
            rows = ctx.extract(inst.n_starts, inst.steps, inst.lr, inst.seed).rows()
            t = ctx.timings()
            same = ref is None or np.array_equal(ref, rows)
            ref = rows if ref is None else ref
            print(f"{name} algo {algo}: filter {t['filter']:.2f} ms, rows {rows.shape[0]}, identical {same}", flush=True)


if __name__ == "__main__":
    main()
