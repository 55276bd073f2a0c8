"""One C5 extraction (SIMT descent) for ncu captures: python tools/c5_one.py N T"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_13576_b200 import maple
    from synth import c5
    N, T = (int(x) for x in sys.argv[1:3])
    inst = c5()
    maple.load()
    ctx = maple.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(N, T, inst.lr, inst.seed)
    torch.cuda.synchronize()
    print(ctx.descent_kernel, N, T, "descent ms", ctx.timings()["descent"], "rows", ds.size)


if __name__ == "__main__":
    main()
