"""Where the SIMT descent's time goes: device time of the descent phase of an extraction (harvest on) at
T = 1, 2, 10, 50, 200 for C3 and C5 — the T -> 0 limit is the start computation (g0, z0 = B+ g0 in fp64)."""
import sys
sys.path.insert(0, '.')
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import config  # noqa: E402

for name, N in (("C3", 65536), ("C5", 16384), ("C2a", 65536)):
    inst = config(name)
    ctx = maple.Context(inst.A, inst.l, inst.u)
    for T in (1, 2, 10, 50, 200):
        ctx.extract(N, T, inst.lr, inst.seed).free()
        ds = ctx.extract(N, T, inst.lr, inst.seed)
        print(name, N, T, "descent %.3f ms" % ctx.timings()["descent"], flush=True)
        ds.free()
    ctx.close()
