"""Small tcgen05 harvest run (C1, 256 starts, T=20) for debugging under compute-sanitizer. GPU box only."""
import sys

sys.path.insert(0, ".")
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
inst = config(name)
ctx = maple.Context(inst.A, inst.l, inst.u)
ctx.set_descent_kernel(2)
ds = ctx.extract(256, 20, inst.lr, inst.seed)
print(name, "rows", ds.size, flush=True)
