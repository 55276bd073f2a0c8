"""Small tcgen05 harvest run (256 starts, T=20): a quick hang / fault check before the full tests. GPU box only."""
import sys

sys.path.insert(0, ".")
from paper_2412_13576_b200 import maple  # noqa: E402
from synth import config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else 2
inst = config(name)
ctx = maple.Context(inst.A, inst.l, inst.u)
ctx.set_descent_kernel(kernel)
ds = ctx.extract(256, 20, inst.lr, inst.seed)
print(name, "rows", ds.size, flush=True)
