import sys
sys.path.insert(0, '.')
from paper_2412_13576_b200 import maple
from synth import c2a
inst = c2a()
ctx = maple.Context(inst.A, inst.l, inst.u)
for _ in range(3):
    ctx.extract(inst.n_starts, 1, inst.lr, inst.seed).free()
print("ok")
