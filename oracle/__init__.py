"""MAPLE oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the hot path computes, written from
PAPER.md (arXiv 2412.13576) with the readings of SURVEY.md §8(c)-2 (listed in DESIGN.md §3).
Floating point is fp64 (the paper fixes no precision); integer work is exact (Python ints / int64).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import it.
The product path (paper_2412_13576_b200) never imports, calls or links anything here, and this package
never imports the product path: the two share no code. The only shared module is `synth`, the seeded
instance generator, which holds none of the method's arithmetic.

Modules
  lattice      HNF (Prop. 1), GSO, LLL (Alg. 1, Siegel factor 2), reducedness (Def. P:136-144),
               pseudoinverse (Remark P:321-324), saturation check (Thm. 1)
  graver       conformal order (Def. 1), brute-force Ker_Z(A) ∩ box and Graver basis (Def. 2)
  extraction   counter RNG, start sampling, Eq. 3 loss / subgradient, Adam, Alg. 3
  postprocess  rounding, exact check (C1-C3), dedupe + sign twins, ⊑-minimal filter (C4), lex sort
  augment      objective, step bounds, Alg. 2 Graver-best augmentation, multi-start best

Parity pins: tests/test_oracle_*.py (closed forms, SPEC worked examples, brute force, invariants).
Parity unpinned: the descent trajectory itself (a chaotic heuristic; only pinned relative to IEEE fp32
arithmetic of the same algorithm, gate G2 in DESIGN.md) — see DESIGN.md §3.
"""
