"""North-star post-processing of the harvested set (oracle), each by its plain definition.

  check     (C1)-(C3) of §4: A g = 0 exactly (int64), g != 0, l - u <= g <= u - l.
  dedupe    set semantics (Alg. 3 "𝒢 ∪ {·}") with sign twins collapsed to the canonical
            representative (first nonzero > 0; reading #13).
  minimal   (C4) / Def. 2: keep g iff no other h of the set has h ⊑ g or h ⊑ -g (Def. 1,
            P:91-94; negation closure of the ± pairs, reading #14). Plain pairwise test.
  lex_sort  rows sorted lexicographically (SPEC S:284 output order).
"""
from __future__ import annotations

import numpy as np

from .graver import canonical


def check_rows(A, l, u, G) -> np.ndarray:
    """Boolean per row: A g == 0 (exact int64), g != 0 and g in [l-u, u-l]."""
    A = np.asarray(A, dtype=np.int64)
    G = np.asarray(G, dtype=np.int64).reshape(-1, A.shape[1])
    box = np.asarray(u, np.int64) - np.asarray(l, np.int64)
    return (np.all(G @ A.T == 0, axis=1) & np.any(G != 0, axis=1)
            & np.all(np.abs(G) <= box[None, :], axis=1))


def dedupe(rows) -> set:
    """Canonical set of the given integer rows (duplicates and sign twins collapse)."""
    return {canonical(r) for r in np.asarray(rows, dtype=np.int64).tolist()}


def minimal_filter(S, return_witness: bool = False):
    """⊑-minimal subset of a canonical set S: g is kept iff no h in S, h != g, with h ⊑ g or h ⊑ -g.
    Pairwise by definition (O(|S|^2 n)). Optionally returns {removed g: some dominating h}."""
    S = sorted(S)
    if not S:
        return (set(), {}) if return_witness else set()
    M = np.array(S, dtype=np.int64)
    aM = np.abs(M)
    keep, wit = set(), {}
    for i, g in enumerate(M):
        ag = np.abs(g)
        le = np.all(aM <= ag, axis=1)
        pos = np.all(M * g >= 0, axis=1)        # h ⊑ g
        neg = np.all(M * g <= 0, axis=1)        # h ⊑ -g
        dom = le & (pos | neg)
        dom[i] = False
        if dom.any():
            wit[S[i]] = S[int(np.argmax(dom))]
        else:
            keep.add(S[i])
    return (keep, wit) if return_witness else keep


def is_antichain(S) -> bool:
    """No element of S is ⊑ another element or its negation."""
    return len(minimal_filter(S)) == len(set(S))


def lex_sort(S):
    return sorted(S)


def postprocess(A, l, u, candidates, filter_minimal: bool = True):
    """check -> dedupe -> (⊑ filter) -> lex sort on a candidate multiset (rows of g)."""
    C = np.asarray(candidates, dtype=np.int64).reshape(-1, np.asarray(A).shape[1])
    ok = check_rows(A, l, u, C)
    S = dedupe(C[ok])
    if filter_minimal:
        S = minimal_filter(S)
    return lex_sort(S), int((~ok).sum())
