"""Pair structure of the ⊑ filter on a dumped pool (tools/dump_pool.py): L1 / support histograms and the
number of (g, h) pairs the key-coordinate index makes each g test, total and for the kept rows."""
import sys

import numpy as np


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pool_C2b.npz"
    z = np.load(path)
    P = z["pool"].astype(np.int64)
    K = z["kept"]
    n = P.shape[1]
    nz = P != 0
    l1 = np.abs(P).sum(1)
    supp = nz.sum(1)
    print("pool", P.shape, "kept", K.shape[0], "L1 range", l1.min(), l1.max(), "mean supp", supp.mean())
    freq = nz.sum(0)
    # key coordinate: rarest coordinate of supp(h) (ties lowest index)
    key = np.where(nz, freq[None, :], np.iinfo(np.int64).max).argmin(1)
    Lmax = int(l1.max())
    cnt = np.zeros((n, Lmax + 2), np.int64)
    np.add.at(cnt, (key, l1), 1)
    cum = np.concatenate([np.zeros((n, 1), np.int64), np.cumsum(cnt, 1)], 1)   # cum[c, L] = #h with key c, L1 < L
    pairs = (nz * cum[np.arange(n)[None, :], l1[:, None]]).sum(1)
    kept_set = {r.tobytes() for r in K}
    kept = np.array([r.astype(np.int8).tobytes() in kept_set for r in P])
    print("idx pairs total %.3e, kept rows %.3e, dominated rows %.3e" % (pairs.sum(), pairs[kept].sum(), pairs[~kept].sum()))
    print("pairs per kept row: mean %.0f max %d" % (pairs[kept].mean(), pairs[kept].max()))
    print("list length per coordinate: min %d max %d" % (cnt.sum(1).min(), cnt.sum(1).max()))
    print("L1 hist", np.bincount(l1)[:20])
    print("supp hist", np.bincount(supp)[:20])


if __name__ == "__main__":
    main()


def minimal_only(path="gpurun_out/pool_C2b.npz"):
    """The level-synchronous variant: g meets only the ⊑-minimal rows of smaller L1 filed under its support."""
    z = np.load(path)
    P = z["pool"].astype(np.int64)
    K = z["kept"]
    n = P.shape[1]
    nz = P != 0
    l1 = np.abs(P).sum(1)
    freq = nz.sum(0)
    key = np.where(nz, freq[None, :], np.iinfo(np.int64).max).argmin(1)
    kept_set = {r.tobytes() for r in K}
    kept = np.array([r.astype(np.int8).tobytes() in kept_set for r in P])
    Lmax = int(l1.max())
    cnt = np.zeros((n, Lmax + 2), np.int64)
    np.add.at(cnt, (key[kept], l1[kept]), 1)
    cum = np.concatenate([np.zeros((n, 1), np.int64), np.cumsum(cnt, 1)], 1)
    pairs = (nz * cum[np.arange(n)[None, :], l1[:, None]]).sum(1)
    print("minimal-only lists: kept-row pairs %.3e (mean %.0f), dominated-row upper bound %.3e"
          % (pairs[kept].sum(), pairs[kept].mean(), pairs[~kept].sum()))
