"""World-size-2 gloo tests (CPU) of the multi-GPU exchange logic in paper_2412_13576_b200/distributed.py:
start sharding, the padded variable-count all-gather, the local-filter-then-global-merge soundness, the
row-sharded global ⊑ pass (keep-byte all-gather), and the cross-rank best with the lexicographic tie-break. The local compute is the oracle here (CPU); on the GPU the
same functions run with NCCL around libmaple (tests cannot stand in more GPUs than the one available)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_13576_b200 import distributed as D
        from oracle import extraction as OX, lattice as OL, postprocess as OP
        from synth import c1
        out = {}
        # 1) variable-count padded all-gather
        k = 3 if rank == 0 else 0
        local = torch.full((k, 16), rank + 1, dtype=torch.int8)
        rows = D.gather_rows(local)
        out["gather_shape"] = tuple(rows.shape)
        # 2) sharded extraction with local filter + global merge == single-process result
        inst = c1()
        B = np.array(OL.lll_reduce(OL.kernel_basis(inst.A)), dtype=np.int64)
        Bp = OL.pinv(B)
        N, T = 200, 60
        a, b = D.shard_range(N, rank, world)
        pool, _ = OX.extract_pool(B, Bp, inst.l, inst.u, N, T, 0.05, seed=4, starts=np.arange(a, b))
        loc = np.array(sorted(OP.minimal_filter(pool)), dtype=np.int8).reshape(-1, 4)
        glob = D.gather_rows(torch.from_numpy(loc))
        merged, _ = OP.postprocess(inst.A, inst.l, inst.u, glob.numpy().astype(np.int64))
        out["merged"] = merged
        full_pool, _ = OX.extract_pool(B, Bp, inst.l, inst.u, N, T, 0.05, seed=4)
        out["single"] = sorted(OP.minimal_filter(full_pool))
        out["range"] = (a, b)
        # 3) row-sharded global ⊑ pass: keep bytes of this rank's rows of the (identical) union pool, one
        # all-gather of the bytes, selection == the single-process minimal set
        U = np.array(sorted(full_pool), dtype=np.int64).reshape(-1, 4)   # the deduped, sorted union
        mins = set(OP.minimal_filter(full_pool))
        seen = {}

        def keep_fn(lo, hi):
            seen["range"] = (lo, hi)
            return torch.tensor([1 if tuple(int(v) for v in U[i]) in mins else 0 for i in range(lo, hi)],
                                dtype=torch.uint8)

        sel = D.sharded_global_pass(len(U), keep_fn, lambda kb: [tuple(int(v) for v in U[i])
                                                                  for i in range(len(U)) if kb[i]])
        out["sharded_pass"] = sorted(sel)
        out["keep_range"] = seen["range"]
        out["n_union"] = len(U)
        # 4) best across ranks, tie on f broken by lexicographically smallest x
        xb = np.array([2, 0, 1, 3]) if rank == 0 else np.array([1, 2, 0, 3])
        out["best"] = D.best_across_ranks(xb, 5.0, "cpu")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["gather_shape"] == (3, 16) and res[1]["gather_shape"] == (3, 16)
    assert res[0]["range"] == (0, 100) and res[1]["range"] == (100, 200)
    assert res[0]["merged"] == res[1]["merged"] == res[0]["single"]
    assert len(res[0]["single"]) == 6
    assert res[0]["sharded_pass"] == res[1]["sharded_pass"] == sorted(res[0]["single"])
    nu = res[0]["n_union"]
    assert res[0]["keep_range"] == (0, nu // 2) and res[1]["keep_range"] == (nu // 2, nu)
    bx, bf = res[0]["best"]
    assert bx.tolist() == [1, 2, 0, 3] and bf == 5.0
    assert res[1]["best"][0].tolist() == [1, 2, 0, 3]


def test_shard_range_partitions():
    from paper_2412_13576_b200.distributed import shard_range
    for n in (1, 7, 65536, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
