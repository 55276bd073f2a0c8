"""The multi-GPU product path (paper_2412_13576_b200/distributed.py) executed for real on the one
GPU available: sharded_extract / sharded_augment with NCCL at world size 1, and with gloo at world size 2 (two
processes, each driving the same GPU with its own context; the exchange goes through host staging, so no kernel
ever waits on another process). Both must reproduce maple_extract / maple_augment bit for bit: starts are keyed
by their global index, a locally non-minimal row is globally non-minimal, and the global pass re-runs the exact
dedupe + lexicographic sort of the union and the row-sharded ⊑ filter (keep bytes per rank, one all-gather).
The row-sharded pass itself is also checked through the C ABI with uneven shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reference(name, N, T):
    from paper_2412_13576_b200 import maple
    from synth import config
    maple.load()
    inst = config(name)
    ctx = maple.Context(inst.A, inst.l, inst.u)
    ds = ctx.extract(N, T, inst.lr, inst.seed)
    from synth import feasible_points
    X0 = feasible_points(inst, 8, seed=3)
    xb, fb, _, _ = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
    return ds.rows(), np.asarray(xb), fb, X0


@pytest.mark.parametrize("name,N,T", [("C2a", 4096, 200), ("C3", 2048, 60)])
def test_sharded_path_nccl_world1(gpu_lib, name, N, T):
    from paper_2412_13576_b200 import distributed as D
    from synth import config
    ref_rows, ref_x, ref_f, X0 = _reference(name, N, T)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        inst = config(name)
        ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)       # the library on its own non-blocking stream, as bench.py runs it
        merged, local = D.sharded_extract(ctx, N, T, inst.lr, inst.seed)
        np.testing.assert_array_equal(merged.rows(), ref_rows)
        np.testing.assert_array_equal(local.rows(), ref_rows)
        xb, fb = D.sharded_augment(ctx, merged, inst.Q, inst.c, inst.c0, inst.b, X0)
        assert xb.tolist() == ref_x.tolist() and fb == ref_f
    finally:
        dist.destroy_process_group()


def _gloo_worker(rank, world, port, name, N, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_13576_b200 import distributed as D
        from paper_2412_13576_b200 import maple
        from synth import config, feasible_points
        maple.load()
        inst = config(name)
        ctx = maple.Context(inst.A, inst.l, inst.u)
        merged, local = D.sharded_extract(ctx, N, T, inst.lr, inst.seed)
        X0 = feasible_points(inst, 8, seed=3)
        xb, fb = D.sharded_augment(ctx, merged, inst.Q, inst.c, inst.c0, inst.b, X0)
        q.put((rank, merged.rows(), local.size, xb.tolist(), fb))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,N,T", [("C2a", 4096, 200), ("C3", 2048, 60)])
def test_sharded_path_gloo_world2(gpu_lib, name, N, T):
    ref_rows, ref_x, ref_f, _ = _reference(name, N, T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, name, N, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=500) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows, local_size, xb, fb in res:
        np.testing.assert_array_equal(rows, ref_rows)          # every rank ends with the identical global set
        assert xb == ref_x.tolist() and fb == ref_f
    assert sum(r[2] for r in res) >= len(ref_rows)            # local sets cover the global one


@pytest.mark.parametrize("name,N,cuts", [("C2b", 8192, (0, 1, 3)), ("C3", 4096, (0, 2, 7))])
def test_keep_range_shards_equal_merge(gpu_lib, name, N, cuts):
    """maple_dirset_keep_range over uneven shards [b_i, b_{i+1}) of the union pool + maple_dirset_select equals
    the filtered merge bit for bit (the keep bit is pairwise against the whole pool, so shards are independent)."""
    from synth import config
    inst = config(name)
    ctx = gpu_lib.Context(inst.A, inst.l, inst.u)
    ref = ctx.extract(N, inst.steps, inst.lr, inst.seed)
    ctx.set_filter_minimal(False)
    raw = ctx.extract(N, inst.steps, inst.lr, inst.seed)          # the unfiltered (deduped, sorted) pool
    buf = torch.empty((max(raw.size, 1), raw.stride), dtype=torch.int8, device="cuda:0")
    torch.cuda.synchronize()
    raw.copy_device(buf.data_ptr())
    pool = ctx.merge_device(buf.data_ptr(), raw.size, raw.stride)   # a union as the ranks would gather it
    ctx.set_filter_minimal(True)
    assert pool.size == raw.size == ref.pool_size
    M = pool.size
    bounds = [M * c // 8 for c in cuts] + [M]
    keep = torch.zeros(M, dtype=torch.uint8, device="cuda:0")
    torch.cuda.synchronize()
    for a, b in zip(bounds[:-1], bounds[1:]):
        ctx.keep_range(pool, a, b, keep.data_ptr() + a)
    assert int(keep.sum().item()) == ref.size
    sel = ctx.select(pool, keep.data_ptr())
    np.testing.assert_array_equal(sel.rows(), ref.rows())
