"""Multi-GPU plumbing for the hot path: one process per GPU, torch.distributed for the one
real exchange step.

Extraction shards naturally: rank r of W owns global starts [r N / W, (r+1) N / W) (the RNG is keyed by the
global start index, so the union of the shards' candidates equals the single-GPU candidate set). Each rank
extracts, checks, dedupes and ⊑-filters locally (a locally non-minimal row is globally non-minimal), then
ONE all-gather of the padded local rows (NCCL over NVLink on the GPU path) gives every rank the identical
union; its dedupe + lex sort (the pool) is replicated, and the global ⊑ pass is ROW-SHARDED: rank r decides
rows shard_range(|pool|, r, W) of the pool against the whole pool (maple_dirset_keep_range), one all-gather
of the keep bytes follows, and every rank selects the same rows (maple_dirset_select) — identical sets on
every rank, the filter work split W ways. Augmentation incumbents are sharded the same way and the per-rank
bests are all-gathered (f, x) with the lexicographic tie-break (reading #19).

The functions take the local compute as callables so that the same exchange logic runs with NCCL on the
GPU (product path: libmaple) and with gloo on CPU tensors in the tests.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced start range of `rank` (global indices)."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def gather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a (k_r, stride) int8 tensor of varying k_r across ranks: one all-gather of the counts,
    one all-gather of the rows padded to max k_r. Returns the concatenated (sum k_r, stride) rows, in rank
    order, on local.device."""
    world = dist.get_world_size(group)
    dev = local.device
    k = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    ks = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(ks, k, group=group)
    counts = ks.cpu().tolist()                     # one device-to-host read for all ranks' counts
    kmax = max(max(counts), 1)
    stride = local.shape[1]
    pad = torch.zeros((kmax, stride), dtype=local.dtype, device=dev)
    pad[: local.shape[0]] = local
    out = torch.empty((world * kmax, stride), dtype=local.dtype, device=dev)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * kmax: r * kmax + counts[r]] for r in range(world)]
    return torch.cat(parts, dim=0) if parts else out[:0]


def gather_bytes(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """All-gather 1-D uint8 tensors whose per-rank lengths `counts` every rank already knows (no count
    exchange): one all-gather of the pieces padded to max(counts). Returns the concatenation in rank order."""
    world = dist.get_world_size(group)
    kmax = max(max(counts), 1)
    pad = torch.zeros(kmax, dtype=torch.uint8, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty(world * kmax, dtype=torch.uint8, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * kmax: r * kmax + counts[r]] for r in range(world)])


def sharded_global_pass(n_pool: int, keep_range_fn, select_fn, group=None):
    """Row-sharded global ⊑ pass: rank r computes the keep bytes of pool rows
    shard_range(n_pool, r, W) with keep_range_fn(begin, end) -> uint8 tensor (end - begin,), one all-gather
    of the bytes, then select_fn(keep bytes of all n_pool rows) on every rank."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, e = shard_range(n_pool, rank, world)
    keep_local = keep_range_fn(a, e)
    counts = [shard_range(n_pool, r, world)[1] - shard_range(n_pool, r, world)[0] for r in range(world)]
    return select_fn(gather_bytes(keep_local, counts, group))


def best_across_ranks(x_best: np.ndarray, f_best: float, device, group=None):
    """All-gather every rank's (f, x) and return the global best (min f, ties lexicographically smallest x)."""
    world = dist.get_world_size(group)
    n = x_best.shape[0]
    mine = torch.tensor(np.concatenate([[f_best], x_best.astype(np.float64)]), dtype=torch.float64, device=device)
    allv = [torch.zeros(n + 1, dtype=torch.float64, device=device) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    rows = [v.cpu().numpy() for v in allv]
    best = min(rows, key=lambda r: (r[0], tuple(r[1:].tolist())))
    return best[1:].astype(np.int64), float(best[0])


def _on_host(group) -> bool:
    """gloo exchanges host tensors: the device rows are staged through host memory (CPU staging)."""
    return dist.get_backend(group) == "gloo"


def sharded_extract(ctx, n_total: int, steps: int, lr: float, seed: int, group=None, shard_filter: bool = True):
    """Product path (GPU): local maple_extract_range -> all-gather (NCCL on device buffers; gloo through host
    staging) -> global pass on the device: with shard_filter, the union's dedupe + sort on every rank and the
    row-sharded ⊑ pass (sharded_global_pass); else maple_dirset_merge (dedupe + filter + sort) on every rank.
    Returns (merged set, local set)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = shard_range(n_total, rank, world)
    local = ctx.extract_range(n_total, a, b, steps, lr, seed)
    stride = local.stride
    host = _on_host(group)
    cuda = f"cuda:{ctx.device}"
    if host:
        staged = torch.from_numpy(np.ascontiguousarray(local.rows_pinned()))          # (k, n) int8
        if staged.shape[1] < stride:
            staged = torch.nn.functional.pad(staged, (0, stride - staged.shape[1]))
        rows = gather_rows(staged, group).to(cuda)
        torch.cuda.current_stream().synchronize()
    else:
        buf = torch.empty((max(local.size, 1), stride), dtype=torch.int8, device=cuda)
        # the allocation is ordered on torch's current stream and the library copies on its own stream: drain the
        # current stream first (the copy itself is synchronous), so no earlier use of the block can land afterwards
        torch.cuda.current_stream().synchronize()
        if local.size:
            local.copy_device(buf.data_ptr())
        rows = gather_rows(buf[: local.size], group)
        torch.cuda.current_stream().synchronize()
    if rows.shape[0] == 0:
        return ctx.dirset_from_host(np.zeros((0, ctx.n), np.int32)), local
    if not shard_filter:
        return ctx.merge_device(rows.data_ptr(), rows.shape[0], stride), local
    ctx.set_filter_minimal(False)
    try:
        pool = ctx.merge_device(rows.data_ptr(), rows.shape[0], stride)   # dedupe + sort of the union
    finally:
        ctx.set_filter_minimal(True)

    def keep_range(begin, end):
        keep = torch.empty(max(end - begin, 1), dtype=torch.uint8, device=cuda)
        torch.cuda.current_stream().synchronize()
        ctx.keep_range(pool, begin, end, keep.data_ptr())
        keep = keep[: end - begin]
        return keep.cpu() if host else keep

    def select(keep_all):
        keep_all = keep_all.to(cuda)
        torch.cuda.current_stream().synchronize()
        return ctx.select(pool, keep_all.data_ptr())

    merged = sharded_global_pass(pool.size, keep_range, select, group)
    pool.free()
    return merged, local


def sharded_augment(ctx, ds, Q, c, c0, b, X0, group=None, kind=0):
    """Incumbents sharded by rank; local maple_augment; all-gather of the per-rank bests."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, e = shard_range(len(X0), rank, world)
    if e > a:
        xb, fb, _, _ = ctx.augment(ds, Q, c, c0, b, X0[a:e], kind=kind)
    else:
        xb, fb = np.zeros(ctx.n, np.int64), float("inf")
    return best_across_ranks(np.asarray(xb), fb, "cpu" if _on_host(group) else f"cuda:{ctx.device}", group)
