"""Multi-GPU plumbing: templates sharded over the ranks of one box (one process per GPU, NCCL over
NVLink/NVSwitch via torch.distributed).  Data path per step:

  a0  each rank: rsvd_kernel_partials on its template shard (global, fixed 32-template chunks)
      -> all-gather of the chunk partials (rank order == global chunk order) -> rsvd_kernel_reduce
      -> host eigen-solver.  The fixed chunking makes C and U bitwise identical for any G.
  a1  each rank compresses all images (replicated) and its template shard.
  a4  each rank: rsvd_align_argmax(PER_IMAGE, t_offset = shard start) -> packed winner keys [M]
      -> all-gather of the keys [G, M] (M * 8 bytes per rank) -> rsvd_combine_winners.

The collectives are the only cross-GPU traffic.  Functions here are device-agnostic (gloo/CPU
tensors work) so the host logic is testable without GPUs; the compute they wrap lives in api.py."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(T: int, world: int, rank: int, chunk: int):
    """Contiguous, chunk-aligned template shard [t0, t1) of rank `rank` (the last may be short)."""
    nch = (T + chunk - 1) // chunk
    per = (nch + world - 1) // world
    c0 = min(rank * per, nch)
    c1 = min(c0 + per, nch)
    return min(c0 * chunk, T), min(c1 * chunk, T)


def _all_gather_equal(x: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equally shaped tensors into [G, *x.shape] (NCCL: one all_gather_into_tensor)."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, x.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), x.contiguous(), group=group)
    return out


def gather_chunk_partials(partials: torch.Tensor, T: int, chunk: int, group=None) -> torch.Tensor:
    """Concatenate every rank's [n_r, R, R] chunk partials in global chunk order."""
    world = dist.get_world_size(group)
    counts = []
    for r in range(world):
        t0, t1 = shard_range(T, world, r, chunk)
        counts.append((t1 - t0 + chunk - 1) // chunk if t1 > t0 else 0)
    cmax = max(counts)
    pad = torch.zeros((cmax,) + tuple(partials.shape[1:]), dtype=partials.dtype, device=partials.device)
    pad[: partials.shape[0]] = partials
    allp = _all_gather_equal(pad, group)
    return torch.cat([allp[r, : counts[r]] for r in range(world)], dim=0)


def gather_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's packed per-image keys [M] -> [G, M]."""
    return _all_gather_equal(keys, group)


def basis_from_shards(tmpl_shard: torch.Tensor, T_total: int, w_dev: torch.Tensor, H: int, group=None):
    """Rows a0 across ranks: (U [R, H], lambda [R]) identical on every rank and for any world size."""
    from . import api
    Q = tmpl_shard.shape[2]
    chunk = api.kernel_chunk()
    part = api.kernel_partials(tmpl_shard)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        part = gather_chunk_partials(part, T_total, chunk, group)
    C = api.kernel_reduce(part, T_total, Q, w_dev)
    return api.eigen_basis(C.cpu().numpy(), H)


def combine_keys(keys: torch.Tensor, Q: int, group=None):
    """Per-image winners over all ranks: (keys, val, t, k) on every rank."""
    from . import api
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        return api.combine_winners(gather_keys(keys, group), Q)
    return api.combine_winners(keys.view(1, -1), Q)


def pack_key_reference(val: np.ndarray, t: np.ndarray, k: np.ndarray, Q: int) -> np.ndarray:
    """Host mirror of the ABI's packed-key format (include/rsvd.h), for tests of the host logic:
    (ord(float32 val) << 32) | (0xFFFFFFFF - (t*Q + k)) as uint64."""
    u = np.asarray(val, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & np.uint64(0x80000000)) != 0
    ordv = np.where(neg, (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000))
    idx = np.asarray(t, dtype=np.uint64) * np.uint64(Q) + np.asarray(k, dtype=np.uint64)
    return (ordv << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - idx)
