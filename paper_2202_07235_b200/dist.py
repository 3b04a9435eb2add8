"""Multi-GPU plumbing: one process per GPU of one box, NCCL over NVLink/NVSwitch via torch.distributed.
The pairs (image, template) are split over a GI x GT grid of ranks (rank = rt * GI + ri): rank
(ri, rt) aligns image shard ri against template shard rt (GT = world, GI = 1 is the plain template
sharding of north_star; grid_shape picks GI to balance the per-rank compress rows).  Data path per
step:

  a0  each rank: rsvd_kernel_partials on its basis sub-shard (piece ri of template shard rt; global,
      fixed rsvd_kernel_chunk() = 8-template chunks) -> all-gather of the chunk partials (rank order == global chunk
      order) -> rsvd_kernel_reduce -> host eigen-solver.  The fixed chunking makes C and U bitwise
      identical for any world size and grid.
  a1  each rank compresses its image shard and its template shard.
  a4  each rank: rsvd_align_argmax(PER_IMAGE, t_offset = template shard start) into its image
      shard's slice of the packed winner keys [M] (zeros elsewhere) -> all-gather of the keys
      [G, M] (M * 8 bytes per rank) -> rsvd_combine_winners (max of packed keys).

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
    elif x.is_cuda:                       # gloo (tests): stage through host memory
        host = torch.empty((world,) + tuple(x.shape), dtype=x.dtype)
        dist.all_gather(list(host.unbind(0)), x.detach().cpu().contiguous(), group=group)
        out.copy_(host)
    else:
        dist.all_gather(list(out.unbind(0)), x.contiguous(), group=group)
    return out


def grid_shape(world: int, M: int, T: int):
    """(GI, GT) with GI * GT = world: the rank grid minimising the per-rank compress rows
    ceil(M / GI) + ceil(T / GT) (the part of the step that does not shrink with 1-D template
    sharding); ties go to more template shards."""
    best = None
    for gi in range(1, world + 1):
        if world % gi:
            continue
        gt = world // gi
        key = (-(-M // gi) + -(-T // gt), gi)
        if best is None or key < best[0]:
            best = (key, gi, gt)
    return best[1], best[2]


def grid_coords(rank: int, GI: int):
    """(ri, rt) of `rank` in the GI x GT grid (template-shard major: rank = rt * GI + ri)."""
    return rank % GI, rank // GI


def image_range(M: int, GI: int, ri: int, align: int = 128):
    """Contiguous image shard [m0, m1) of grid row ri (multiples of `align`, the last may be short)."""
    return shard_range(M, GI, ri, align)


def basis_range(T: int, world: int, rank: int, chunk: int, GI: int = 1):
    """Templates [b0, b1) whose kernel partials rank `rank` computes: piece ri of its template
    shard rt, chunk-aligned, so the ranks in order cover the global chunks in order."""
    ri, rt = grid_coords(rank, GI)
    a, b = shard_range(T, world // GI, rt, chunk)
    s0, s1 = shard_range(b - a, GI, ri, chunk)
    return a + s0, a + s1


def gather_chunk_partials(partials: torch.Tensor, T: int, chunk: int, group=None, GI: int = 1) -> torch.Tensor:
    """Concatenate every rank's [n_r, R, R] chunk partials in global chunk order."""
    world = dist.get_world_size(group)
    counts = []
    for r in range(world):
        t0, t1 = basis_range(T, world, r, chunk, GI)
        counts.append((t1 - t0 + chunk - 1) // chunk if t1 > t0 else 0)
    cmax = max(max(counts), 1)
    pad = torch.zeros((cmax,) + tuple(partials.shape[1:]), dtype=partials.dtype, device=partials.device)
    pad[: partials.shape[0]] = partials[:cmax]
    allp = _all_gather_equal(pad, group)
    return torch.cat([allp[r, : counts[r]] for r in range(world)], dim=0)


def gather_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's packed per-image keys [M] -> [G, M]."""
    return _all_gather_equal(keys, group)


def kernel_from_shards(tmpl_shard: torch.Tensor, T_total: int, w_dev: torch.Tensor, group=None, GI: int = 1):
    """Row a0 across ranks: the kernel C (device fp64 [R, R]), bitwise identical on every rank and for
    any world size.  tmpl_shard: this rank's basis sub-shard (basis_range)."""
    from . import api
    Q = tmpl_shard.shape[2]
    chunk = api.kernel_chunk()
    part = api.kernel_partials(tmpl_shard)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        part = gather_chunk_partials(part, T_total, chunk, group, GI)
    return api.kernel_reduce(part, T_total, Q, w_dev)


def basis_from_shards(tmpl_shard: torch.Tensor, T_total: int, w_dev: torch.Tensor, H: int, group=None, GI: int = 1):
    """Rows a0 across ranks: (U [R, H], lambda [R]) identical on every rank and for any world size."""
    from . import api
    C = kernel_from_shards(tmpl_shard, T_total, w_dev, group, GI)
    return api.eigen_basis(C.cpu().numpy(), H)


def basis_from_shards_device(tmpl_shard: torch.Tensor, T_total: int, w_dev: torch.Tensor, H: int, group=None,
                             GI: int = 1):
    """Rows a0 across ranks without a host round trip: (U [R, H], lambda [R], info) as device tensors from
    the device eigen-solver (R <= 128), identical on every rank and for any world size."""
    from . import api
    C = kernel_from_shards(tmpl_shard, T_total, w_dev, group, GI)
    return api.eigen_basis_device(C, H)


def combine_keys(keys: torch.Tensor, Q: int, group=None):
    """Per-image winners over all ranks: (keys, val, t, k) on every rank."""
    from . import api
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        return api.combine_winners(gather_keys(keys, group), Q)
    return api.combine_winners(keys.view(1, -1), Q)


def align_from_host(h_images: torch.Tensor, h_tmpl_shard: torch.Tensor, T_total: int, t_offset: int, w_dev: torch.Tensor,
                    H: int, d_images: torch.Tensor, d_tmpl: torch.Tensor, img_block: int = 2048,
                    tmpl_block: int = 1024, work: torch.Tensor | None = None, group=None, *,
                    M_total: int | None = None, m_offset: int = 0, basis_sub: tuple | None = None, GI: int = 1):
    """The whole per-image path (rows a0-a4 + combine) from pinned HOST rings, with the host->device
    copies overlapped with the computation instead of preceding it:

      copy stream    template blocks, then image blocks, back to back (PCIe never idles);
      compute stream kernel partials per template block as it lands -> (all-gather) -> reduce ->
                     host eigen-solve -> compress the template shard -> for each image block as it
                     lands: compress it and align it against the whole shard (per-image keys are
                     independent, so blocks write disjoint key slices) -> (all-gather) -> combine.

    h_images [M, R, Q] / h_tmpl_shard [T_loc, R, Q]: pinned complex64 host tensors; d_images /
    d_tmpl: device buffers of the same shapes (caller-owned, reused across calls).  On a GI x GT grid
    h_images is the rank's image shard (global rows m_offset.., of M_total) and basis_sub = (b0, b1)
    the shard-relative template rows of its kernel partials (dist.basis_range).  Returns
    ((keys, val, t, k) on the device, U).  Same results as compressing/aligning everything at once."""
    from . import api
    dev = d_images.device
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    M, R, Q = h_images.shape
    T_loc = h_tmpl_shard.shape[0]
    chunk = api.kernel_chunk()
    tmpl_block = max(chunk, (tmpl_block // chunk) * chunk)
    img_block = max(128, (img_block // 128) * 128)
    copy.wait_stream(comp)                                  # device buffers are free
    t_ev, i_ev = [], []
    with torch.cuda.stream(copy):
        for b0 in range(0, T_loc, tmpl_block):
            d_tmpl[b0:b0 + tmpl_block].copy_(h_tmpl_shard[b0:b0 + tmpl_block], non_blocking=True)
            t_ev.append(torch.cuda.Event())
            t_ev[-1].record(copy)
        for b0 in range(0, M, img_block):
            d_images[b0:b0 + img_block].copy_(h_images[b0:b0 + img_block], non_blocking=True)
            i_ev.append(torch.cuda.Event())
            i_ev[-1].record(copy)
    # a0: partials per template block as it arrives (fixed global chunks), over this rank's basis rows
    bs0, bs1 = basis_sub if basis_sub is not None else (0, T_loc)
    nch = (bs1 - bs0 + chunk - 1) // chunk
    part = torch.empty((max(nch, 1), R, R), dtype=torch.float64, device=dev)
    for i, b0 in enumerate(range(0, T_loc, tmpl_block)):
        comp.wait_event(t_ev[i])
        lo, hi = max(b0, bs0), min(b0 + tmpl_block, T_loc, bs1)
        if hi > lo:
            api.kernel_partials(d_tmpl[lo:hi], out=part[(lo - bs0) // chunk:(hi - bs0 + chunk - 1) // chunk])
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        part = gather_chunk_partials(part[:nch], T_total, chunk, group, GI)
    C = api.kernel_reduce(part, T_total, Q, w_dev)
    U, lam = api.eigen_basis(C.cpu().numpy(), H)           # host solve (syncs comp; copies keep going)
    U_dev = torch.tensor(U, dtype=torch.float64, device=dev)
    # a1 templates, then a1-a4 per image block
    tb = api.compress(d_tmpl, w_dev, U_dev, api.SIDE_TEMPLATE) if T_loc else None
    keys = torch.zeros(M_total if M_total is not None else M, dtype=torch.int64, device=dev)
    if work is None:
        work = torch.empty(api.align_workspace_bytes(img_block, T_loc, Q, H) // 4, dtype=torch.float32, device=dev)
    for i, b0 in enumerate(range(0, M, img_block)):
        comp.wait_event(i_ev[i])
        nb = min(img_block, M - b0)
        ib = api.compress(d_images[b0:b0 + nb], w_dev, U_dev, api.SIDE_IMAGE)
        if T_loc:
            api.align_argmax(ib, nb, tb, T_loc, Q, H, api.PER_IMAGE, work,
                             best_key=keys[m_offset + b0:m_offset + b0 + nb], t_offset=t_offset)
    return combine_keys(keys, Q, group), U


def pack_key_reference(val: np.ndarray, t: np.ndarray, k: np.ndarray, Q: int) -> np.ndarray:
    """Host mirror of the ABI's packed-key format (include/rsvd.h), for tests of the host logic:
    (ord(float32 val) << 32) | (0xFFFFFFFF - (t*Q + k)) as uint64."""
    u = np.asarray(val, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & np.uint64(0x80000000)) != 0
    ordv = np.where(neg, (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000))
    idx = np.asarray(t, dtype=np.uint64) * np.uint64(Q) + np.asarray(k, dtype=np.uint64)
    return (ordv << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - idx)
