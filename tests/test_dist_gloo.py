"""Multi-rank host logic on CPU (gloo, world_size 2): template sharding, the all-gather order of the
chunk partials and of the packed winner keys, and that combining per-shard winners reproduces the
single-process per-image winners (computed by the fp64 oracle).  The GPU kernels are exercised by
the -m gpu tests; here the per-shard compute is the oracle, and the keys use the ABI's documented
packing (dist.pack_key_reference)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_07235_b200.dist import (gather_chunk_partials, gather_keys, pack_key_reference,
                                        shard_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_covers_and_aligns():
    for T in [1, 8, 31, 32, 33, 1000, 8192]:
        for world in [1, 2, 3, 4, 8]:
            spans = [shard_range(T, world, r, 32) for r in range(world)]
            covered = []
            for (a, b) in spans:
                assert a <= b
                assert a % 32 == 0 or a == b == T          # empty trailing shards sit at T
                covered.extend(range(a, b))
            assert covered == list(range(T))


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ref
        from synth import make_dataset
        d = make_dataset("tiny", T=8, M=6)
        A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
        Q = d.Q
        U, _ = ref.basis(ref.kernel_C(B, w), 4)
        T = B.shape[0]
        t0, t1 = shard_range(T, world, rank, 4)          # chunk of 4 templates -> 2 shards of 4
        # per-shard per-image winners (oracle), packed with global template indices
        keys = np.zeros(A.shape[0], dtype=np.uint64)
        for m in range(A.shape[0]):
            X = ref.landscape_rank(A, B, w, U, np.full(t1 - t0, m), np.arange(t0, t1)).real
            v, tl, k = ref.per_image_winner(X)
            keys[m] = pack_key_reference(np.float32(v), t0 + tl, k, Q)
        g = gather_keys(torch.from_numpy(keys.view(np.int64)))
        comb = g.numpy().view(np.uint64).max(axis=0)
        # synthetic chunk partials: value = global chunk index, shape [n_r, 2, 2]
        Tp, chunk = 10 * world + 3, 4
        a, b = shard_range(Tp, world, rank, chunk)
        n_r = (b - a + chunk - 1) // chunk
        part = torch.arange(a // chunk, a // chunk + n_r, dtype=torch.float64)[:, None, None].repeat(1, 2, 2)
        allp = gather_chunk_partials(part, Tp, chunk)
        result_q.put((rank, comb.tolist(), allp[:, 0, 0].tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_winners_and_partials():
    from oracle import ref
    from synth import make_dataset
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = make_dataset("tiny", T=8, M=6)
    A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
    U, _ = ref.basis(ref.kernel_C(B, w), 4)
    want = []
    for m in range(A.shape[0]):
        X = ref.landscape_rank(A, B, w, U, np.full(8, m), np.arange(8)).real
        v, t, k = ref.per_image_winner(X)
        want.append(int(pack_key_reference(np.float32(v), t, k, d.Q)))
    Tp, chunk = 10 * world + 3, 4
    nch = (Tp + chunk - 1) // chunk
    for rank, comb, parts in res:
        assert [int(x) for x in comb] == want
        assert parts == list(range(nch))


def test_pack_key_reference_orders_like_float():
    vals = np.array([-3.0, -0.5, 0.0, 0.25, 7.0], dtype=np.float32)
    keys = pack_key_reference(vals, np.zeros(5, int), np.zeros(5, int), 64)
    assert np.all(np.diff(keys.astype(np.float64)) > 0)
    # equal values: smaller (t, k) wins
    k1 = pack_key_reference(np.float32(1.0), 0, 5, 64)
    k2 = pack_key_reference(np.float32(1.0), 0, 6, 64)
    k3 = pack_key_reference(np.float32(1.0), 1, 0, 64)
    assert k1 > k2 > k3


def test_grid_shape_and_ranges_cover_in_order():
    from paper_2202_07235_b200.dist import basis_range, grid_coords, grid_shape, image_range
    assert grid_shape(1, 16384, 8192) == (1, 1)
    assert grid_shape(8, 16384, 8192) == (4, 2)          # 4096 + 4096 compress rows per rank
    assert grid_shape(4, 100, 10000) == (1, 4)
    for world in [1, 2, 3, 4, 6, 8]:
        for M, T in [(16384, 8192), (1000, 33), (5, 700)]:
            GI, GT = grid_shape(world, M, T)
            assert GI * GT == world
            # basis rows: every rank in rank order covers the templates once, chunk-aligned, in order
            spans = [basis_range(T, world, r, 16, GI) for r in range(world)]
            covered = [t for a, b in spans for t in range(a, b)]
            assert covered == list(range(T))
            for r, (a, b) in enumerate(spans):
                ri, rt = grid_coords(r, GI)
                ta, tb = shard_range(T, GT, rt, 16)
                assert ta <= a <= b <= tb                  # inside the rank's own template shard
                assert a == b or a % 16 == 0
            rows = [m for ri in range(GI) for m in range(*image_range(M, GI, ri))]
            assert rows == list(range(M))


def _worker_grid(rank, world, GI, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ref
        from synth import make_dataset
        from paper_2202_07235_b200.dist import basis_range, grid_coords, image_range
        d = make_dataset("tiny", T=8, M=6)
        A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
        Q = d.Q
        U, _ = ref.basis(ref.kernel_C(B, w), 4)
        T, M = B.shape[0], A.shape[0]
        GT = world // GI
        ri, rt = grid_coords(rank, GI)
        t0, t1 = shard_range(T, GT, rt, 4)
        m0, m1 = image_range(M, GI, ri, 2)
        keys = np.zeros(M, dtype=np.uint64)                # zero outside this rank's image shard
        for m in range(m0, m1):
            X = ref.landscape_rank(A, B, w, U, np.full(t1 - t0, m), np.arange(t0, t1)).real
            v, tl, k = ref.per_image_winner(X)
            keys[m] = pack_key_reference(np.float32(v), t0 + tl, k, Q)
        comb = gather_keys(torch.from_numpy(keys.view(np.int64))).numpy().view(np.uint64).max(axis=0)
        Tp, chunk = 10 * world + 3, 4
        a, b = basis_range(Tp, world, rank, chunk, GI)
        n_r = (b - a + chunk - 1) // chunk
        part = torch.arange(a // chunk, a // chunk + n_r, dtype=torch.float64)[:, None, None].repeat(1, 2, 2)
        allp = gather_chunk_partials(part, Tp, chunk, GI=GI)
        result_q.put((rank, comb.tolist(), allp[:, 0, 0].tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world4_image_by_template_grid():
    """2 x 2 grid: per-image winners over image and template shards equal the single-process ones,
    and the chunk partials gather in global chunk order."""
    from oracle import ref
    from synth import make_dataset
    world, GI = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_grid, args=(r, world, GI, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = make_dataset("tiny", T=8, M=6)
    A, B, w = d.images.numpy(), d.templates.numpy(), d.w.numpy()
    U, _ = ref.basis(ref.kernel_C(B, w), 4)
    want = []
    for m in range(A.shape[0]):
        X = ref.landscape_rank(A, B, w, U, np.full(8, m), np.arange(8)).real
        v, t, k = ref.per_image_winner(X)
        want.append(int(pack_key_reference(np.float32(v), t, k, d.Q)))
    nch = (10 * world + 3 + 3) // 4
    for rank, comb, parts in res:
        assert [int(x) for x in comb] == want
        assert parts == list(range(nch))
