"""Multi-rank path with the real kernels (-m gpu): world sizes 2 and 4 as processes sharing cuda:0
over gloo (a functional check of dist.py's sharding, gathers and combine around the CUDA kernels --
not a scaling measurement; the ranks' kernels never wait on one another).  Each rank runs the
bench's step on its GI x GT grid cell; the combined per-image winners must equal the single-process
ones bit for bit (the basis is bitwise identical by construction, so every pair's landscape is)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG, M, T, H = "small", 512, 512, 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _step(images, tmpl, w, T_total, t0, m0, GI, world):
    from paper_2202_07235_b200 import api
    from paper_2202_07235_b200 import dist as pdist
    chunk = api.kernel_chunk()
    Mloc, R, Q = images.shape
    rank = torch.distributed.get_rank() if world > 1 else 0
    b0, b1 = pdist.basis_range(T_total, world, rank, chunk, GI)
    U, _ = pdist.basis_from_shards(tmpl[b0 - t0:b1 - t0], T_total, w, H, GI=GI)
    Ud = torch.tensor(U, device="cuda")
    keys = torch.zeros(M, dtype=torch.int64, device="cuda")
    if Mloc and tmpl.shape[0]:
        ib = api.compress(images, w, Ud, api.SIDE_IMAGE)
        tb = api.compress(tmpl, w, Ud, api.SIDE_TEMPLATE)
        work = torch.empty(api.align_workspace_bytes(Mloc, tmpl.shape[0], Q, H) // 4, dtype=torch.float32, device="cuda")
        api.align_argmax(ib, Mloc, tb, tmpl.shape[0], Q, H, api.PER_IMAGE, work, best_key=keys[m0:m0 + Mloc], t_offset=t0)
    out = pdist.combine_keys(keys, Q)
    torch.cuda.synchronize()
    return out[0].cpu().numpy(), U


def _worker(rank, world, GI, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth import make_dataset
        from paper_2202_07235_b200 import api
        from paper_2202_07235_b200 import dist as pdist
        chunk = api.kernel_chunk()
        ri, rt = pdist.grid_coords(rank, GI)
        t0, t1 = pdist.shard_range(T, world // GI, rt, chunk)
        m0, m1 = pdist.image_range(M, GI, ri)
        d = make_dataset(CFG, device="cuda", M=M, T=T, t_range=(t0, t1))
        keys, U = _step(d.images[m0:m1].contiguous(), d.templates, d.w.contiguous(), T, t0, m0, GI, world)
        q.put((rank, keys.tolist(), U.tolist()))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("world,GI", [(2, 1), (2, 2), (4, 2)])
def test_rank_grid_winners_equal_single_process(world, GI):
    from synth import make_dataset
    d = make_dataset(CFG, device="cuda", M=M, T=T)
    want, U1 = _step(d.images, d.templates, d.w.contiguous(), T, 0, 0, 1, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, GI, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, keys, U in res:
        assert np.array_equal(np.asarray(U), U1), rank           # bitwise identical basis
        assert np.array_equal(np.asarray(keys, dtype=np.int64), want), rank
