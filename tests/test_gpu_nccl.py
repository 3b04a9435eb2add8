"""The NCCL code path of dist.py on a one-GPU box (-m gpu): a world-size-1 NCCL process group runs the
exact collectives the multi-GPU bench uses (all_gather_into_tensor of fp64 chunk partials and of the
packed int64 per-image keys, on device tensors), and their results feed the library's reduce and
combine kernels.  With one rank every gather is the identity, so the outputs must equal the
non-distributed path bit for bit.  (Ranks on distinct GPUs are not available here; the gloo tests
cover world sizes 2 and 4 of the same sharding logic.)"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    import torch.distributed as tdist
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from synth import make_dataset
        from paper_2202_07235_b200 import api
        from paper_2202_07235_b200 import dist as pdist
        assert tdist.get_backend() == "nccl"
        d = make_dataset("small", device="cuda", M=256, T=200)
        w = d.w.contiguous()
        T, R, Q = d.templates.shape
        chunk = api.kernel_chunk()
        part = api.kernel_partials(d.templates)
        gathered = pdist.gather_chunk_partials(part, T, chunk)           # NCCL all_gather_into_tensor (fp64)
        lower = torch.tril(torch.ones(R, R, dtype=torch.bool, device="cuda"))
        ok_part = bool(torch.equal(gathered[:, lower], part[:, lower]))
        C_dist = pdist.kernel_from_shards(d.templates, T, w)              # world 1: no gather inside
        C_ref = api.kernel_reduce(gathered, T, Q, w)
        ok_C = bool(torch.equal(C_dist, C_ref))
        g = torch.Generator(device="cuda").manual_seed(3)
        keys = torch.randint(0, 2 ** 62, (1000,), dtype=torch.int64, device="cuda", generator=g)
        gk = pdist.gather_keys(keys)                                      # NCCL all_gather_into_tensor (int64)
        ok_keys = bool(torch.equal(gk, keys.view(1, -1)))
        a = api.combine_winners(gk, Q)
        b = pdist.combine_keys(keys, Q)
        bits = lambda x: x.view(torch.int32) if x.dtype == torch.float32 else x   # noqa: E731 (random keys decode to NaNs)
        ok_comb = all(bool(torch.equal(bits(x), bits(y))) for x, y in zip(a, b))
        torch.cuda.synchronize()
        q.put((ok_part, ok_C, ok_keys, ok_comb))
    except Exception as e:  # noqa: BLE001
        q.put(repr(e))
    finally:
        tdist.destroy_process_group()


def test_nccl_world1_collectives_match_local_path():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(0, _free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert res == (True, True, True, True), res
