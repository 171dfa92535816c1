"""run_rank (the torchrun slab path bench.py uses) end to end on GPU: 2 and 3
ranks (gloo, sharing the box's GPU, exchange staged through host memory)
must assemble exactly the single-GPU output."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
CASES = {"4d": dict(shape=(64, 32, 16, 16), kernel=(8, 8, 4, 4), n_bins=64, clip_limit=0.02,
                    adaptive=True),
         "l4d": dict(shape=(64, 32, 16, 16), kernel=(16, 8, 4, 8), n_bins=128, clip_limit=0.01,
                     adaptive=False)}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1906_11355_b200 import datasets, slabs as S
        c = CASES[name]
        x = datasets.make(name, seed=5, shape=c["shape"])
        cuts = S.slab_cuts(c["shape"][0], c["kernel"][0], world)
        a, b = cuts[rank]
        out, _, _ = S.run_rank(x[a:b].contiguous().cuda(), c["shape"], c["kernel"], c["n_bins"],
                               c["clip_limit"], c["adaptive"], rank, world)
        torch.cuda.synchronize()
        q.put((rank, a, b, out.cpu().numpy()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("name,world", [("4d", 2), ("4d", 3), ("l4d", 2)])
def test_run_rank_matches_single_gpu(name, world):
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    c = CASES[name]
    x = datasets.make(name, seed=5, shape=c["shape"])
    want = M.enhance(x.cuda(), c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"]).cpu()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    got = np.empty(c["shape"], np.float32)
    for r in res:
        assert len(r) == 4, r
        _, a, b, o = r
        got[a:b] = o
    assert np.array_equal(got, want.numpy())


def _nccl_worker(port, name, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
        from paper_1906_11355_b200 import datasets, slabs as S
        c = CASES[name]
        x = datasets.make(name, seed=5, shape=c["shape"]).cuda()
        out, _, _ = S.run_rank(x, c["shape"], c["kernel"], c["n_bins"], c["clip_limit"],
                               c["adaptive"], 0, 1)
        # the exchange object's own device all-reduce (int64 keys, MAX) over NCCL
        t = torch.tensor([3, -7, 2 ** 40], dtype=torch.int64, device="cuda")
        S.DistExchange([], 0).allreduce_max(t)
        torch.cuda.synchronize()
        q.put((out.cpu().numpy(), t.cpu().tolist(), dist.get_backend()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((repr(e),))


@pytest.mark.parametrize("name", ["4d", "l4d"])
def test_run_rank_nccl_world1(name):
    """The NCCL leg of run_rank on the box's one GPU: process group on the
    device, the range all-reduce on device tensors (no host staging), output
    identical to the plain single-GPU call.  (More than one NCCL rank needs
    more than one GPU; the 2/3-rank cases above run over gloo.)"""
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    c = CASES[name]
    x = datasets.make(name, seed=5, shape=c["shape"])
    want = M.enhance(x.cuda(), c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"]).cpu()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_port(), name, q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert len(res) == 3, res
    got, t, backend = res
    assert backend == "nccl"
    assert t == [3, -7, 2 ** 40]
    assert np.array_equal(got, want.numpy())
