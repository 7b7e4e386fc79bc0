"""BP=2 on the CUDA path: two processes share cuda:0 and exchange the
branch messages over gloo (host-synchronised collectives, so no kernel
waits on another process).  The native BP=2 step must be BITWISE equal to
the native BP=1 step (src/schedules.py:12-15), for fp32 and bf16."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(s=32, r=64, c_m=64, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=2)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, precision, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_2211_00235_b200 as pkg
        cfg = pkg.EvoConfig(**KW)
        store = pkg.init_params(cfg, 32, device="cuda:0")
        res = pkg.run_bp(cfg, store, seed=32, precision=precision)
        q.put((rank, res.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_native_bp2_bitwise_equals_bp1(precision):
    import paper_2211_00235_b200 as pkg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, precision, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = pkg.EvoConfig(**KW)
    single = pkg.run_single(cfg, pkg.init_params(cfg, 32), seed=32, precision=precision).numpy()
    for rank in (0, 1):
        rep = pkg.compare_runs(single, got[rank], rtol=0.0)
        assert rep.bitwise, f"rank {rank}\n{rep}"
