"""DAP host logic over gloo on CPU, world_size 4 (dp=1, bp=2, dap=2) and 2
(dap=2): the process groups of every axis (src/schedules.py:43-93), the
allgather collective (src/comm.py:241-243: shards concatenated in rank
order, recorded with the gathered size), and the DAP stage of the parameter
sync (src/schedules.py:300-316): every gradient of the rank's branch summed
over its DAP group except the replicated opm.out_b, then the BP owner
broadcast.  The sharded compute itself needs the CUDA kernels
(tests/test_gpu_dap.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class BankExec:
    """Two flat banks per block; bank values encode (rank, block, branch)."""

    def __init__(self, rank, nblk, n=10, rep=(3, 2)):
        self.rank, self.rep = rank, rep
        self.banks = {(b, br): torch.full((n,), float(100 * rank + 10 * b + (br == "pair")),
                                          dtype=torch.float64)
                      for b in range(nblk) for br in ("msa", "pair")}

    def grad_bank(self, blk, branch):
        return self.banks[(blk, branch)]

    def replicated(self, blk, branch):
        return [self.rep] if branch == "msa" else []

    def div_scalar(self, x, d):
        x /= d


def _worker(rank, world, port, lay_kw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2211_00235_b200 import distributed as D
        from paper_2211_00235_b200.schedules import ParallelLayout
        lay = ParallelLayout(**lay_kw)
        comm = D.Comm(lay)
        # allgather over the DAP group: rank-ordered concatenation
        t = torch.full((2, 3), float(rank))
        out = torch.empty(2 * lay.dap, 3)
        comm.allgather(comm.dapg, t, out, "fwd")
        gathered = out[:, 0].tolist()
        ex = BankExec(rank, 2)
        D.sync_param_grads(ex, comm, 2)
        banks = {f"{k[0]}.{k[1]}": v.tolist() for k, v in ex.banks.items()}
        recs = [(r.kind, r.group, r.elements, r.phase) for r in comm.trace]
        q.put((rank, comm.dapg, comm.pair, gathered, banks, recs))
    finally:
        dist.destroy_process_group()


def _run(world, lay_kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lay_kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {}
    for _ in range(world):
        rank, *rest = q.get(timeout=240)
        outs[rank] = rest
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return outs


def test_dap2_groups_allgather_and_param_sync():
    outs = _run(2, dict(dap=2))
    for rank in (0, 1):
        dapg, pair, gathered, banks, recs = outs[rank]
        assert dapg == (0, 1) and pair == (rank,)
        assert gathered == [0.0, 0.0, 1.0, 1.0]
        for b in range(2):
            for br, off in (("msa", 0), ("pair", 1)):
                v = banks[f"{b}.{br}"]
                want = float(10 * b + off) * 2 + 100.0        # ranks 0 + 1
                own = float(100 * rank + 10 * b + off)
                for i, x in enumerate(v):
                    replicated = br == "msa" and 3 <= i < 5
                    assert x == (own if replicated else want), (rank, b, br, i, x)
        ar = [r for r in recs if r[0] == "allreduce_sum"]
        # per block: msa bank in two pieces around out_b, pair bank whole
        assert [r[2] for r in ar] == [3, 5, 10] * 2
        assert [r for r in recs if r[0] == "allgather"] == [("allgather", (0, 1), 12, "fwd")]


def test_bp2_dap2_four_ranks():
    outs = _run(4, dict(bp=2, dap=2))
    # rank = bp_i * dap + dap_i
    assert outs[0][0] == (0, 1) and outs[2][0] == (2, 3)
    assert outs[0][1] == (0, 2) and outs[3][1] == (1, 3)
    for rank in range(4):
        dapg, pair, gathered, banks, recs = outs[rank]
        assert gathered == [float(dapg[0])] * 2 + [float(dapg[1])] * 2
        # after the DAP sums the BP owner broadcast: msa from bp 0, pair from bp 1
        msa_owner, pair_owner = (0, 1), (2, 3)
        for b in range(2):
            v = banks[f"{b}.msa"]
            assert v[0] == sum(100 * r + 10 * b for r in msa_owner)
            assert v[3] == 100 * pair[0] + 10 * b        # replicated: the owner's own value
            w = banks[f"{b}.pair"]
            assert w[0] == sum(100 * r + 10 * b + 1 for r in pair_owner)
        kinds = [(r[0], r[3]) for r in recs]
        # DAP stage only on the rank's own branch, then 2 broadcasts per block
        n_ar = 2 * (2 if rank < 2 else 1)
        assert kinds.count(("allreduce_sum", "param")) == n_ar
        assert kinds.count(("broadcast", "param")) == 4


def test_dap_axes_validation():
    from paper_2211_00235_b200 import EvoConfig
    from paper_2211_00235_b200.errors import ConfigError
    from paper_2211_00235_b200.schedules import ParallelLayout
    cfg = EvoConfig(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=1)
    ParallelLayout(dap=4).validate_model(cfg)
    with pytest.raises(ConfigError):
        ParallelLayout(dap=4).validate_model(EvoConfig(**{**cfg.__dict__, "r": 6}))
