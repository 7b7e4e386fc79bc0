"""The reference's train-step API called from ONE process, as the reference's
tests do (tests/test_schedules.py:59-141 of the reference): run_bp / run_dp /
run_distributed launch their own world (src/schedules.py:338-361).  On a
one-GPU box every rank shares cuda:0 and the collectives run over gloo
(host-synchronised, so no kernel waits on another process); with one GPU per
rank they run over NCCL.  Properties:
  * run_bp(cfg, store) is BITWISE equal to run_single(cfg, store);
  * BP=2 x DP=2 (four ranks) equals the mean of the two BP=1 replicas;
  * the returned CommTrace matches expected_comm_volume (the reference's
    closed form; parameter collectives bucketed per branch and block);
  * rank_fwd_seconds has one forward time per rank.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

KW = dict(s=32, r=64, c_m=64, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=2)


@pytest.fixture(scope="module")
def pkg():
    import paper_2211_00235_b200 as p
    assert torch.cuda.is_available()
    return p


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_run_bp_self_launched_bitwise_equals_run_single(pkg, precision):
    cfg = pkg.EvoConfig(**KW)
    store = pkg.init_params(cfg, 32)
    bp = pkg.run_bp(cfg, store, 32, None, precision=precision)   # reference positional order
    single = pkg.run_single(cfg, store, seed=32, precision=precision)
    rep = pkg.compare_runs(single, bp, rtol=0.0)
    assert rep.bitwise, str(rep)
    assert sorted(bp.rank_fwd_seconds) == [0, 1]
    assert all(t > 0 for t in bp.rank_fwd_seconds.values())
    # one record per collective of the world, matching the closed form
    want = pkg.expected_comm_volume(cfg, pkg.ParallelLayout(bp=2))
    got = pkg.trace_volume(bp.trace)
    for key in (("fwd", "broadcast"), ("bwd", "broadcast"), ("bwd", "allreduce_sum")):
        assert got[key] == want[key], key
    assert got[("param", "broadcast")][1] == want[("param", "broadcast")][1]
    assert got[("param", "broadcast")][0] == 2 * cfg.n_blocks     # one bucket per branch
    assert set(p for p, _ in got) == {"fwd", "bwd", "param"}       # no result-assembly records
    assert bp.trace.by_phase()["fwd"][0] == 2 * cfg.n_blocks
    assert bp.trace.csv_text().startswith("seq,kind,group,src,elements,bytes,phase")


def test_bp2_dp2_four_ranks_matches_replica_mean(pkg):
    cfg = pkg.EvoConfig(**KW)
    store = pkg.init_params(cfg, 32)
    lay = pkg.ParallelLayout(dp=2, bp=2)
    res = pkg.run_distributed(cfg, store, lay, 32, precision="fp32")
    # the two replicas' samples: make_batch(cfg, 32, 2)[i]
    from paper_2211_00235_b200 import schedules as S
    samples = S.make_batch(cfg, 32, 2)
    reps = []
    for m, z in samples:
        st = S.StepState(cfg, store, "fp32")
        out = S.full_step(st, m, z)
        torch.cuda.synchronize()
        reps.append((out, st.grad_dict()))
    # replica 0's outputs come back; the gradients are the dp mean
    (m0, z0, l0, dm0, dz0), g0 = reps[0]
    (_, _, l1, _, _), g1 = reps[1]
    assert torch.equal(res.m_out, m0) and torch.equal(res.z_out, z0)
    assert torch.equal(res.dm, dm0) and torch.equal(res.dz, dz0)
    assert abs(res.loss - (float(l0) + float(l1)) / 2) <= 1e-6 * abs(res.loss)
    for n in g0:
        want = (g0[n].double() + g1[n].double()) / 2
        err = float((res.grads[n].double() - want).norm() / want.norm().clamp_min(1e-30))
        assert err <= 1e-6, n
    vol = pkg.trace_volume(res.trace)
    ref = pkg.expected_comm_volume(cfg, lay)
    for key in (("fwd", "broadcast"), ("bwd", "broadcast"), ("bwd", "allreduce_sum")):
        assert vol[key] == ref[key], key
    for key in (("param", "broadcast"), ("param", "allreduce_sum")):
        assert vol[key][1] == ref[key][1], key
    assert sorted(res.rank_fwd_seconds) == [0, 1, 2, 3]


def test_run_dp(pkg):
    cfg = pkg.EvoConfig(**{**KW, "n_blocks": 1})
    store = pkg.init_params(cfg, 32)
    res = pkg.run_dp(cfg, store, 2, precision="fp32")
    assert np.isfinite(res.loss)
    assert pkg.trace_volume(res.trace)[("param", "allreduce_sum")][1] == \
        pkg.expected_comm_volume(cfg, pkg.ParallelLayout(dp=2))[("param", "allreduce_sum")][1]


def _graphed_worker(rank, init_file, q):
    import traceback
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                                world_size=2)
        import paper_2211_00235_b200 as pkg
        from paper_2211_00235_b200 import distributed as D, schedules as S
        cfg = pkg.EvoConfig(**KW)
        store = pkg.init_params(cfg, 32, device="cuda:0")
        runner = D.DistributedStep(cfg, store, pkg.ParallelLayout(bp=2), precision="bf16",
                                   graphs=True)
        m, z = S.make_batch(cfg, 32, 1)[0]
        outs = []
        for _ in range(4):      # eager, capture, replay, replay
            out = runner.step(m.clone(), z.clone())
            torch.cuda.synchronize()
            # numpy (pickled by value: a torch CPU tensor would travel as
            # shared memory that dies with this process)
            outs.append([None if t is None else t.detach().float().cpu().numpy() for t in out])
        grads = {k: v.detach().cpu().numpy() for k, v in runner.ex.grad_dict().items()}
        q.put(("ok", rank, outs, grads, len(runner.ex.seg.graphs)))
        dist.destroy_process_group()
    except Exception:
        q.put(("err", rank, traceback.format_exc(), None, None))


def test_graphed_bp_segments_replay_bitwise(pkg):
    """DistributedStep(graphs=True): every compute segment between two
    collectives replays as a CUDA graph; replayed steps are bitwise equal to
    the eager first step and to the BP=1 step."""
    import os
    import tempfile
    import torch.multiprocessing as mp
    fd, init_file = tempfile.mkstemp()
    os.close(fd)
    os.unlink(init_file)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_graphed_worker, args=(r, init_file, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        status, rank, outs, grads, ngraphs = q.get()
        assert status == "ok", outs
        got[rank] = (outs, grads, ngraphs)
    for p in procs:
        p.join(timeout=60)
    cfg = pkg.EvoConfig(**KW)
    single = pkg.run_single(cfg, pkg.init_params(cfg, 32), seed=32, precision="bf16")
    for rank in (0, 1):
        outs, grads, ngraphs = got[rank]
        assert ngraphs >= 2 * cfg.n_blocks          # one graph per segment
        for step in range(1, 4):
            for a, b in zip(outs[0], outs[step]):
                assert (a is None and b is None) or np.array_equal(a, b), (rank, step)
        for n, g in single.grads.items():
            assert np.array_equal(grads[n], g.cpu().numpy()), n
    m_out = got[0][0][3][0]
    z_out = got[1][0][3][1]
    assert np.array_equal(m_out, single.m_out.cpu().numpy())
    assert np.array_equal(z_out, single.z_out.cpu().numpy())


def test_graphed_single_step_matches_eager(pkg):
    from paper_2211_00235_b200 import schedules as S
    cfg = pkg.EvoConfig(**KW)
    store = pkg.init_params(cfg, 32)
    m, z = S.make_batch(cfg, 32, 1)[0]
    st = S.StepState(cfg, store, "bf16")
    eager = [t.clone() for t in S.full_step(st, m, z)]
    g_eager = {k: v.clone() for k, v in st.grad_dict().items()}
    gs = st.capture(m, z, warmup=1, slots=2)
    for slot in (0, 1, 0):
        mi, zi = gs.inputs(slot)
        mi.copy_(m)
        zi.copy_(z)
        out = gs.step(mi, zi, slot=slot)
        torch.cuda.synchronize()
        for a, b in zip(eager, out):
            assert torch.equal(a, b)
        for k, v in st.grad_dict().items():
            assert torch.equal(v, g_eager[k]), k


EXTRA = dict(s=64, r=64, c_m=32, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=2)
MAIN = dict(s=32, r=64, c_m=64, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=1)


def _c3_inputs(cfg_e, cfg_m):
    rng = np.random.default_rng(32)
    return [torch.as_tensor(rng.standard_normal(shape).astype(np.float32), device="cuda")
            for shape in ((cfg_e.s, cfg_e.r, cfg_e.c_m), (cfg_m.s, cfg_m.r, cfg_m.c_m),
                          (cfg_m.r, cfg_m.r, cfg_m.c_z))]


def _c3_worker(rank, init_file, precision, q, ckpt=False):
    import traceback
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                                world_size=2)
        import paper_2211_00235_b200 as pkg
        from paper_2211_00235_b200 import distributed as D
        ce, cm = pkg.EvoConfig(**EXTRA), pkg.EvoConfig(**MAIN)
        lay = pkg.ParallelLayout(bp=2)
        comm = D.Comm(lay)
        ex_e = D.CudaExec(ce, pkg.init_params(ce, 33, device="cuda:0"), precision,
                          checkpoint=ckpt)
        ex_m = D.CudaExec(cm, pkg.init_params(cm, 32, device="cuda:0"), precision,
                          checkpoint=ckpt)
        out = D.composed_bp_step(ex_e, ex_m, comm, *_c3_inputs(ce, cm))
        torch.cuda.synchronize()
        grads = {**{"extra." + k: v.cpu().numpy() for k, v in ex_e.grad_dict().items()},
                 **{"main." + k: v.cpu().numpy() for k, v in ex_m.grad_dict().items()}}
        q.put(("ok", rank, [None if t is None else t.float().cpu().numpy() for t in out], grads))
        dist.destroy_process_group()
    except Exception:
        q.put(("err", rank, traceback.format_exc(), None))


@pytest.mark.parametrize("precision,ckpt", [("fp32", False), ("bf16", False), ("bf16", True)])
def test_c3_composed_stack_bp2_bitwise_equals_bp1(pkg, precision, ckpt):
    """C3 (extra-MSA stack -> main stack) under BP=2: bitwise equal to the
    one-GPU composition (schedules.composed_step); with per-block activation
    checkpointing on both BP ranks too (the C4 memory layout)."""
    import os
    import tempfile
    import torch.multiprocessing as mp
    from paper_2211_00235_b200 import schedules as S
    fd, init_file = tempfile.mkstemp()
    os.close(fd)
    os.unlink(init_file)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_c3_worker, args=(r, init_file, precision, q, ckpt))
             for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        status, rank, out, grads = q.get()
        assert status == "ok", out
        got[rank] = (out, grads)
    for p in procs:
        p.join(timeout=60)
    ce, cm = pkg.EvoConfig(**EXTRA), pkg.EvoConfig(**MAIN)
    ste = S.StepState(ce, pkg.init_params(ce, 33), precision)
    stm = S.StepState(cm, pkg.init_params(cm, 32), precision)
    m_out, z_out, loss, dm_e, dm, dz = S.composed_step(ste, stm, *_c3_inputs(ce, cm))
    torch.cuda.synchronize()
    (r0, g0), (r1, g1) = got[0], got[1]
    assert np.array_equal(r0[0], m_out.cpu().numpy())
    assert np.array_equal(r0[3], dm_e.cpu().numpy())
    assert np.array_equal(r0[4], dm.cpu().numpy())
    assert np.array_equal(r1[1], z_out.cpu().numpy())
    assert np.array_equal(r1[5], dz.cpu().numpy())
    assert np.float32(r0[2][0] + r1[2][0]) == np.float32(loss.item())
    want = {**{"extra." + k: v.cpu().numpy() for k, v in ste.grad_dict().items()},
            **{"main." + k: v.cpu().numpy() for k, v in stm.grad_dict().items()}}
    for n, g in want.items():
        assert np.array_equal(g0[n], g) and np.array_equal(g1[n], g), n


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_activation_checkpointing_bitwise(pkg, precision):
    """StepState(checkpoint=True) recomputes each block's forward before its
    backward: same kernels, same inputs -> bitwise the same step."""
    from paper_2211_00235_b200 import schedules as S
    cfg = pkg.EvoConfig(**KW)
    store = pkg.init_params(cfg, 32)
    m, z = S.make_batch(cfg, 32, 1)[0]
    a = S.StepState(cfg, store, precision)
    b = S.StepState(cfg, store, precision, checkpoint=True)
    out_a = [t.clone() for t in S.full_step(a, m, z)]
    out_b = S.full_step(b, m, z)
    for x, y in zip(out_a, out_b):
        assert torch.equal(x, y)
    ga, gb = a.grad_dict(), b.grad_dict()
    for k in ga:
        assert torch.equal(ga[k], gb[k]), k


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_branch_streams_bitwise(pkg, precision, monkeypatch):
    """The pair track on a second stream (engine.BRANCH_STREAMS) is the same
    launches on the same inputs: bitwise equal to running them back to back,
    eager and graph-captured."""
    from paper_2211_00235_b200 import engine as E, schedules as S
    cfg = pkg.EvoConfig(**KW)
    store = pkg.init_params(cfg, 32)
    m, z = S.make_batch(cfg, 32, 1)[0]
    monkeypatch.setattr(E, "BRANCH_STREAMS", False)
    a = S.StepState(cfg, store, precision)
    ref = [t.clone() for t in S.full_step(a, m, z)]
    g_ref = {k: v.clone() for k, v in a.grad_dict().items()}
    monkeypatch.setattr(E, "BRANCH_STREAMS", True)
    b = S.StepState(cfg, store, precision)
    out = S.full_step(b, m, z)
    torch.cuda.synchronize()
    for x, y in zip(ref, out):
        assert torch.equal(x, y)
    for k, v in b.grad_dict().items():
        assert torch.equal(v, g_ref[k]), k
    gs = b.capture(m, z, warmup=0)
    out = gs.step(m, z)
    torch.cuda.synchronize()
    for x, y in zip(ref, out):
        assert torch.equal(x, y)
    for k, v in b.grad_dict().items():
        assert torch.equal(v, g_ref[k]), k


def test_self_launched_world_of_one_runs_over_nccl(pkg):
    """A one-rank layout self-launches a world of one process with one GPU,
    so the NCCL backend is the one initialised (process group, groups,
    world ledger gather); the step equals run_single bitwise."""
    cfg = pkg.EvoConfig(**{**KW, "n_blocks": 1})
    store = pkg.init_params(cfg, 32)
    from paper_2211_00235_b200 import distributed as D
    assert torch.cuda.device_count() >= 1
    res = pkg.run_distributed(cfg, store, pkg.ParallelLayout(), 32, precision="bf16")
    single = pkg.run_single(cfg, store, seed=32, precision="bf16")
    rep = pkg.compare_runs(single, res, rtol=0.0)
    assert rep.bitwise, str(rep)
    assert sorted(res.rank_fwd_seconds) == [0]
    assert D.dist.is_available()
