"""Run configuration, cost model and command line front end
(src/config.py, src/costmodel.py, src/cli.py; the reference's
tests/test_cli.py and tests/test_costmodel.py are the model).  CPU: config
parsing and errors, the cost model against the reference's closed forms
(imported when /root/reference is present), the cost command.  GPU: verify,
gradcheck and bench on the toy config."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "configs")


def _ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import branchpar.costmodel as RC
        import branchpar.evoformer as RE
        import branchpar.schedules as RS
    except ImportError:
        pytest.skip("reference not present on this machine")
    return RC, RE, RS


def test_reference_config_files_load():
    from paper_2211_00235_b200.config import load_config
    for name in ("toy", "bench_large", "initial_training", "fine_tuning",
                 "initial_training_b200", "fine_tuning_b200"):
        rc = load_config(os.path.join(CFG, f"{name}.cfg"))
        assert rc.model.n_blocks >= 2 and rc.precision in ("f32", "bf16")
    rc = load_config(os.path.join(CFG, "fine_tuning_b200.cfg"))
    assert rc.device.msa_rate and rc.device.pair_rate and rc.device.precision_bytes == 2
    ref = "/root/reference/pkg/configs/toy.cfg"
    if os.path.exists(ref):            # the reference's own file, f64 -> f32
        rc = load_config(ref)
        assert rc.precision == "f32" and rc.notes and rc.layout.bp == 2


@pytest.mark.parametrize("text,msg", [
    ("model.s = 8\nmodel.r = 16\nmodel.c_m = 8\nmodel.c_z = 8\nmodel.h = 2\nmodel.bogus = 1\n",
     "unknown config key"),
    ("model.s = 8\nmodel.s = 8\n", "repeated key"),
    ("model.s = 8\n", "missing required model keys"),
    ("model.s = eight\n", "cannot parse"),
    ("model.s\n", "expected 'key = value'"),
    ("model.s = 8\nmodel.r = 16\nmodel.c_m = 8\nmodel.c_z = 8\nmodel.h = 2\n"
     "run.precision = f16\n", "precision must be one of"),
])
def test_config_errors(text, msg):
    from paper_2211_00235_b200.config import parse_config
    from paper_2211_00235_b200.errors import ConfigError
    with pytest.raises(ConfigError, match=msg):
        parse_config(text)


def test_cost_model_matches_reference_closed_forms():
    RC, RE, RS = _ref()
    from paper_2211_00235_b200 import EvoConfig, ParallelLayout
    from paper_2211_00235_b200 import costmodel as C
    layouts = [(1, 1, 1), (1, 2, 1), (1, 1, 2), (1, 2, 2), (1, 1, 4), (1, 2, 4), (2, 2, 2),
               (4, 2, 1)]
    for kw in (dict(s=128, r=256, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=52),
               dict(s=512, r=384, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=52),
               dict(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=2)):
        mine_cfg, ref_cfg = EvoConfig(**kw), RE.EvoConfig(**kw)
        assert C.op_flops(mine_cfg) == RC.op_flops(ref_cfg)
        for dev_kw in ({}, dict(non_evoformer_time=3.67, precision_bytes=4)):
            md, rd = C.DeviceModel(**dev_kw), RC.DeviceModel(**dev_kw)
            for dp, bp, dap in layouts:
                ml, rl = ParallelLayout(dp=dp, bp=bp, dap=dap), RS.ParallelLayout(dp=dp, bp=bp,
                                                                                   dap=dap)
                if kw["s"] % dap or kw["r"] % dap:
                    continue
                a, b = C.step_time(mine_cfg, ml, md), RC.step_time(ref_cfg, rl, rd)
                assert abs(a.total - b.total) <= 1e-12 * b.total, (kw, dev_kw, dp, bp, dap)
                assert a.bottleneck == b.bottleneck
            bl = RS.ParallelLayout(bp=2)
            assert C.schedule_bytes(mine_cfg, ParallelLayout(bp=2), md) == \
                RC.schedule_bytes(ref_cfg, bl, rd)
    assert C.end_to_end_days(1.0, 2.0) == RC.end_to_end_days(1.0, 2.0)


def test_b200_model_prices_branches_apart():
    from paper_2211_00235_b200 import ParallelLayout
    from paper_2211_00235_b200 import costmodel as C
    cfg = C.INITIAL_TRAINING_MODEL
    t1 = C.step_time(cfg, ParallelLayout(), C.B200_DEVICE)
    t2 = C.step_time(cfg, ParallelLayout(bp=2), C.B200_DEVICE)
    assert t2.bottleneck == "pair"            # the slower branch on B200
    msa, pair = C.branch_flops(cfg)
    # the two branches' measured fwd+bwd times, 1.33 + 1.96 ms per C2 block
    per_block = (msa / C.B200_DEVICE.msa_rate + pair / C.B200_DEVICE.pair_rate) * 3
    assert abs(per_block - 3.29e-3) < 0.02e-3
    assert 1.3 < t1.total / t2.total < 1.7


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2211_00235_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_cost_and_errors(tmp_path):
    p = _cli("cost", os.path.join(CFG, "initial_training.cfg"), "--out", str(tmp_path / "c.csv"))
    assert p.returncode == 0, p.stderr
    lines = p.stdout.strip().splitlines()
    assert lines[0] == "layout,step_seconds,proteins_per_second,speedup_pct"
    assert lines[1].startswith("dp1.bp1.dap1,")
    assert sum(ln.startswith("dp") for ln in lines) == 6 and lines[-1].startswith("wrote ")
    assert (tmp_path / "c.csv").read_text().startswith("layout,")
    bad = tmp_path / "bad.cfg"
    bad.write_text("model.s = 8\nmodel.typo = 3\n")
    p = _cli("cost", str(bad))
    assert p.returncode == 2 and "unknown config key" in p.stderr
    p = _cli("cost", str(tmp_path / "missing.cfg"))
    assert p.returncode == 2 and "cannot read config" in p.stderr
    p = _cli("nonsense")
    assert p.returncode == 2


@pytest.mark.gpu
def test_cli_verify_gradcheck_bench(tmp_path):
    p = _cli("verify", os.path.join(CFG, "toy.cfg"))
    assert p.returncode == 0 and "verify: PASS" in p.stdout, p.stdout + p.stderr
    assert "dp1.bp2.dap1" in p.stdout
    dap = tmp_path / "dap.cfg"
    dap.write_text(open(os.path.join(CFG, "toy.cfg")).read().replace("layout.bp = 2",
                                                                     "layout.bp = 1")
                   .replace("layout.dap = 1", "layout.dap = 2"))
    p = _cli("verify", str(dap))
    assert p.returncode == 0 and "verify: PASS" in p.stdout, p.stdout + p.stderr
    p = _cli("gradcheck", os.path.join(CFG, "toy.cfg"))
    assert p.returncode == 0 and "gradcheck: PASS" in p.stdout, p.stdout + p.stderr
    assert p.stdout.count("PASS") == 11          # 9 sub-ops, the block, the summary
    p = _cli("bench", os.path.join(CFG, "toy.cfg"), "--repeat", "8")
    assert p.returncode == 0, p.stdout + p.stderr
    assert "bench single:" in p.stdout and "bench speedup:" in p.stdout
