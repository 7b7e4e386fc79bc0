"""CPU tests of the host side: the C-ABI library loads and exports every
symbol include/evo_b200.h declares (no compute call without a GPU), and
the host logic mirrors the reference (params, layout math, comm ledger)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "evo_b200.h")).read()
    return sorted(set(re.findall(r"\b(evo_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2211_00235_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED)


def test_library_identity_without_gpu():
    from paper_2211_00235_b200 import _native
    L = _native.lib()
    assert L.evo_version() == 1
    assert L.evo_launch_count() >= 0


def test_so_is_sm100a():
    from paper_2211_00235_b200 import _native
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_params_bit_identical_to_reference_rng():
    from oracle import evoformer_np as O
    import paper_2211_00235_b200 as pkg
    cfg = pkg.EvoConfig(s=5, r=6, c_m=4, c_z=6, h=2, c_opm=3, n_blocks=2)
    store = pkg.init_params(cfg, 7, device="cpu")
    P = O.init_params(O.Dims.of(cfg), 7, dtype=np.float32)
    assert store.names() == list(P)
    for n in P:
        assert np.array_equal(store[n].numpy(), P[n]), n
    assert pkg.param_count(cfg) == store.total_size() == sum(v.size for v in P.values())
    assert len(store) == 93 * cfg.n_blocks


def test_config_validation():
    import paper_2211_00235_b200 as pkg
    with pytest.raises(pkg.ConfigError):
        pkg.EvoConfig(c_m=8, h=3)
    with pytest.raises(pkg.ConfigError):
        pkg.EvoConfig(variant="serial")
    with pytest.raises(pkg.ConfigError):
        pkg.EvoConfig(s=0)
    with pytest.raises(pkg.ConfigError):
        pkg.set_precision("fp8")


def test_layout_rank_math_matches_reference():
    from paper_2211_00235_b200 import ParallelLayout, ConfigError
    lay = ParallelLayout(dp=4, bp=2)
    assert lay.world_size == 8
    assert lay.bp_group(5) == (4, 5)
    assert lay.dp_group(5) == (1, 3, 5, 7)
    assert lay.dp_group(0) == (0, 2, 4, 6)
    for r in range(8):
        assert lay.rank_of(*lay.coords(r)) == r
    with pytest.raises(ConfigError, match="two branches"):
        ParallelLayout(bp=3)


def test_comm_volume_matches_reference_closed_form():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from branchpar import evoformer as RE, schedules as RS
    except ImportError:
        pytest.skip("reference not present on this machine")
    import paper_2211_00235_b200 as pkg
    kw = dict(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=2)
    for dp, bp, dap in ((1, 2, 1), (2, 1, 1), (4, 2, 1), (2, 2, 1), (1, 1, 2), (1, 1, 4),
                        (1, 2, 2), (2, 2, 2), (2, 1, 4)):
        mine = pkg.expected_comm_volume(pkg.EvoConfig(**kw),
                                        pkg.ParallelLayout(dp=dp, bp=bp, dap=dap))
        ref = RS.expected_comm_volume(RE.EvoConfig(**kw), RS.ParallelLayout(dp=dp, bp=bp, dap=dap))
        assert mine == ref, (dp, bp, dap)


def test_product_path_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2211_00235_b200 import _native
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeLibraryMissing):
        _native.lib()
