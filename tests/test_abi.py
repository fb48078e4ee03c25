"""CPU tests of the C ABI: the library loads, exports every symbol include/gna.h
declares, validates arguments, and its host planner produces the tile plans
DESIGN.md describes (no device work)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from gna_inputs import WORKLOADS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gna():
    from paper_2504_16922_b200 import build

    build.build()
    import paper_2504_16922_b200 as pkg

    pkg.load()
    return pkg


def _header_functions():
    src = open(os.path.join(ROOT, "include", "gna.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(gna_\w+)\s*\(", src, flags=re.M)))


def test_exports_every_header_symbol(gna):
    from paper_2504_16922_b200.gna import EXPORTS

    names = _header_functions()
    assert len(names) >= 14
    assert sorted(EXPORTS) == names
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2504_16922_b200", "libgna_b200.so"))
    for n in names:
        assert hasattr(lib, n), n


def test_sm100a_code_in_library():
    """The .so carries sm_100a SASS with tcgen05 MMA, TMEM and TMA instructions."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump missing")
    lib = os.path.join(ROOT, "paper_2504_16922_b200", "libgna_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "STTM", "UTMALDG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


@pytest.mark.parametrize("bad,msg", [
    (dict(stride=(9,)), "holes"),
    (dict(dilation=(3,)), "exceeds extent"),
    (dict(window=(0,)), ">= 1"),
])
def test_validation_rejects(gna, bad, msg):
    from paper_2504_16922_b200.gna import GnaError

    kw = dict(spatial=(16,), window=(8,), stride=(1,), dilation=(1,))
    kw.update(bad)
    with pytest.raises(GnaError, match=msg):
        gna.workspace_size(1, 1, 64, kw["spatial"], kw["window"], kw["stride"], kw["dilation"])


def test_validation_unsupported_head_dim(gna):
    from paper_2504_16922_b200.gna import GnaError

    with pytest.raises(GnaError, match="head_dim"):
        gna.plan_info(1, 1, 96, (16,), (8,))


def test_spec_validate_examples(gna):
    """SPEC validate(): w=8,s=8,L=8 ok."""
    gna.plan_info(1, 1, 64, (8,), (8,), (8,))


@pytest.mark.parametrize("name", ["c2b_flux64_s16", "c3_cosmos", "c4a_hunyuan_blocked", "x1_hunyuan_s16", "x2_flux4k"])
def test_planner_reaches_flopwise_bound_on_block_sparse(gna, name):
    """Perfectly block-sparse configs: the planner's tiles give a
    NATTENSim bound equal to the FLOP-wise speedup N / prod(w)."""
    w = WORKLOADS[name]
    info = gna.plan_info(w.batch, w.heads, w.head_dim, **w.full())
    flop = w.n_tokens / np.prod(w.window)
    assert info["bound"] == pytest.approx(flop, rel=1e-9), info


def test_planner_kept_pairs_matches_oracle_count(gna):
    for name in ["c1_tiny1d", "c2a_flux64_s8", "s2c_sweep2d_causal", "s3_sweep3d"]:
        w = WORKLOADS[name]
        f = w.full()
        info = gna.plan_info(w.batch, w.heads, w.head_dim, **f)
        tot, _ = O.count_pairs(O.Params(f["spatial"], f["window"], f["stride"], f["dilation"], f["causal"]))
        assert info["kept_pairs"] == tot, name


def test_planner_bound_matches_oracle_sim_at_same_tiles(gna):
    """The plan's bound (dense boxes / max visited) equals the oracle simulator's
    at the plan's own tile shapes, when every item is one paired sub-tile
    block of identical range (paired within stride groups) or the Q tile is the
    sub-tile pair."""
    w = WORKLOADS["c4b_hunyuan_na"]
    f = w.full()
    info = gna.plan_info(1, 1, 128, **f)
    # NA items pair neighbouring sub-tiles: the union's visited count is the
    # visited count of the union tile, bounded by the oracle's per-sub-tile sim
    sim_sub = O.sim(O.Params(f["spatial"], f["window"], f["stride"]), info["q_sub"], info["box"])
    assert info["bound"] <= sim_sub["bound"] + 1e-9
    assert info["dense_boxes"] == sim_sub["dense_tiles"]


def test_worklist_covers_every_subtile_once(gna):
    for name in ["c1_tiny1d", "c2a_flux64_s8", "c4a_hunyuan_blocked", "s3_sweep3d", "s1_sweep1d"]:
        w = WORKLOADS[name]
        f = w.full()
        wl = gna.debug_worklist(**f)
        info = gna.plan_info(1, 1, w.head_dim, **f)
        seen = {}
        for cls, a, b, nbx in wl:
            for s in (a, b):
                if s >= 0:
                    assert (cls, s) not in seen
                    seen[(cls, s)] = True
        # every non-empty sub-tile of every class appears (sub-tiles fully in padding are skipped)
        q_sub = info["q_sub"]
        for cls in range(info["n_classes"]):
            Lc = O.class_extents(O.Params(f["spatial"], f["window"], f["stride"], f["dilation"], f["causal"]), cls)
            n_nonempty = int(np.prod([-(-Lc[a] // q_sub[a]) for a in range(3)]))
            assert sum(1 for (c, _s) in seen if c == cls) == n_nonempty, name


def test_plan_info_extra_tokens(gna):
    """Extra KV tokens: kept pairs grow by N*T; the NATTENSim bound counts the extra
    tiles as always visited: (dense + e) / (visited_max + e)."""
    w = WORKLOADS["x1_hunyuan_s16"]
    f = w.full()
    base = gna.plan_info(1, 1, 128, **f)
    ext = gna.plan_info(1, 1, 128, **f, n_extra=256)
    e = -(-256 // base["box_vol"])
    assert ext["kept_pairs"] == base["kept_pairs"] + w.n_tokens * 256
    assert ext["bound"] == pytest.approx((base["dense_boxes"] + e) / (base["visited_max"] + e))


def test_extra_tokens_validation(gna):
    from paper_2504_16922_b200.gna import GnaError

    with pytest.raises(GnaError, match="head_dim >= 64"):
        gna.plan_info(1, 1, 32, (64,), (8,), n_extra=4)
    with pytest.raises(GnaError, match="n_extra"):
        gna.plan_info(1, 1, 64, (64,), (8,), n_extra=-1)


def test_fp8_validation_without_gpu():
    """GNA_DTYPE_FP8_E4M3 argument checks run before any device access (nothing launched)."""
    import ctypes
    import paper_2504_16922_b200.gna as G
    lib = G.load()
    a = G.make_args(1, 1, 64, (64,), (16,), dtype=G.GNA_DTYPE_FP8_E4M3)
    assert lib.gna_forward_ex(ctypes.byref(a)) == G.GNA_EUNSUPPORTED  # head_dim 64
    a = G.make_args(1, 1, 128, (64,), (16,), dtype=G.GNA_DTYPE_FP8_E4M3, scales=(-1.0, 1.0, 1.0))
    assert lib.gna_forward_ex(ctypes.byref(a)) == G.GNA_EINVAL
    a = G.make_args(1, 1, 128, (64,), (16,), dtype=7)
    assert lib.gna_forward_ex(ctypes.byref(a)) == G.GNA_EUNSUPPORTED
