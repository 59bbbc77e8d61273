"""CPU: pin the oracles (C restatement + NumPy sort) against the reference's own
golden vectors / known answers and against fixtures generated
from the unmodified reference (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPECS = [(0, 0), (0, 1), (1, 0), (1, 1)]


def test_eq1_key_golden_vectors():
    """test_flatten.cpp:26-60 examples + window-boundary keys, bit-exact (fp64 hex)."""
    keys = json.load(open(os.path.join(GOLD, "keys.json")))
    for k in keys:
        wm, wn, lm, ln = O.np_sort_keys(np.array([[k["x"], k["y"]]]), k["w_x"], k["w_y"],
                                         k["shift"], k["axis_y"])
        assert (int(wm[0]), int(wn[0])) == (k["win_major"], k["win_minor"])
        assert float(lm[0]).hex() == k["loc_major"] and float(ln[0]).hex() == k["loc_minor"]
    # the reference's literal expectations (test_flatten.cpp)
    assert (keys[0]["win_major"], keys[0]["win_minor"]) == (1, 0)          # (3.5,1.0), w=2
    assert (keys[1]["win_major"], keys[1]["win_minor"]) == (-1, 0)         # floor for negatives
    assert float.fromhex(keys[1]["loc_major"]) == 1.5
    assert float.fromhex(keys[2]["loc_major"]) == 1.0                      # shift by w/2
    assert (keys[3]["win_major"], keys[3]["win_minor"]) == (2, 1)          # Y-major swap


@pytest.mark.parametrize("impl", ["numpy", "port"])
def test_sort_oracles_match_reference(impl):
    d = np.load(os.path.join(GOLD, "sort_cases.npz"))
    for name in d["names"]:
        c = d[f"{name}_coords"]
        wx, wy = d[f"{name}_w"]
        for ay, sh in SPECS:
            want = d[f"{name}_perm_{ay}{sh}"]
            got = O.np_sort(c, wx, wy, sh, ay) if impl == "numpy" else O.port_sort(c, wx, wy, sh, ay)
            assert np.array_equal(got, want), (impl, name, ay, sh)
    assert list(d["ident_perm_00"]) == [0, 1, 2]  # test_flatten.cpp:62-66


def test_group_counts_known_answers():
    import paper_2301_08739_b200 as F
    m, dr = F.group(np.arange(10, dtype=np.int32), 4)       # test_flatten.cpp:156-168
    assert m.shape == (2, 4) and list(dr) == [8, 9]
    m, dr = F.group(np.arange(69, dtype=np.int32), 69)      # 178-185
    assert m.shape == (1, 69) and len(dr) == 0
    with pytest.raises(F.ConfigError):
        F.group(np.arange(3, dtype=np.int32), 0)
    sched = F.block_schedule(8, 2.88, 2.88)                 # flatten.hpp:150-161
    assert [(s.major_axis, s.shift) for s in sched[:4]] == [("X", False), ("X", True), ("Y", False), ("Y", True)]


def _small_cfg(**kw):
    base = dict(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=8)
    base.update(kw)
    return O.make_cfg(**base)


def _grid(n, d, seed, grid_w=200):
    """acceptance.cpp:435-449 grid_pillars (features from numpy here)."""
    i = np.arange(n)
    coords = np.stack([((i % grid_w) + 0.5) * 0.32, ((i // grid_w) + 0.5) * 0.32], 1)
    feats = np.random.default_rng(seed).normal(size=(n, d))
    return coords, feats


def _blob(cfg, seed):
    import paper_2301_08739_b200 as F
    return F.init_backbone_params(F.FwaConfig(cfg.resolution, cfg.window_px, cfg.window_py,
                                              cfg.group_size, cfg.n_blocks, cfg.d_model,
                                              cfg.n_heads, cfg.d_ff), seed)


def test_port_cache_and_drop_known_answers():
    # 8-block drop-free: 4 computed, 4 hits (acceptance.cpp:451-465; test_backbone.cpp:149-183)
    cfg = _small_cfg()
    c, f = _grid(640, 16, 8001)
    r = O.port_run_backbone(c, f.astype(np.float32), cfg, _blob(cfg, 5))
    assert r["cache"] == (4, 4) and r["dropped_per_block"].sum() == 0 and len(r["kept"]) == 640
    # single block: 1 / 0
    cfg1 = _small_cfg(n_blocks=1)
    r = O.port_run_backbone(c, f.astype(np.float32), cfg1, _blob(cfg1, 5))
    assert r["cache"] == (1, 0)
    # drops in block 0: 5 / 3 and N mod G dropped (acceptance.cpp:496-536: 30000 mod 69 = 54)
    cfg2 = _small_cfg(group_size=69, n_blocks=8)
    c2, f2 = _grid(30000, 16, 10001)
    r = O.port_run_backbone(c2, f2.astype(np.float32), cfg2, _blob(cfg2, 13))
    assert list(r["dropped_per_block"]) == [54, 0, 0, 0, 0, 0, 0, 0]
    assert r["cache"] == (5, 3)
    assert len(r["kept"]) == 30000 - 54 and np.all(np.diff(r["kept"]) > 0)
    assert not np.isin(r["dropped"], r["kept"]).any()


def test_port_zero_weights_identity():
    """acceptance.cpp:477-493: zero-weight blocks are the identity on kept pillars."""
    cfg = _small_cfg(group_size=13, n_blocks=4)
    c, f = _grid(901, 16, 9001)
    zero = b"".join([b"FWAP" + np.array([16, 4, 32], np.uint32).tobytes() +
                     np.zeros(3 * 256 + 48 + 256 + 16 + 64 + 512 + 32 + 512 + 16, np.float32).tobytes()
                     for _ in range(4)])
    r = O.port_run_backbone(c, f.astype(np.float32), cfg, zero)
    assert np.array_equal(r["features"], f.astype(np.float32)[r["kept"]])


def test_port_backbone_matches_reference_golden_small():
    g = np.load(os.path.join(GOLD, "backbone_small.npz"))
    d, h, dff, G, nb = (int(x) for x in g["cfg"])
    cfg = O.make_cfg(d_model=d, n_heads=h, d_ff=dff, group_size=G, n_blocks=nb)
    r = O.port_run_backbone(g["coords"], g["feats"].astype(np.float32), cfg, g["blob"].tobytes(),
                            want_perms=True)
    assert np.array_equal(r["features"], g["features"])          # bit-exact
    assert np.array_equal(r["kept"], g["kept"])
    assert np.array_equal(r["dropped"], g["dropped"])
    assert np.array_equal(r["dropped_per_block"], g["dropped_per_block"])
    assert tuple(r["cache"]) == tuple(g["cache"])
    for b in range(nb):
        plan = g[f"plan{b}"]
        assert np.array_equal(r["block_perms"][b, :len(plan)], plan)


def test_port_backbone_matches_reference_golden_d128():
    import paper_2301_08739_b200 as F
    g = np.load(os.path.join(GOLD, "backbone_d128.npz"))
    s = [float(x) for x in g["scene"]]
    scene = F.SceneSpec(int(s[0]), int(s[1]), int(s[2]), s[3], s[4], s[5], int(s[6]), int(s[7]))
    ps = F.make_pillars(scene, int(g["scene_seed"]))
    cfg = O.make_cfg()
    blob = F.init_backbone_params(F.FwaConfig(), int(g["param_seed"]))
    r = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), cfg, blob, want_perms=True)
    assert np.array_equal(r["features"], g["features"])
    assert np.array_equal(r["kept"], g["kept"]) and np.array_equal(r["dropped"], g["dropped"])
    assert tuple(r["cache"]) == tuple(g["cache"]) == (5, 3)
    for b in range(8):
        plan = g[f"plan{b}"]
        assert np.array_equal(r["block_perms"][b, :len(plan)], plan)


def test_port_block_matches_reference_golden():
    import paper_2301_08739_b200 as F
    g = np.load(os.path.join(GOLD, "block_d128.npz"))
    blob = F.init_backbone_params(F.FwaConfig(), int(g["param_seed"]))
    rec = blob[:len(blob) // 8]
    out = O.port_block_forward(g["f"], g["pe"], 3, rec)
    assert np.array_equal(out, g["out32"])
    assert O.max_rel_err(g["out32"], g["out64"]) < 1e-5      # acceptance.cpp:203-239 bar


def test_port_positional_embedding_examples():
    """SPEC.md kernels examples: (0,0) -> sin 0, cos 1."""
    pe = O.port_positional_embedding(np.zeros((1, 2)), 16)
    assert np.all(pe[0, 0::2] == 0.0) and np.all(pe[0, 1::2] == 1.0)


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_port_equals_reference_live():
    """The C restatement against the compiled reference on fresh random inputs."""
    rng = np.random.default_rng(5)
    for trial in range(3):
        n = int(rng.integers(300, 900))
        c = rng.uniform(-20, 20, size=(n, 2))
        f = rng.normal(size=(n, 16))
        cfg = _small_cfg(group_size=int(rng.integers(5, 40)), n_blocks=int(rng.integers(1, 9)))
        blob = O.ref_init_params(cfg, 16, trial)
        a = O.ref_run_backbone(c, f, cfg, blob)
        b = O.port_run_backbone(c, f.astype(np.float32), cfg, blob)
        assert np.array_equal(a["features"], b["features"])
        assert np.array_equal(a["dropped"], b["dropped"]) and a["cache"] == b["cache"]
        for ay, sh in SPECS:
            assert np.array_equal(O.ref_sort(c, 2.88, 2.88, sh, ay), O.port_sort(c, 2.88, 2.88, sh, ay))
            assert np.array_equal(O.ref_sort(c, 2.88, 2.88, sh, ay, brute=True),
                                  O.np_sort(c, 2.88, 2.88, sh, ay))


def test_np_pillarize_matches_reference_pillars():
    """The pillarize restatement (oracle.np_pillarize) reproduces the compiled reference's
    generate_synthetic + pillarize bit for bit on a small scene (coords, order, features)."""
    import paper_2301_08739_b200 as F
    scene = F.SceneSpec(6, 20, 40, 1.0, 20.0, 20.0, 150, 2)
    xy, f = F.generate_points(scene, 9)
    w = F.pillar_params(2, 16, 9)
    coords, feats = O.np_pillarize(xy, f, 0.32, w)
    want = F.make_pillars(scene, 9, d_out=16)          # host port, pinned to the reference
    assert np.array_equal(coords, want.coords)
    assert np.array_equal(feats, want.features)
    if O.have_ref():
        r = O.ref_make_pillars({"n_clusters": 6, "ppc_min": 20, "ppc_max": 40, "sigma": 1.0, "ext_x": 20.0,
                                "ext_y": 20.0, "n_bg": 150, "f_in": 2}, 9, d_out=16)
        assert np.array_equal(coords, r[0]) and np.array_equal(feats, r[1])
