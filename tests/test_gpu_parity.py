"""GPU parity: the CUDA path (through the C ABI) vs the oracles.

Integer outputs (window-sort permutations, groups, drops, kept set, cache stats)
must be bit-exact.  Features: normwise max rel err (tests/test_kernels.cpp:25-33)
<= 1e-4 in the fp32 check mode and <= 1e-2 in the bf16 tensor-core mode (the
north-star tolerances).  Full-size frames are checked through size-independent
properties (sortedness of the reference keys, permutation/partition invariants,
zero-weight identity, determinism, batch == per-frame)."""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2301_08739_b200 as F

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPECS = [(0, 0), (0, 1), (1, 0), (1, 1)]
TOL_FP32, TOL_BF16 = 1e-4, 1e-2


@pytest.fixture(scope="module")
def ctx32():
    return F.Context(0, precision="fp32")


@pytest.fixture(scope="module")
def ctx16():
    return F.Context(0, precision="bf16")


def _spec(w, ay, sh):
    return F.WindowSpec(w[0], w[1], bool(sh), "Y" if ay else "X")


# ----------------------------------------------------------------------------- sort

def test_sort_golden_cases(ctx32):
    d = np.load(os.path.join(GOLD, "sort_cases.npz"))
    for name in d["names"]:
        c = d[f"{name}_coords"]
        w = d[f"{name}_w"]
        for ay, sh in SPECS:
            got = ctx32.sort(c, _spec(w, ay, sh))
            assert np.array_equal(got, d[f"{name}_perm_{ay}{sh}"]), (name, ay, sh)


def test_sort_random_scenes_vs_numpy_oracle(ctx32):
    """acceptance.cpp:138-179 style: random scenes up to 10k points, w = 2.88, all specs,
    plus boundary/duplicate scenes and an oversize-window scene (CTA + bitonic bins)."""
    rng = np.random.default_rng(1001)
    for trial in range(24):
        n = int(rng.integers(100, 10000))
        c = rng.uniform(-50, 50, size=(n, 2))
        ay, sh = SPECS[trial % 4]
        assert np.array_equal(ctx32.sort(c, _spec((2.88, 2.88), ay, sh)), O.np_sort(c, 2.88, 2.88, sh, ay))
    for v in range(4):
        c = 2.0 * (rng.integers(0, 9, size=(2000, 2)).astype(np.float64) - 4.0)
        if v >= 2:
            c = np.concatenate([c, c[::3]])
        for ay, sh in SPECS:
            assert np.array_equal(ctx32.sort(c, _spec((2.0, 2.0), ay, sh)), O.np_sort(c, 2.0, 2.0, sh, ay))
    # big windows: bins of ~300 (CTA rank sort) and ~6000 (bitonic network) points
    for w in (10.0, 60.0):
        c = rng.uniform(-60, 60, size=(20000, 2)).round(1)  # many exact ties in loc
        for ay, sh in SPECS:
            assert np.array_equal(ctx32.sort(c, _spec((w, w), ay, sh)), O.np_sort(c, w, w, sh, ay))
    # identical points sort by original index (test_flatten.cpp:62-66); non-square windows
    assert list(ctx32.sort(np.ones((3, 2)), F.WindowSpec(2.0, 2.0))) == [0, 1, 2]
    c = rng.uniform(-10, 10, size=(500, 2))
    assert np.array_equal(ctx32.sort(c, F.WindowSpec(1.5, 0.75, True, "Y")), O.np_sort(c, 1.5, 0.75, 1, 1))


def test_sort_full_size_frames_all_specs(ctx32):
    """F60 (60,897 pillars) and F250 (255,066): bit-exact vs the NumPy oracle, and the
    reference keys are lexicographically non-decreasing along the GPU permutation."""
    w = 9 * 0.32
    for name in ("F60", "F250"):
        ps = F.make_pillars(F.SCENES[name], 42)
        for ay, sh in SPECS:
            got = ctx32.sort(ps.coords, _spec((w, w), ay, sh))
            assert np.array_equal(got, O.np_sort(ps.coords, w, w, sh, ay)), (name, ay, sh)
            wm, wn, lm, ln = O.np_sort_keys(ps.coords, w, w, sh, ay)
            k = np.stack([wm[got], wn[got]], 1)
            assert np.all((np.diff(k[:, 0]) > 0) | ((np.diff(k[:, 0]) == 0) & (np.diff(k[:, 1]) >= 0)))
            assert np.array_equal(np.sort(got), np.arange(ps.size()))


# ----------------------------------------------------------------------------- positional embedding

def test_positional_embedding(ctx32):
    ps = F.make_pillars(F.SCENES["F10"], 42)
    got = ctx32.positional_embedding(ps.coords, 128)
    want = O.port_positional_embedding(ps.coords, 128)
    assert np.max(np.abs(got - want)) <= 1e-6  # fp64 sin/cos, f32 rounding


def test_positional_embedding_fp16_fast_path(ctx16):
    """fp16 PE rows of the bf16 path: within fp16 rounding of the reference's fp64 values,
    on F60 and on coordinates far from the origin (large phases, exact range reduction)."""
    for coords in (F.make_pillars(F.SCENES["F60"], 42).coords,
                   np.random.default_rng(7).uniform(-3000.0, 3000.0, size=(5000, 2))):
        got = ctx16.positional_embedding_f16(coords, 128).astype(np.float64)
        want = O.port_positional_embedding(coords, 128).astype(np.float64)
        # half an fp16 ulp of |v| <= 1 is 2^-12; + 1e-6 for the fp32 sincospi
        assert np.max(np.abs(got - want)) <= 2.0 ** -12 + 1e-6


# ----------------------------------------------------------------------------- block

def test_block_forward_fp32_vs_f64_oracle(ctx32):
    """acceptance.cpp:203-239 (C3): f32 block vs dense f64 oracle; here on the GPU
    fp32 check path at several (G, D, H) shapes incl. G=1 and identical tokens."""
    rng = np.random.default_rng(1003)
    shapes = [(1, 16, 4), (7, 8, 2), (13, 32, 8), (31, 64, 4), (5, 12, 1), (29, 48, 8),
              (17, 24, 2), (32, 40, 8), (3, 4, 1), (20, 56, 8)]
    for trial, (G, D, H) in enumerate(shapes):
        ng = int(rng.integers(1, 4))
        cfg = F.FwaConfig(d_model=D, n_heads=H, d_ff=2 * D, n_blocks=1)
        rec = F.init_backbone_params(cfg, trial)
        f = rng.normal(size=(ng * G, D)).astype(np.float32)
        pe = (0.3 * rng.normal(size=(ng * G, D))).astype(np.float32)
        if trial == 1:
            f[:] = f[0]
            pe[:] = pe[0]
        got = ctx32.fwa_block_forward(f, pe, rec, ng)
        want = O.port_block_forward(f, pe, ng, rec)
        assert O.max_rel_err(got, want) <= 1e-5, (trial, G, D, H)


def test_block_forward_golden_d128(ctx32, ctx16):
    g = np.load(os.path.join(GOLD, "block_d128.npz"))
    blob = F.init_backbone_params(F.FwaConfig(), int(g["param_seed"]))
    rec = blob[:len(blob) // 8]
    e32 = O.max_rel_err(ctx32.fwa_block_forward(g["f"], g["pe"], rec, 3), g["out64"])
    e16 = O.max_rel_err(ctx16.fwa_block_forward(g["f"], g["pe"], rec, 3), g["out64"])
    assert e32 <= 1e-5, e32
    assert e16 <= TOL_BF16, e16
    assert ctx16.fast_path(F.FwaConfig(group_size=69))


@pytest.mark.parametrize("G", [16, 33, 64, 69, 128])
def test_block_forward_bf16_group_sizes(ctx16, G):
    """tcgen05 QKV / out-proj+FFN and mma.sync attention at several group sizes."""
    rng = np.random.default_rng(G)
    cfg = F.FwaConfig(group_size=G)
    rec = F.init_backbone_params(cfg, 3)[:16 + 4 * 132480]
    ng = 300 // G + 1
    f = rng.normal(size=(ng * G, 128)).astype(np.float32)
    pe = (0.3 * rng.normal(size=(ng * G, 128))).astype(np.float32)
    got = ctx16.fwa_block_forward(f, pe, rec, ng)
    want = O.port_block_forward(f, pe, ng, rec)
    assert O.max_rel_err(got, want) <= TOL_BF16


def test_fused_attention_shifted_fallback(ctx16, monkeypatch):
    """The fused kernel's attention runs P = 2^S without the row-max shift and re-runs a
    task with the reference's max-subtracted softmax when a row sum leaves [1/lmax, lmax].
    Forcing lmax = 2 sends most tasks down the shifted path: both agree with the oracle and
    with each other (same math, different rounding)."""
    rng = np.random.default_rng(5)
    cfg = F.FwaConfig()
    rec = F.init_backbone_params(cfg, 3)[:16 + 4 * 132480]
    ng = 12
    f = rng.normal(size=(ng * 69, 128)).astype(np.float32)
    pe = (0.3 * rng.normal(size=(ng * 69, 128))).astype(np.float32)
    fast = ctx16.fwa_block_forward(f, pe, rec, ng)
    monkeypatch.setenv("FWA_B200_ATTN_LMAX", "2")
    shifted = ctx16.fwa_block_forward(f, pe, rec, ng)
    want = O.port_block_forward(f, pe, ng, rec)
    assert O.max_rel_err(fast, want) <= TOL_BF16
    assert O.max_rel_err(shifted, want) <= TOL_BF16
    assert O.max_rel_err(shifted, fast) <= 3e-3
    assert not np.array_equal(shifted, fast)  # the shifted path did run


# ----------------------------------------------------------------------------- backbone

def _check_ints(res, want_kept, want_dropped, want_dpb, want_cache):
    assert np.array_equal(res.kept_indices, want_kept)
    assert np.array_equal(np.concatenate(res.dropped_indices), want_dropped)
    assert list(res.stats.dropped_per_block) == list(want_dpb)
    assert (res.stats.cache.computed, res.stats.cache.hits) == tuple(want_cache)


def test_backbone_golden_small(ctx32):
    g = np.load(os.path.join(GOLD, "backbone_small.npz"))
    d, h, dff, G, nb = (int(x) for x in g["cfg"])
    cfg = F.FwaConfig(d_model=d, n_heads=h, d_ff=dff, group_size=G, n_blocks=nb)
    ctx32.load_params(cfg, g["blob"].tobytes())
    r = ctx32.run_backbone(F.PillarSet(g["coords"], g["feats"]), cfg, want_block_perms=True)
    _check_ints(r, g["kept"], g["dropped"], g["dropped_per_block"], g["cache"])
    for b in range(nb):
        assert np.array_equal(r.block_perms[b], g[f"plan{b}"]), b
    assert O.max_rel_err(r.features, g["features"]) <= TOL_FP32


@pytest.mark.parametrize("prec,tol", [("fp32", TOL_FP32), ("bf16", TOL_BF16)])
def test_backbone_golden_d128(prec, tol, ctx32, ctx16):
    ctx = ctx32 if prec == "fp32" else ctx16
    g = np.load(os.path.join(GOLD, "backbone_d128.npz"))
    s = [float(x) for x in g["scene"]]
    scene = F.SceneSpec(int(s[0]), int(s[1]), int(s[2]), s[3], s[4], s[5], int(s[6]), int(s[7]))
    ps = F.make_pillars(scene, int(g["scene_seed"]))
    cfg = F.FwaConfig()
    ctx.load_params(cfg, F.init_backbone_params(cfg, int(g["param_seed"])))
    r = ctx.run_backbone(ps, cfg, want_block_perms=True)
    _check_ints(r, g["kept"], g["dropped"], g["dropped_per_block"], g["cache"])
    for b in range(8):
        assert np.array_equal(r.block_perms[b], g[f"plan{b}"]), b
    err = O.max_rel_err(r.features, g["features"])
    assert err <= tol, err


@pytest.mark.parametrize("prec,tol", [("fp32", TOL_FP32), ("bf16", TOL_BF16)])
def test_backbone_config1_f30_one_block(prec, tol, ctx32, ctx16):
    """BASELINE config 1: one block (X, no shift), G 69, D 128, H 8 on F30 (30,212 pillars)."""
    ctx = ctx32 if prec == "fp32" else ctx16
    ps = F.make_pillars(F.SCENES["F30"], 42)
    cfg = F.FwaConfig(n_blocks=1)
    blob = F.init_backbone_params(cfg, 42)
    ctx.load_params(cfg, blob)
    r = ctx.run_backbone(ps, cfg)
    w = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), O.make_cfg(n_blocks=1), blob)
    _check_ints(r, w["kept"], w["dropped"], w["dropped_per_block"], w["cache"])
    assert r.stats.dropped_per_block == [30212 % 69]
    err = O.max_rel_err(r.features, w["features"])
    assert err <= tol, err


def test_backbone_cache_counts_and_drops(ctx32):
    """test_backbone.cpp:149-183 / acceptance.cpp:451-465, 496-536."""
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=8)
    i = np.arange(640)
    c = np.stack([((i % 200) + 0.5) * 0.32, ((i // 200) + 0.5) * 0.32], 1)
    f = np.random.default_rng(0).normal(size=(640, 16))
    ctx32.load_params(cfg, F.init_backbone_params(cfg, 5))
    r = ctx32.run_backbone(F.PillarSet(c, f), cfg)
    assert (r.stats.cache.computed, r.stats.cache.hits) == (4, 4) and len(r.kept_indices) == 640
    cfg1 = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=1)
    ctx32.load_params(cfg1, F.init_backbone_params(cfg1, 5))
    r = ctx32.run_backbone(F.PillarSet(c, f), cfg1)
    assert (r.stats.cache.computed, r.stats.cache.hits) == (1, 0)
    cfg2 = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=69, n_blocks=8)
    i = np.arange(30000)
    c2 = np.stack([((i % 200) + 0.5) * 0.32, ((i // 200) + 0.5) * 0.32], 1)
    f2 = np.random.default_rng(1).normal(size=(30000, 16))
    blob = F.init_backbone_params(cfg2, 13)
    ctx32.load_params(cfg2, blob)
    r = ctx32.run_backbone(F.PillarSet(c2, f2), cfg2)
    assert r.stats.dropped_per_block == [54, 0, 0, 0, 0, 0, 0, 0]
    assert (r.stats.cache.computed, r.stats.cache.hits) == (5, 3)
    w = O.port_run_backbone(c2, f2.astype(np.float32), O.make_cfg(d_model=16, n_heads=4, d_ff=32,
                                                                  group_size=69), blob)
    assert np.array_equal(r.kept_indices, w["kept"]) and np.array_equal(r.dropped_indices[0], w["dropped"])
    assert O.max_rel_err(r.features, w["features"]) <= TOL_FP32


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_zero_weights_identity_bit_exact(prec, ctx32, ctx16):
    """test_backbone.cpp:69-86: gather -> zero block -> scatter moves the f32 bits unchanged."""
    ctx = ctx32 if prec == "fp32" else ctx16
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig(n_blocks=4)
    rec_len = 16 + 4 * 132480
    zero = (b"FWAP" + np.array([128, 8, 256], np.uint32).tobytes() + bytes(rec_len - 16)) * 4
    ctx.load_params(cfg, zero)
    r = ctx.run_backbone(ps, cfg)
    assert np.array_equal(r.features, ps.features.astype(np.float32)[r.kept_indices])


def test_determinism(ctx16):
    """acceptance.cpp:467-476: bitwise determinism (no FP atomics on the feature path)."""
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig(n_blocks=2)
    blob = F.init_backbone_params(cfg, 7)
    ctx16.load_params(cfg, blob)
    a = ctx16.run_backbone(ps, cfg)
    b = ctx16.run_backbone(ps, cfg)
    assert np.array_equal(a.features, b.features) and np.array_equal(a.kept_indices, b.kept_indices)
    w = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), O.make_cfg(n_blocks=2), blob)
    assert np.array_equal(a.kept_indices, w["kept"])
    assert O.max_rel_err(a.features, w["features"]) <= TOL_BF16


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_batch_equals_per_frame(prec, ctx32, ctx16):
    """Frame-parallel batch (config 3 machinery): bitwise equal to per-frame runs."""
    ctx = ctx32 if prec == "fp32" else ctx16
    cfg = F.FwaConfig(n_blocks=3)
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    frames = [F.make_pillars(F.SCENES["F10"], s) for s in (42, 43, 44)]
    off = np.cumsum([0] + [p.size() for p in frames])
    res = ctx.run_batch(np.concatenate([p.coords for p in frames]),
                        np.concatenate([p.features for p in frames]), off, cfg)
    ko = np.concatenate([[0], np.cumsum(res["kept_per_frame"])])
    for i, p in enumerate(frames):
        r = ctx.run_backbone(p, cfg)
        assert np.array_equal(res["kept"][ko[i]:ko[i + 1]] - off[i], r.kept_indices)
        assert np.array_equal(res["features"][ko[i]:ko[i + 1]], r.features)


def test_batch_many_drops_sorting_network(ctx16):
    """A batch whose block-0 drops exceed one CTA's rank sort (> 1024: the drop tables take
    the bitonic network): still bitwise equal to per-frame runs, dropped ids included."""
    cfg = F.FwaConfig(n_blocks=2)
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    frames = [F.make_pillars(F.SCENES["F10"], s) for s in range(100, 148)]
    assert sum(p.size() % cfg.group_size for p in frames) > 1024
    off = np.cumsum([0] + [p.size() for p in frames])
    res = ctx16.run_batch(np.concatenate([p.coords for p in frames]),
                          np.concatenate([p.features for p in frames]), off, cfg)
    ko = np.concatenate([[0], np.cumsum(res["kept_per_frame"])])
    for i, p in enumerate(frames):
        r = ctx16.run_backbone(p, cfg)
        assert np.array_equal(res["kept"][ko[i]:ko[i + 1]] - off[i], r.kept_indices)
        assert np.array_equal(res["features"][ko[i]:ko[i + 1]], r.features)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_frame_stream_equals_per_frame(prec, ctx32, ctx16):
    """Pipelined frame stream (fwa_b200_backbone_forward_frames): every frame bitwise
    equal to its own run_backbone -- growing and shrinking frame sizes (workspace moves),
    f64 features, a wide frame that overflows the sync-free bin histogram (re-run alone)."""
    ctx = ctx32 if prec == "fp32" else ctx16
    cfg = F.FwaConfig(n_blocks=4)
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    frames = [F.make_pillars(F.SCENES[s], seed) for s, seed in
              (("F10", 1), ("F30", 2), ("F10", 3), ("PINNED", 4), ("F30", 5))]
    rng = np.random.default_rng(9)
    frames.insert(2, F.PillarSet(rng.uniform(-5000, 5000, size=(3000, 2)), rng.normal(size=(3000, 128))))
    outs = ctx.run_frames(frames, cfg)
    assert len(outs) == len(frames)
    for ps, o in zip(frames, outs):
        r = ctx.run_backbone(ps, cfg)
        assert np.array_equal(o.kept_indices, r.kept_indices)
        assert np.array_equal(o.features, r.features)
        assert [d.tolist() for d in o.dropped_indices] == [d.tolist() for d in r.dropped_indices]
        assert (o.stats.cache.computed, o.stats.cache.hits) == (r.stats.cache.computed, r.stats.cache.hits)
        assert o.stats.dropped_per_block == r.stats.dropped_per_block
    # f32 features (feats_is_f64 = 0) through the same stream
    f32 = [F.PillarSet(p.coords, p.features.astype(np.float32)) for p in frames[:3]]
    for ps, o in zip(f32, ctx.run_frames(f32, cfg)):
        r = ctx.run_backbone(ps, cfg)
        assert np.array_equal(o.kept_indices, r.kept_indices) and np.array_equal(o.features, r.features)
    small = F.PillarSet(np.zeros((5, 2)), np.zeros((5, 128)))
    with pytest.raises(F.NumericError):  # backbone.hpp:218-222, raised before any frame runs
        ctx.run_frames([frames[0], small], cfg)
    bad = F.PillarSet(frames[0].coords, frames[0].features.copy())
    bad.features[7, 3] = np.inf
    with pytest.raises(F.NumericError):  # kernels.hpp:460-461
        ctx.run_frames([frames[1], bad], cfg)


@pytest.mark.parametrize("prec", ["bf16", "bf16_3k"])
def test_repeated_calls_bitwise_stable(prec):
    """Repeated host-API and frame-stream calls on one context (workspaces reused, a
    bin-overflow frame in the mix) reproduce the first results bit for bit -- a guard
    against cross-stream / cross-launch races (it caught one: programmatic dependent
    launch on the schedule kernels)."""
    ctx = F.Context(0, precision=prec)
    cfg = F.FwaConfig(n_blocks=4)
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    frames = [F.make_pillars(F.SCENES[s], seed) for s, seed in (("F10", 1), ("F30", 2), ("PINNED", 4), ("F30", 5))]
    rng = np.random.default_rng(9)
    frames.insert(2, F.PillarSet(rng.uniform(-5000, 5000, size=(3000, 2)), rng.normal(size=(3000, 128))))
    ref = [ctx.run_backbone(ps, cfg) for ps in frames]
    for _ in range(3):
        for ps, r0 in zip(frames, ref):
            r = ctx.run_backbone(ps, cfg)
            assert np.array_equal(r.kept_indices, r0.kept_indices) and np.array_equal(r.features, r0.features)
        for o, r0 in zip(ctx.run_frames(frames, cfg), ref):
            assert np.array_equal(o.kept_indices, r0.kept_indices) and np.array_equal(o.features, r0.features)


def test_device_graph_cache_double_buffered(ctx16):
    """The device-resident forward with two alternating output buffers (a double-buffered
    frame stream): both keys are captured as graphs and replayed; a third buffer set runs
    eagerly; every output is bitwise equal to the first eager result."""
    import torch
    cfg = F.FwaConfig(n_blocks=4)
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    ps = F.make_pillars(F.SCENES["F10"], 7)
    n = ps.size()
    dev = torch.device("cuda", 0)
    dc = torch.from_numpy(ps.coords).to(dev)
    df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
    outs = [torch.zeros((n, cfg.d_model), dtype=torch.float32, device=dev) for _ in range(3)]
    ref = None
    for i in range(9):
        o = outs[2] if i == 7 else outs[i % 2]
        o.zero_()
        nk = ctx16.forward_device(dc.data_ptr(), df.data_ptr(), [0, n], cfg, o.data_ptr())
        ctx16.sync_check()
        got = o[:nk].cpu().numpy()
        if ref is None:
            ref = got
        assert np.array_equal(got, ref), i


def test_errors_mirror_reference(ctx32):
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=8, n_blocks=2)
    blob = F.init_backbone_params(cfg, 1)
    ctx32.load_params(cfg, blob)
    c = np.random.default_rng(0).uniform(0, 5, size=(5, 2))
    with pytest.raises(F.NumericError):          # backbone.hpp:218-222 (N < G)
        ctx32.run_backbone(F.PillarSet(c, np.zeros((5, 16))), cfg)
    c = np.random.default_rng(0).uniform(0, 5, size=(40, 2))
    f = np.zeros((40, 16))
    f[3, 2] = np.nan
    with pytest.raises(F.NumericError):          # kernels.hpp:460-461
        ctx32.run_backbone(F.PillarSet(c, f), cfg)
    with pytest.raises(F.ParseError):            # kernels.hpp:179-180
        ctx32.load_params(cfg, b"XXXX" + blob[4:])
    with pytest.raises(F.ParseError):            # truncated tensor
        ctx32.load_params(cfg, blob[:-8])
    with pytest.raises(F.ConfigError):           # backbone.hpp:164-169
        ctx32.load_params(F.FwaConfig(d_model=16, n_heads=4, d_ff=32, n_blocks=3), blob)
    with pytest.raises(F.ConfigError):
        ctx32.load_params(F.FwaConfig(d_model=16, n_heads=2, d_ff=32, n_blocks=2), blob)
    with pytest.raises(F.ConfigError):
        F.sort(c, F.WindowSpec(0.0, 1.0))


def test_full_size_f60_properties(ctx16):
    """BASELINE config 2 sizes (F60, 8 blocks): integer schedule bit-exact vs the
    NumPy oracle's plans restricted to the kept set; zero-weight identity at full size."""
    ps = F.make_pillars(F.SCENES["F60"], 42)
    cfg = F.FwaConfig()
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    r = ctx16.run_backbone(ps, cfg, want_block_perms=True)
    w = 9 * 0.32
    p0 = O.np_sort(ps.coords, w, w, 0, 0)
    n = ps.size()
    nk = (n // 69) * 69
    assert np.array_equal(np.sort(p0[nk:]), np.sort(r.dropped_indices[0]))
    assert np.array_equal(r.dropped_indices[0], p0[nk:])
    kept = np.sort(p0[:nk])
    assert np.array_equal(r.kept_indices, kept)
    assert (r.stats.cache.computed, r.stats.cache.hits) == (5, 3)
    for b in range(8):
        ay, sh = (b % 4) >= 2, b % 2
        full = O.np_sort(ps.coords, w, w, sh, ay)
        if b == 0:
            want = full
        else:  # reference re-sorts the compacted coords: local indices into the kept list
            want = O.np_sort(ps.coords[kept], w, w, sh, ay)
            # restriction identity
            rank = np.full(n, -1)
            rank[kept] = np.arange(nk)
            restricted = rank[full[np.isin(full, kept)]]
            assert np.array_equal(restricted, want)
        assert np.array_equal(r.block_perms[b], want), b
    assert np.all(np.isfinite(r.features)) and r.features.shape == (nk, 128)


def test_sparse_wide_scene_bin_overflow_fallback(ctx32):
    """A frame whose dense window range (~12M windows) exceeds the sync-free histogram
    capacity: the host API detects the overflow flag and re-runs with exact bins."""
    rng = np.random.default_rng(77)
    c = rng.uniform(-5000, 5000, size=(3000, 2))
    f = rng.normal(size=(3000, 16))
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=4)
    blob = F.init_backbone_params(cfg, 3)
    ctx32.load_params(cfg, blob)
    r = ctx32.run_backbone(F.PillarSet(c, f), cfg, want_block_perms=True)
    w = O.port_run_backbone(c, f.astype(np.float32), O.make_cfg(d_model=16, n_heads=4, d_ff=32,
                                                                group_size=16, n_blocks=4), blob,
                            want_perms=True)
    assert np.array_equal(r.kept_indices, w["kept"])
    for b in range(4):
        assert np.array_equal(r.block_perms[b], w["block_perms"][b, :len(r.block_perms[b])])
    assert O.max_rel_err(r.features, w["features"]) <= TOL_FP32


def test_device_api_graph_replay_matches_host_api(ctx16):
    """Device-resident forward: eager on first sighting, captured into a CUDA graph on
    the second, replayed after -- bitwise equal to the host-buffer API every time."""
    import torch
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig()
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    want = ctx16.run_backbone(F.PillarSet(ps.coords, ps.features.astype(np.float32)), cfg)
    dev = torch.device("cuda", 0)
    dc = torch.from_numpy(ps.coords).to(dev)
    df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
    out = torch.empty((ps.size(), 128), dtype=torch.float32, device=dev)
    kept = torch.empty(ps.size(), dtype=torch.int32, device=dev)
    for i in range(4):
        out.zero_()
        torch.cuda.synchronize()
        nk = ctx16.forward_device(dc.data_ptr(), df.data_ptr(), [0, ps.size()], cfg, out.data_ptr(),
                                  kept.data_ptr())
        ctx16.sync_check()
        assert nk == len(want.kept_indices)
        assert np.array_equal(kept[:nk].cpu().numpy(), want.kept_indices), i
        assert np.array_equal(out[:nk].cpu().numpy(), want.features), i


# ----------------------------------------------------------------------------- fused block kernel

def test_fused_block_kernel_matches_three_kernel_pipeline():
    """The one-launch CTA-pair block kernel (default bf16 path) and the three-kernel bf16
    pipeline (FWA_PREC_BF16_3K) compute the same block with the same bf16 numerics."""
    ps = F.make_pillars(F.SCENES["F10"], 43)
    cfg = F.FwaConfig(n_blocks=4)
    blob = F.init_backbone_params(cfg, 11)
    outs = {}
    for prec in ("bf16", "bf16_3k"):
        ctx = F.Context(0, precision=prec)
        ctx.load_params(cfg, blob)
        outs[prec] = ctx.run_backbone(ps, cfg)
    a, b = outs["bf16"], outs["bf16_3k"]
    assert np.array_equal(a.kept_indices, b.kept_indices)
    assert O.max_rel_err(a.features, b.features) <= 2e-3
    w = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), O.make_cfg(n_blocks=4), blob)
    assert O.max_rel_err(a.features, w["features"]) <= TOL_BF16


@pytest.mark.parametrize("n", [69, 70, 137, 138, 207, 208, 276, 415, 1000])
def test_fused_block_kernel_partial_units(ctx16, n):
    """Frames whose kept rows end inside a CTA pair's unit (1..3 groups of 69, rank 1 empty
    or partly filled, the straddling group present or not): ints exact, features in tol."""
    rng = np.random.default_rng(n)
    c = rng.uniform(-8.0, 8.0, size=(n, 2)).round(2)
    f = rng.normal(size=(n, 128))
    cfg = F.FwaConfig(n_blocks=2)
    blob = F.init_backbone_params(cfg, 5)
    ctx16.load_params(cfg, blob)
    r = ctx16.run_backbone(F.PillarSet(c, f), cfg)
    w = O.port_run_backbone(c, f.astype(np.float32), O.make_cfg(n_blocks=2), blob)
    _check_ints(r, w["kept"], w["dropped"], w["dropped_per_block"], w["cache"])
    assert O.max_rel_err(r.features, w["features"]) <= TOL_BF16


@pytest.mark.parametrize("G", [16, 32, 33, 48, 96, 100, 128])  # + BASELINE config 5's G sweep (32..128)
def test_fused_block_kernel_group_sizes_backbone(ctx16, G):
    """Full backbone through the fused kernel at non-default group sizes (other unit
    geometries and row splits)."""
    ps = F.make_pillars(F.SCENES["F10"], 44)
    cfg = F.FwaConfig(group_size=G, n_blocks=2)
    blob = F.init_backbone_params(cfg, 6)
    ctx16.load_params(cfg, blob)
    r = ctx16.run_backbone(ps, cfg)
    w = O.port_run_backbone(ps.coords, ps.features.astype(np.float32), O.make_cfg(group_size=G, n_blocks=2), blob)
    _check_ints(r, w["kept"], w["dropped"], w["dropped_per_block"], w["cache"])
    assert O.max_rel_err(r.features, w["features"]) <= TOL_BF16


def test_fused_block_kernel_nonfinite_input_raises(ctx16):
    """kernels.hpp:460-461 through the fused kernel's gather (numeric_error)."""
    cfg = F.FwaConfig(n_blocks=1)
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 1))
    rng = np.random.default_rng(3)
    c = rng.uniform(0, 10, size=(300, 2))
    f = rng.normal(size=(300, 128))
    f[17, 5] = np.inf
    with pytest.raises(F.NumericError):
        ctx16.run_backbone(F.PillarSet(c, f), cfg)


# ----------------------------------------------------------------------------- pillarization (§8f next-1)

@pytest.mark.parametrize("name", ["F10", "PINNED", "F60"])
def test_gpu_pillarize_matches_reference_pillars(ctx16, name):
    """geometry::pillarize on the GPU vs the reference's generate_synthetic + pillarize
    (host port pinned bit-exact to it): cell order and coordinates bit-exact; features
    equal up to CUDA's erf vs libm's (<= a few ulp)."""
    scene = F.SCENES[name]
    xy, f = F.generate_points(scene, 42)
    w = F.pillar_params(scene.f_in, 128, 42)
    got = ctx16.pillarize(xy, f, 0.32, w)
    want = F.make_pillars(scene, 42)
    assert np.array_equal(got.coords, want.coords)
    np.testing.assert_allclose(got.features, want.features, rtol=1e-14, atol=1e-15)  # CUDA vs libm erf


def test_gpu_pillarize_edge_cases_vs_oracle(ctx16):
    """Cell-boundary coordinates, negative cells, crowded cells (pairwise recursion past
    8 and 32 members), non-zero bias, f_in = 3, and an empty cloud."""
    rng = np.random.default_rng(5)
    res = 0.32
    grid = np.stack(np.meshgrid(np.arange(-6, 7) * res, np.arange(-5, 6) * res), -1).reshape(-1, 2)
    crowd = np.full((70, 2), [1.01, -2.17]) + rng.uniform(0, 0.05, size=(70, 2))
    rand = rng.uniform(-4, 4, size=(400, 2))
    xy = np.concatenate([grid, crowd, rand, grid[::7]])
    f = rng.normal(size=(xy.shape[0], 3))
    w = rng.normal(size=(24, 3))
    b = rng.normal(size=24)
    got = ctx16.pillarize(xy, f, res, w, b)
    wc, wf = O.np_pillarize(xy, f, res, w, b)
    assert np.array_equal(got.coords, wc)
    np.testing.assert_allclose(got.features, wf, rtol=1e-14, atol=1e-15)
    empty = ctx16.pillarize(np.zeros((0, 2)), np.zeros((0, 3)), res, w, b)
    assert empty.size() == 0


def test_gpu_pillarize_feeds_backbone(ctx16):
    """points -> GPU pillarize -> backbone == host pillars -> backbone (ints exact)."""
    scene = F.SCENES["F10"]
    xy, f = F.generate_points(scene, 42)
    ps = ctx16.pillarize(xy, f, 0.32, F.pillar_params(scene.f_in, 128, 42))
    cfg = F.FwaConfig(n_blocks=2)
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    a = ctx16.run_backbone(ps, cfg)
    b = ctx16.run_backbone(F.make_pillars(scene, 42), cfg)
    assert np.array_equal(a.kept_indices, b.kept_indices)
    assert O.max_rel_err(a.features, b.features) <= 1e-3


# ----------------------------------------------------------------------------- `fwa attend` (§8f next-2)

def test_fwa_bench_cli_modes(tmp_path):
    """`fwa bench` (tools/fwa_bench.py, fwa_cli.cpp:249-281) in all three modes on a small
    FWPC file: the reference's BenchResult document, its config digest, exit code 2 for an
    unknown mode."""
    import subprocess
    import sys
    from paper_2301_08739_b200.attend import config_digest
    if not O.have_ref():
        pytest.skip("reference oracle not built (point-file writer)")
    scene = {"n_clusters": 6, "ppc_min": 150, "ppc_max": 300, "sigma": 1.5, "ext_x": 40.0, "ext_y": 40.0,
             "n_bg": 500, "f_in": 2}
    path = str(tmp_path / "pts.fwpc")
    O.ref_write_points(scene, 5, path, True)
    tool = os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "fwa_bench.py")
    for mode in ("group", "global", "equal-window"):
        r = subprocess.run([sys.executable, tool, path, "--mode", mode, "--runs", "4", "--warmup", "1"],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        j = json.loads(r.stdout)
        assert j["name"] == mode and j["runs"] == 4 and j["warmup"] == 1 and j["n_points"] > 0
        assert j["config_digest"] == config_digest(F.FwaConfig())
        w = j["wall_time_ms"]
        assert 0 < w["p50"] <= w["p95"] and w["mean"] > 0
        if mode == "group":
            assert j["stage_ms"].get("block_fused", 0) > 0 and j["stage_ms"].get("schedule", 0) > 0
    r = subprocess.run([sys.executable, tool, path, "--mode", "nope"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 2


def test_attend_json_matches_reference(tmp_path, ctx16):
    """`fwa attend` on the B200 path (points -> GPU pillarize -> GPU backbone -> GPU row
    checksums) vs the reference library on the same FWPC file: every integer / structural
    field exact, row checksums within the bf16 feature tolerance, and the checksums bit-exact
    sums of the FWFB-dumped features (fwa_cli.cpp:214-218)."""
    from paper_2301_08739_b200.attend import attend, config_digest
    if not O.have_ref():
        pytest.skip("reference oracle not built")
    scene = {"n_clusters": 12, "ppc_min": 150, "ppc_max": 300, "sigma": 1.5, "ext_x": 60.0, "ext_y": 60.0,
             "n_bg": 2000, "f_in": 2}
    path = str(tmp_path / "pts.fwpc")
    O.ref_write_points(scene, 11, path, True)
    cfg = F.FwaConfig(n_blocks=4)
    fwfb = str(tmp_path / "feat.fwfb")
    j = attend(ctx16, path, cfg, None, 11, fwfb)
    # the reference: generate -> pillarize -> init_backbone_params(seed) -> run_backbone
    rc = O.make_cfg(n_blocks=4)
    coords, feats64 = O.ref_make_pillars(scene, 11, d_out=128, param_seed=11)
    blob = O.ref_init_params(rc, 128, 11)
    w = O.ref_run_backbone(coords, feats64, rc, blob)
    assert j["n_input"] == coords.shape[0] and j["n_kept"] == len(w["kept"])
    assert (j["cache"]["computed"], j["cache"]["hits"]) == tuple(w["cache"])
    assert j["dropped_per_block"] == list(w["dropped_per_block"])
    assert j["config_digest"] == config_digest(cfg)
    assert np.array_equal(np.array(j["coords"]), coords[w["kept"]])
    want_sums = np.cumsum(w["features"].astype(np.float64), axis=1)[:, -1]
    got_sums = np.array(j["row_checksums"])
    assert np.max(np.abs(got_sums - want_sums)) <= TOL_BF16 * np.max(np.abs(want_sums))
    raw = open(fwfb, "rb").read()
    assert raw[:4] == b"FWFB"
    n, d = np.frombuffer(raw[4:12], np.uint32)
    f = np.frombuffer(raw[12:], np.float32).reshape(n, d)
    assert np.array_equal(np.cumsum(f.astype(np.float64), axis=1)[:, -1], got_sums)
    assert j["feature_hash"] == F.fnv1a64_hex(f.tobytes())


# ----------------------------------------------------------------------------- equal-window baseline (§8f next-3)

def test_equal_window_baseline_vs_oracle(ctx16):
    """The SST-style padded baseline (bench.hpp:266-326) on the GPU == the reference block
    run on the same padded windows (oracle), and its WorkloadReport statistics."""
    import torch
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig(n_blocks=1)
    blob = F.init_backbone_params(cfg, 3)
    ctx16.load_params(cfg, blob)
    n = ps.size()
    f32 = ps.features.astype(np.float32)
    d_c = torch.from_numpy(ps.coords).cuda()
    d_f = torch.from_numpy(f32).cuda()
    d_o = torch.empty_like(d_f)
    torch.cuda.synchronize()
    rep = ctx16.equal_window_forward(d_c.data_ptr(), d_f.data_ptr(), n, cfg, d_o.data_ptr())
    got = d_o.cpu().numpy()
    w = 9 * 0.32
    want = O.np_equal_window_forward(ps.coords, f32, blob[:16 + 4 * 132480], w, w)
    assert O.max_rel_err(got, want) <= TOL_BF16
    wm, wn, _, _ = O.np_sort_keys(ps.coords, w, w, 0, 0)
    _, counts = np.unique(np.stack([wm, wn], 1), axis=0, return_counts=True)
    assert rep["n_windows"] == counts.size
    assert rep["max_occ"] == counts.max() and rep["min_nonzero_occ"] == counts.min()
    assert rep["rows_padded"] >= n and rep["padding_factor"] >= 1.0


# ----------------------------------------------------------------------------- block backward (§8f next-4)

def _fwap_tensors(blob, d, dff):
    v = np.frombuffer(blob[16:], np.float32)
    sizes = [3 * d * d, 3 * d, d * d, d, d, d, d, d, dff * d, dff, d * dff, d]
    out, o = [], 0
    for n in sizes:
        out.append(v[o:o + n])
        o += n
    return out


@pytest.mark.parametrize("d,h,dff,G,ng", [(32, 4, 64, 8, 4), (128, 8, 256, 69, 3), (16, 2, 32, 1, 5), (64, 4, 96, 33, 2)])
def test_block_backward_vs_reference(ctx32, d, h, dff, G, ng):
    """fwa_block_backward (kernels.hpp:660-765) on the GPU vs the compiled reference: the
    input gradient and all twelve parameter gradients (normwise rel err <= 1e-4, fp32)."""
    if not O.have_ref():
        pytest.skip("reference oracle not built")
    cfg = F.FwaConfig(d_model=d, n_heads=h, d_ff=dff, group_size=G, n_blocks=1)
    rec = F.init_backbone_params(cfg, d + G)
    # non-trivial norms / biases so every gradient path is exercised
    v = np.frombuffer(rec[16:], np.float32).copy()
    v += 0.05 * np.random.default_rng(G).normal(size=v.shape).astype(np.float32)
    rec = rec[:16] + v.tobytes()
    rng = np.random.default_rng(d * 7 + G)
    rows = ng * G
    f = rng.normal(size=(rows, d)).astype(np.float32)
    pe = (0.3 * rng.normal(size=(rows, d))).astype(np.float32)
    go = rng.normal(size=(rows, d)).astype(np.float32)
    gf, gr = ctx32.fwa_block_backward(f, pe, rec, ng, go)
    wf, wr = O.ref_block_backward(f, pe, ng, rec, go)
    assert O.max_rel_err(gf, wf) <= 1e-4
    assert gr[:16] == wr[:16]
    for i, (a, b) in enumerate(zip(_fwap_tensors(gr, d, dff), _fwap_tensors(wr, d, dff))):
        assert O.max_rel_err(a, b) <= 1e-4, i


def test_batch_frames_far_apart_per_frame_bins(ctx32):
    """Frames in world coordinates kilometres apart (a batch whose union window range
    would need ~10^9 dense bins): each frame gets its own window range (exact path), the
    outputs equal the per-frame runs bit for bit (per-frame bins)."""
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=4)
    ctx32.load_params(cfg, F.init_backbone_params(cfg, 2))
    rng = np.random.default_rng(9)
    frames = []
    for k in range(3):
        c = np.unique(np.round(rng.uniform(-15, 15, size=(400, 2)) / 0.32) * 0.32 + 0.16, axis=0)
        c = c + np.array([[k * 40000.0, -k * 25000.0]])
        frames.append(F.PillarSet(c, rng.normal(size=(c.shape[0], 16))))
    off = np.cumsum([0] + [p.size() for p in frames])
    res = ctx32.run_batch(np.concatenate([p.coords for p in frames]),
                          np.concatenate([p.features for p in frames]), off, cfg)
    ko = np.concatenate([[0], np.cumsum(res["kept_per_frame"])])
    for i, p in enumerate(frames):
        r = ctx32.run_backbone(p, cfg)
        assert np.array_equal(res["kept"][ko[i]:ko[i + 1]] - off[i], r.kept_indices)
        assert np.array_equal(res["features"][ko[i]:ko[i + 1]], r.features)


def test_device_batch_far_apart_no_bin_overflow(ctx16):
    """The device-resident (sync-free) forward of a batch whose frames lie kilometres apart:
    per-frame window bins on the device, so no capacity overflow is raised (round 1 and the
    union layout needed ~10^9 bins there) and the rows equal the host-API batch bit for bit."""
    import torch
    cfg = F.FwaConfig(n_blocks=2)
    ctx16.load_params(cfg, F.init_backbone_params(cfg, 42))
    frames = []
    for k in range(3):
        p = F.make_pillars(F.SCENES["F10"], 60 + k)
        frames.append(F.PillarSet(p.coords + np.array([[k * 40000.0, -k * 25000.0]]), p.features))
    off = np.cumsum([0] + [p.size() for p in frames])
    coords = np.concatenate([p.coords for p in frames])
    feats = np.concatenate([p.features for p in frames]).astype(np.float32)
    dev = torch.device("cuda", 0)
    dc, df = torch.from_numpy(coords).to(dev), torch.from_numpy(feats).to(dev)
    dout = torch.empty((coords.shape[0], cfg.d_model), dtype=torch.float32, device=dev)
    dkept = torch.empty(coords.shape[0], dtype=torch.int32, device=dev)
    nk = ctx16.forward_device(dc.data_ptr(), df.data_ptr(), off.tolist(), cfg, dout.data_ptr(), dkept.data_ptr())
    ctx16.sync_check()  # raised FWA_ERR_INTERNAL (bin capacity) with the union layout
    res = ctx16.run_batch(coords, feats, off, cfg)
    assert nk == len(res["kept"])
    assert np.array_equal(dkept[:nk].cpu().numpy(), res["kept"])
    assert np.array_equal(dout[:nk].cpu().numpy(), res["features"][:nk])


def test_far_outlier_window_rank_fallback(ctx32):
    """One pillar 10^8 m away: no dense window layout fits (the round-1 code raised
    FWA_ERR_INTERNAL); the exact path rank-compresses the windows with a radix sort and the
    result equals the oracle bit for bit in every integer output."""
    rng = np.random.default_rng(10)
    c = np.unique(np.round(rng.uniform(-20, 20, size=(600, 2)) / 0.32) * 0.32 + 0.16, axis=0)
    c = np.concatenate([c, [[1.0e8 + 0.16, -3.0e7 + 0.48]]])
    f = rng.normal(size=(c.shape[0], 16))
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=4)
    blob = F.init_backbone_params(cfg, 3)
    ctx32.load_params(cfg, blob)
    r = ctx32.run_backbone(F.PillarSet(c, f), cfg, want_block_perms=True)
    w = O.port_run_backbone(c, f.astype(np.float32), O.make_cfg(d_model=16, n_heads=4, d_ff=32,
                                                                group_size=16, n_blocks=4), blob,
                            want_perms=True)
    assert np.array_equal(r.kept_indices, w["kept"])
    assert np.array_equal(np.concatenate(r.dropped_indices), w["dropped"])
    for b in range(4):
        assert np.array_equal(r.block_perms[b], w["block_perms"][b, :len(r.block_perms[b])])
    assert O.max_rel_err(r.features, w["features"]) <= TOL_FP32
    for spec in [F.WindowSpec(2.88, 2.88, sh, ax) for sh in (False, True) for ax in ("X", "Y")]:
        assert np.array_equal(ctx32.sort(c, spec), O.np_sort(c, 2.88, 2.88, int(spec.shift), int(spec.major_axis == "Y")))
