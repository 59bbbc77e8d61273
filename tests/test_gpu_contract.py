"""GPU: the rest of the drop-in contract of run_backbone (backbone.hpp:159-325).

  * BackboneParams::input_proj (backbone.hpp:74-81, 179-190) on the device: the seed
    initialiser's projection (drawn first, N(0, 0.1^2)) is bit-identical to the
    reference's, the projected rows are bit-exact (fp32 check mode with zero block weights
    is the identity, so the output IS the projection), and the full backbone matches the
    reference's seed overload within the bars;
  * RunStats.stages (backbone.hpp:109-126) through the C ABI: every stage timed, the sum
    close to the call's device time;
  * per-frame cache statistics of a batch whose frames have N mod G == 0 (reference 4/4)
    and != 0 (5/3)."""
import numpy as np
import pytest

import oracle as O
import paper_2301_08739_b200 as F

pytestmark = pytest.mark.gpu


def _scene(n_in, seed=5):
    cloud_spec = F.SceneSpec(6, 200, 300, 2.0, 60.0, 60.0, 500, 2)
    ps = F.make_pillars(cloud_spec, seed, d_out=n_in)
    return ps


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 1e-2)])
def test_input_projection_matches_reference_seed_overload(prec, tol):
    ps = _scene(16)
    cfg = F.FwaConfig(n_blocks=2)
    want = O.ref_run_backbone_seeded(ps.coords, ps.features, O.make_cfg(n_blocks=2), 9, n_threads=8)
    blob, w = F.init_backbone_params_fin(cfg, 16, 9)
    assert w is not None and np.array_equal(w, want["proj_weight"])
    assert blob == O.ref_init_params(O.make_cfg(n_blocks=2), 16, 9)
    r = F.run_backbone(ps, cfg, 9, precision=prec)  # the seed overload, projection included
    assert np.array_equal(r.kept_indices, want["kept"])
    assert np.array_equal(np.concatenate(r.dropped_indices), want["dropped"])
    assert (r.stats.cache.computed, r.stats.cache.hits) == want["cache"]
    err = O.max_rel_err(r.features, want["features"])
    assert err <= tol, err


def test_input_projection_rows_bit_exact():
    """Zero block weights (kernels::zero_attn_params: every block is the identity in the
    fp32 check mode) -> the backbone output IS the projected input, which must equal the
    reference's fp32 loop bit for bit (acc = b; acc += w*x in order)."""
    ps = _scene(16, seed=3)
    cfg = F.FwaConfig(n_blocks=1)
    rng = np.random.default_rng(0)
    w = rng.normal(0, 0.1, size=(128, 16)).astype(np.float32)
    b = rng.normal(0, 0.1, size=128).astype(np.float32)
    x = ps.features.astype(np.float32)  # static_cast<float>(pillars.features(r, c))
    want = np.tile(b, (x.shape[0], 1)).astype(np.float32)
    for c in range(16):  # the reference's order: acc = bias; acc += w[c] * x[c], fp32 each step
        want = (want + (w[:, c][None, :] * x[:, c][:, None]).astype(np.float32)).astype(np.float32)
    zero = O.ref_zero_params(O.make_cfg(n_blocks=1)) if O.have_ref() else None
    if zero is None:
        pytest.skip("oracle/_ref not built")
    ctx = F.Context(0, precision="fp32")
    ctx.load_params(cfg, zero)
    ctx.load_input_proj(w, b)
    r = ctx.run_backbone(ps, cfg)
    assert np.array_equal(r.features, want[r.kept_indices])
    with pytest.raises(F.ShapeError):  # width != the projection's
        ctx.run_backbone(F.PillarSet(ps.coords, np.zeros((ps.size(), 128))), cfg)
    ctx.load_input_proj(None)
    with pytest.raises(F.ShapeError):  # width != d_model without a projection
        ctx.run_backbone(ps, cfg)


def test_stage_times_through_c_abi():
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig()
    for prec in ("bf16", "bf16_3k", "fp32"):
        ctx = F.Context(0, precision=prec)
        ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
        ctx.run_backbone(ps, cfg)
        r = ctx.run_backbone(ps, cfg)
        st = r.stats.stages
        assert st.sort_ms > 0 and st.group_ms > 0 and st.attention_ms > 0 and st.ffn_ms > 0, (prec, st)
        if prec == "bf16":  # the fused kernel's time split by its phase counters
            assert st.gather_ms > 0 and st.scatter_ms > 0, st
        assert st.total() < 100.0, st
        outs = ctx.run_frames([ps, ps], cfg)
        for o in outs:
            assert o.stats.stages.attention_ms > 0 and o.stats.stages.sort_ms > 0


def test_batch_per_frame_cache_stats():
    """backbone.hpp:224-234, 285-316: a frame with N mod G == 0 computes 4 sorts and hits 4
    (8 blocks), one with N mod G != 0 computes 5 and hits 3; a batch reports each frame's."""
    cfg = F.FwaConfig(d_model=16, n_heads=4, d_ff=32, group_size=16, n_blocks=8)
    rng = np.random.default_rng(4)
    frames = []
    for n in (160, 170, 176, 200):  # 160, 176: N mod 16 == 0
        c = (np.arange(n)[:, None] * np.array([[0.32, 0.0]]) + rng.integers(0, 3, size=(n, 1)) * 0.32 + 0.16)
        frames.append(F.PillarSet(c, rng.normal(size=(n, 16))))
    ctx = F.Context(0, precision="fp32")
    ctx.load_params(cfg, F.init_backbone_params(cfg, 1))
    off = np.cumsum([0] + [p.size() for p in frames])
    res = ctx.run_batch(np.concatenate([p.coords for p in frames]),
                        np.concatenate([p.features for p in frames]), off, cfg)
    for p, st in zip(frames, res["frame_stats"]):
        one = ctx.run_backbone(p, cfg)
        assert st["cache"] == (one.stats.cache.computed, one.stats.cache.hits)
        assert st["n_dropped"] == p.size() % 16 and st["n_kept"] == len(one.kept_indices)
        assert st["cache"] == ((4, 4) if p.size() % 16 == 0 else (5, 3))
