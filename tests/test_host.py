"""CPU: the C-ABI library loads, exports every symbol include/fwa_b200.h declares,
and its host-side input generators are bit-identical to the reference's."""
import json
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2301_08739_b200 as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def fnv(b: bytes) -> str:
    return F.fnv1a64_hex(b)


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fwa_b200.h")).read()
    declared = set(re.findall(r"\b(fwa_b200_\w+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = F.lib()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert declared == set(F.EXPORTS)


def test_generated_frames_match_reference_hashes():
    """generate_synthetic + pillarize (geometry.hpp:246-386), pillar counts of SURVEY §8d."""
    gold = json.load(open(os.path.join(GOLD, "scenes.json")))
    for name in ("F10", "PINNED", "F30", "F60"):
        ps = F.make_pillars(F.SCENES[name], 42)
        g = gold[name]
        assert ps.size() == g["n"], name
        assert fnv(np.ascontiguousarray(ps.coords).tobytes()) == g["coords_fnv"], name
        assert fnv(np.ascontiguousarray(ps.features[:512]).tobytes()) == g["feats_fnv"], name
        assert float(ps.features.sum()) == g["feats_sum"], name
    assert gold["PINNED"]["n"] == 21199 and gold["F60"]["n"] == 60897


def test_init_params_match_reference_hash():
    gold = json.load(open(os.path.join(GOLD, "scenes.json")))
    blob = F.init_backbone_params(F.FwaConfig(), 42)
    assert len(blob) == 8 * (16 + 4 * 132480)
    assert fnv(blob) == gold["params_default_seed42_fnv"]


def test_config_validation_mirrors_reference():
    F.validate(F.FwaConfig())
    for bad in (dict(resolution=0.0), dict(window_px=0), dict(group_size=0), dict(n_blocks=0),
                dict(d_model=6), dict(n_heads=3), dict(d_ff=0)):
        with pytest.raises(F.ConfigError):
            F.validate(F.FwaConfig(**bad))
    c = F.FwaConfig.from_json({"window": [7, 5], "group_size": 32})
    assert (c.window_px, c.window_py, c.group_size, c.d_model) == (7, 5, 32, 128)
    assert c.window_x_m() == 7 * 0.32


def test_no_gpu_fails_loudly():
    """Without a CUDA device the product path raises; it never falls back to the CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(F.FwaError):
        F.Context(0)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfwa_ref.so")),
                    reason="oracle/_ref not built")
def test_generator_equals_reference_live():
    import oracle as O
    ps = F.make_pillars(F.SCENES["F10"], 42)
    s = F.SCENES["F10"]
    c, f = O.ref_make_pillars(dict(n_clusters=s.n_clusters, ppc_min=s.points_per_cluster_min,
                                   ppc_max=s.points_per_cluster_max, sigma=s.cluster_sigma,
                                   ext_x=s.extent_x, ext_y=s.extent_y, n_bg=s.n_background,
                                   f_in=s.f_in), 42, 128)
    assert np.array_equal(ps.coords, c) and np.array_equal(ps.features, f)
    cfg = O.make_cfg(n_blocks=3, d_model=64, n_heads=4, d_ff=96)
    assert F.init_backbone_params(F.FwaConfig(n_blocks=3, d_model=64, n_heads=4, d_ff=96), 9) == \
        O.ref_init_params(cfg, 64, 9)


# ----------------------------------------------------------------------------- `fwa attend` output contract

def test_attend_config_digest_and_fnv_match_reference():
    """config_digest = FNV-1a-64 of nlohmann::json(FwaConfig).dump() (fwa_cli.cpp:71-73,
    backbone.hpp:49-57); fnv1a64_hex = bench.hpp:62-72."""
    from paper_2301_08739_b200.attend import config_digest, config_json
    if not O.have_ref():
        pytest.skip("reference oracle not built")
    for kw in ({}, {"resolution": 0.25, "group_size": 32, "n_blocks": 2}, {"d_model": 64, "n_heads": 4, "d_ff": 96},
               {"resolution": 0.1, "window": (7, 11)}):
        win = kw.pop("window", (9, 9))
        cfg = F.FwaConfig(window_px=win[0], window_py=win[1], **kw)
        rc = O.make_cfg(window=win, **kw)
        assert config_json(cfg) == O.ref_config_json(rc)
        assert config_digest(cfg) == O.ref_fnv1a64_hex(O.ref_config_json(rc).encode())
    b = np.random.default_rng(1).integers(0, 256, size=100_000, dtype=np.uint8).tobytes()
    assert F.fnv1a64_hex(b) == O.ref_fnv1a64_hex(b)


@pytest.mark.parametrize("binary", [True, False])
def test_attend_ingest_reads_reference_point_files(tmp_path, binary):
    """ingest (geometry.hpp:125-200) of FWPC / CSV files written by the reference's own
    writers (geometry.hpp:202-237) == the generated cloud."""
    from paper_2301_08739_b200.attend import ingest_points
    if not O.have_ref():
        pytest.skip("reference oracle not built")
    scene = {"n_clusters": 5, "ppc_min": 10, "ppc_max": 30, "sigma": 1.0, "ext_x": 30.0, "ext_y": 20.0,
             "n_bg": 200, "f_in": 3}
    path = str(tmp_path / ("p.fwpc" if binary else "p.csv"))
    O.ref_write_points(scene, 7, path, binary)
    xy, f = ingest_points(path)
    gxy, gf = F.generate_points(F.SceneSpec(5, 10, 30, 1.0, 30.0, 20.0, 200, 3), 7)
    assert np.array_equal(xy, gxy) and np.array_equal(f, gf)


def test_attend_cache_and_drops_match_port():
    """The cache / drop bookkeeping of the attend JSON == the reference rule (port)."""
    from paper_2301_08739_b200.attend import cache_and_drops
    rng = np.random.default_rng(2)
    for n, nb in ((700, 8), (690, 8), (75, 2), (69, 1), (300, 5)):
        c = rng.uniform(0, 20, size=(n, 2))
        blob = F.init_backbone_params(F.FwaConfig(d_model=16, n_heads=4, d_ff=32, n_blocks=nb), 1)
        w = O.port_run_backbone(c, np.zeros((n, 16), np.float32), O.make_cfg(d_model=16, n_heads=4, d_ff=32,
                                                                             n_blocks=nb), blob)
        (comp, hit), drops = cache_and_drops(n, F.FwaConfig(n_blocks=nb))
        assert (comp, hit) == tuple(w["cache"]) and drops == list(w["dropped_per_block"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_bench_protocol_matches_reference():
    """`fwa bench` protocol (bench.hpp:75-143): linear-interpolation percentiles, the 3x IQR
    outlier exclusion and the mean over the kept samples -- bit-identical to the compiled
    reference on random samples with injected outliers."""
    from paper_2301_08739_b200 import benchcli as B
    rng = np.random.default_rng(11)
    for n in (1, 2, 3, 4, 5, 9, 50, 101):
        for trial in range(5):
            s = list(rng.gamma(2.0, 1.0, size=n))
            if n >= 5 and trial % 2:
                s[n // 2] = 1e3
                s[-1] = -5.0
            want = O.ref_bench_summarize(s, n, 3)
            got = B.summarize("group", 10, "0x0", s, n, 3)
            assert (got["wall_time_ms"]["mean"], got["wall_time_ms"]["p50"], got["wall_time_ms"]["p95"],
                    got["outliers_excluded"]) == want
    assert set(B.summarize("g", 1, "d", [1.0], 1, 0)) == {
        "name", "n_points", "config_digest", "wall_time_ms", "outliers_excluded", "runs", "warmup", "stage_ms"}
