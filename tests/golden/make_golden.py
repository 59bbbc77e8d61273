"""Generate the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libfwa_ref.so, built from /root/reference by `make -C oracle ref`).

    python tests/golden/make_golden.py

Fixtures (all small):
  keys.json            Eq. 1 sort keys of the reference unit tests (test_flatten.cpp:26-60)
                       evaluated by flatten::make_sort_key, plus window-boundary cases.
  sort_cases.npz       coords + reference flatten::sort permutations (4 specs) for random,
                       window-boundary, duplicate-point and pillar-grid scenes.
  backbone_small.npz   run_backbone on a D=16/H=4/D_ff=32/G=8 config (drops in block 0).
  backbone_d128.npz    run_backbone on the default config (D=128, H=8, D_ff=256, G=69,
                       8 blocks) for a ~1.4k-pillar clustered frame.
  block_d128.npz       fwa_block_forward (f32) on 3 groups of 69 rows, default dims.
  scenes.json          pillar counts + FNV-1a hashes of generated frames and params.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def fnv(b: bytes) -> str:
    h = 0xcbf29ce484222325
    for c in b:
        h ^= c
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"0x{h:016x}"


def fnv_np(a: np.ndarray) -> str:
    # vectorised FNV is awkward; hash via the bytes in chunks (small arrays only)
    return fnv(np.ascontiguousarray(a).tobytes())


SPECS = [(0, 0), (0, 1), (1, 0), (1, 1)]  # (axis_y, shift) in block_schedule order


def scene_dict(s):
    return dict(n_clusters=s[0], ppc_min=s[1], ppc_max=s[2], sigma=s[3], ext_x=s[4], ext_y=s[5],
                n_bg=s[6], f_in=s[7])


def main():
    if not O.have_ref():
        O.build(ref=True)
    rng = np.random.default_rng(20261017)

    # --- keys
    keys = []
    cases = [((3.5, 1.0), 2.0, 2.0, 0, 0), ((-0.5, 0.0), 2.0, 2.0, 0, 0), ((0.0, 0.0), 2.0, 2.0, 1, 0),
             ((3.5, 9.0), 2.0, 4.0, 0, 1), ((2.88, -2.88), 2.88, 2.88, 0, 0),
             ((1.28, 1.6), 2.88, 2.88, 1, 0), ((-0.16, 4.32), 2.88, 2.88, 1, 1),
             ((0.16 + 0.32 * 4, -0.16), 9 * 0.32, 9 * 0.32, 1, 0)]
    for (x, y), wx, wy, sh, ay in cases:
        k = O.ref_sort_key(x, y, wx, wy, sh, ay)
        keys.append(dict(x=x, y=y, w_x=wx, w_y=wy, shift=sh, axis_y=ay, win_major=k[0],
                         win_minor=k[1], loc_major=k[2].hex(), loc_minor=k[3].hex()))
    with open(os.path.join(HERE, "keys.json"), "w") as f:
        json.dump(keys, f, indent=1)

    # --- sort cases
    out = {}
    w = 9 * 0.32
    sc = []
    for t in range(6):  # random scenes, extent 50 m, 100..3000 points (acceptance.cpp:138-156)
        n = int(rng.integers(100, 3000))
        sc.append((f"rand{t}", rng.uniform(-50, 50, size=(n, 2)), w, w))
    for v in range(4):  # window-boundary + duplicates, w = 2 (acceptance.cpp:157-173)
        pts = []
        for i in range(2000):
            x = 2.0 * (float(rng.integers(0, 9)) - 4.0)
            y = 2.0 * (float(rng.integers(0, 9)) - 4.0)
            pts.append((x, y))
            if v >= 2 and i % 3 == 0:
                pts.append((x, y))
        sc.append((f"bound{v}", np.array(pts), 2.0, 2.0))
    gx, gy = np.meshgrid(np.arange(61), np.arange(47), indexing="ij")  # pillar grid, w = 9 cells
    grid = np.stack([(gx.ravel() - 30 + 0.5) * 0.32, (gy.ravel() - 20 + 0.5) * 0.32], 1)
    sc.append(("grid", grid, w, w))
    sc.append(("ident", np.array([[1.0, 1.0]] * 3), 2.0, 2.0))  # test_flatten.cpp:62-66
    for name, coords, wx, wy in sc:
        out[f"{name}_coords"] = coords
        out[f"{name}_w"] = np.array([wx, wy])
        for ay, sh in SPECS:
            out[f"{name}_perm_{ay}{sh}"] = O.ref_sort(coords, wx, wy, sh, ay)
    out["names"] = np.array([s[0] for s in sc])
    np.savez_compressed(os.path.join(HERE, "sort_cases.npz"), **out)

    # --- backbone small (test_backbone.cpp make_pillars-style fixture, drops in block 0)
    cfg = O.make_cfg(d_model=16, n_heads=4, d_ff=32, group_size=8, n_blocks=4)
    coords, feats = O.ref_make_pillars(scene_dict((12, 40, 40, 1.2, 80.0, 80.0, 30, 2)), 3, d_out=16,
                                       param_seed=4)
    blob = O.ref_init_params(cfg, 16, 5)
    r = O.ref_run_backbone(coords, feats, cfg, blob)
    plans = O.ref_block_plans(coords, cfg)
    np.savez_compressed(os.path.join(HERE, "backbone_small.npz"), coords=coords, feats=feats,
                        blob=np.frombuffer(blob, np.uint8), features=r["features"], kept=r["kept"],
                        dropped=r["dropped"], dropped_per_block=r["dropped_per_block"],
                        cache=np.array(r["cache"]),
                        cfg=np.array([16, 4, 32, 8, 4]),
                        **{f"plan{b}": plans[b] for b in range(4)})

    # --- backbone default dims
    cfg = O.make_cfg()
    # inputs are regenerated in the tests from (scene, seed) and init_backbone_params(seed 42);
    # both generators are pinned separately by scenes.json
    scene = (4, 200, 400, 2.0, 60.0, 60.0, 400, 2)
    coords, feats = O.ref_make_pillars(scene_dict(scene), 7, d_out=128)
    blob = O.ref_init_params(cfg, 128, 42)
    r = O.ref_run_backbone(coords, feats, cfg, blob, n_threads=8)
    plans = O.ref_block_plans(coords, cfg)
    np.savez_compressed(os.path.join(HERE, "backbone_d128.npz"), scene=np.array(scene, np.float64),
                        scene_seed=7, param_seed=42,
                        coords_fnv=fnv_np(coords), features=r["features"], kept=r["kept"],
                        dropped=r["dropped"], dropped_per_block=r["dropped_per_block"],
                        cache=np.array(r["cache"]),
                        **{f"plan{b}": plans[b] for b in range(8)})

    # --- one block, default dims
    rec_len = len(blob) // 8
    rec = blob[:rec_len]
    f = rng.normal(size=(3 * 69, 128)).astype(np.float32)
    pe = (0.3 * rng.normal(size=(3 * 69, 128))).astype(np.float32)
    o32 = O.ref_block_forward(f, pe, 3, rec)
    o64 = O.ref_oracle_block(f.astype(np.float64), pe.astype(np.float64), 3, rec)
    np.savez_compressed(os.path.join(HERE, "block_d128.npz"), f=f, pe=pe, param_seed=42,
                        out32=o32, out64=o64)  # record = block 0 of init_backbone_params(seed 42)

    # --- scene + param hashes
    scenes = {}
    specs = {"F10": (32, 200, 400, 2.0, 150.0, 150.0, 3200, 2),
             "PINNED": (80, 200, 280, 1.3, 200.0, 200.0, 10000, 2),
             "F30": (100, 200, 400, 2.0, 150.0, 150.0, 10000, 2),
             "F60": (220, 200, 400, 2.0, 150.0, 150.0, 22000, 2)}
    for name, s in specs.items():
        c, fe = O.ref_make_pillars(scene_dict(s), 42, d_out=128)
        scenes[name] = dict(n=int(c.shape[0]), coords_fnv=fnv_np(c), feats_fnv=fnv_np(fe[:512]),
                            coords_sum=float(c.sum()), feats_sum=float(fe.sum()))
    scenes["params_default_seed42_fnv"] = fnv(O.ref_init_params(O.make_cfg(), 128, 42))
    with open(os.path.join(HERE, "scenes.json"), "w") as f:
        json.dump(scenes, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
