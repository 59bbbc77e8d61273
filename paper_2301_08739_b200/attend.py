"""`fwa attend` on the B200 path — the output-side data formats of the hot path
(reference: tools/fwa_cli.cpp:46-73, 82-107, 195-243).

    points file (FWPC binary or CSV, geometry.hpp:125-200)
      -> pillarize (GPU, geometry.hpp:246-300, random_pillar_params(f_in, d_model, seed))
      -> run_backbone (GPU, init_backbone_params(cfg, d_model, seed) or a FWAP file)
      -> JSON {n_input, n_kept, cache, dropped_per_block, config_digest, coords,
               row_checksums (GPU, bit-exact row sums in fp64), feature_hash (FNV-1a-64
               over the f32 feature bytes, bench.hpp:62-72)} [+ FWFB feature dump]

Everything between the file read and the JSON runs on the device (torch tensors are
only the buffers): 2.8 MB of points cross PCIe instead of a 63 MB f64 PillarSet.
"""
from __future__ import annotations

import json
import struct
from typing import Optional

import numpy as np

from . import (ConfigError, FwaConfig, ParseError, SchemaError, Context, fnv1a64_hex, init_backbone_params,
               lib, pillar_params)


# ----------------------------------------------------------------------------- inputs

def ingest_points(path: str):
    """read_points (fwa_cli.cpp:46-56): FWPC binary when the file starts with the magic,
    else CSV with an 'x,y,f0,f1,...' header.  Returns (xy n x 2 f64, features n x f_in f64)."""
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError:
        raise ConfigError(f"missing input file '{path}'") from None  # fwa_cli.cpp:48
    if data[:4] == b"FWPC":  # geometry.hpp:168-193
        if len(data) < 12:
            raise ParseError("truncated header")
        count, f_in = struct.unpack_from("<II", data, 4)
        need = 12 + count * (2 + f_in) * 8
        if len(data) < need:
            raise ParseError("truncated record")
        rec = np.frombuffer(data, "<f8", count * (2 + f_in), 12).reshape(count, 2 + f_in)
        return rec[:, :2].copy(), rec[:, 2:].copy()
    lines = data.decode().splitlines()  # geometry.hpp:125-166
    if not lines:
        raise ParseError("line 1: missing CSV header")
    header = [h.strip() for h in lines[0].strip().split(",")]
    if len(header) < 2 or header[0] != "x" or header[1] != "y":
        raise SchemaError("line 1: header must start with 'x,y'")
    for i, h in enumerate(header[2:]):
        if h != f"f{i}":
            raise SchemaError(f"line 1: expected feature column 'f{i}', got '{h}'")
    rows = []
    for ln, line in enumerate(lines[1:], start=2):
        t = line.strip()
        if not t:
            continue
        fields = t.split(",")
        if len(fields) != len(header):
            raise SchemaError(f"line {ln}: expected {len(header)} fields, got {len(fields)}")
        try:
            vals = [float(x.strip()) for x in fields]
        except ValueError:
            raise ParseError(f"line {ln}: bad number") from None
        if not (np.isfinite(vals[0]) and np.isfinite(vals[1])):
            raise ParseError(f"line {ln}: non-finite coordinate")
        rows.append(vals)
    a = np.array(rows, np.float64).reshape(-1, len(header))
    return a[:, :2].copy(), a[:, 2:].copy()


def read_config(path: Optional[str]) -> FwaConfig:
    """read_config + from_json (fwa_cli.cpp:58-69, backbone.hpp:59-70): missing keys
    take the FwaConfig defaults."""
    if not path:
        return FwaConfig()
    try:
        with open(path) as fh:
            j = json.load(fh)
    except FileNotFoundError:
        raise ConfigError(f"missing config file '{path}'") from None
    except json.JSONDecodeError as e:
        raise ParseError(f"config '{path}': {e}") from None
    w = j.get("window", [9, 9])
    return FwaConfig(resolution=float(j.get("resolution", 0.32)), window_px=int(w[0]), window_py=int(w[1]),
                     group_size=int(j.get("group_size", 69)), n_blocks=int(j.get("n_blocks", 8)),
                     d_model=int(j.get("d_model", 128)), n_heads=int(j.get("n_heads", 8)),
                     d_ff=int(j.get("d_ff", 256)))


def config_json(cfg: FwaConfig) -> str:
    """nlohmann::json(FwaConfig).dump() (backbone.hpp:49-57): compact, keys sorted."""
    return json.dumps({"resolution": cfg.resolution, "window": [cfg.window_px, cfg.window_py],
                       "group_size": cfg.group_size, "n_blocks": cfg.n_blocks, "d_model": cfg.d_model,
                       "n_heads": cfg.n_heads, "d_ff": cfg.d_ff}, separators=(",", ":"), sort_keys=True)


def config_digest(cfg: FwaConfig) -> str:
    """config_digest (fwa_cli.cpp:71-73)."""
    return fnv1a64_hex(config_json(cfg).encode())


def cache_and_drops(n: int, cfg: FwaConfig):
    """The reference's sort-cache rule and drop bookkeeping (backbone.hpp:224-234,
    285-316): a spec's plan is reused while the active count is unchanged; only a block
    whose active count is not a multiple of G drops (then the cache is cleared)."""
    have = {}
    comp = hit = 0
    act = n
    drops = []
    for b in range(cfg.n_blocks):
        s = b % 4
        if have.get(s) == act:
            hit += 1
        else:
            comp += 1
            have[s] = act
        d = act % cfg.group_size
        drops.append(d)
        if d:
            act -= d
            have.clear()
    return (comp, hit), drops


def write_fwfb(path: str, features: np.ndarray):
    """FWFB dump (fwa_cli.cpp:228-239): magic, u32 n, u32 d, f32 rows."""
    f = np.ascontiguousarray(features, np.float32)
    with open(path, "wb") as fh:
        fh.write(b"FWFB" + struct.pack("<II", f.shape[0], f.shape[1]) + f.tobytes())


# ----------------------------------------------------------------------------- the command

def attend(ctx: Context, input_path: str, cfg: Optional[FwaConfig] = None, params_path: Optional[str] = None,
           seed: int = 42, features_out: Optional[str] = None) -> dict:
    """cmd_attend (fwa_cli.cpp:195-243) with the pillarizer, the backbone and the row
    checksums on the device."""
    import torch

    cfg = cfg or FwaConfig()
    xy, feats = ingest_points(input_path)
    n_pts, f_in = xy.shape[0], feats.shape[1]
    if params_path:
        with open(params_path, "rb") as fh:
            blob = fh.read()
    else:
        blob = init_backbone_params(cfg, seed)
    ctx.load_params(cfg, blob)
    dev = torch.device("cuda", ctx.device)
    w = torch.from_numpy(pillar_params(f_in, cfg.d_model, seed)).to(dev)
    d_xy = torch.from_numpy(np.ascontiguousarray(xy)).to(dev)
    d_f = torch.from_numpy(np.ascontiguousarray(feats if f_in else np.zeros((n_pts, 1)))).to(dev)
    d_pc = torch.empty((max(n_pts, 1), 2), dtype=torch.float64, device=dev)
    d_pf = torch.empty((max(n_pts, 1), cfg.d_model), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    n = ctx.pillarize_device(d_xy.data_ptr(), d_f.data_ptr(), n_pts, f_in, cfg.resolution, w.data_ptr(), 0,
                             cfg.d_model, d_pc.data_ptr(), d_pf.data_ptr(), n_pts)
    ctx.sync_check()  # the library's stream -> torch's
    if n < cfg.group_size:
        from . import NumericError
        raise NumericError("fewer active pillars than group size")  # backbone.hpp:218-222
    d_feats = d_pf[:n].float()  # PillarSet f64 -> f32 exactly as backbone.hpp:195-196
    d_out = torch.empty((n, cfg.d_model), dtype=torch.float32, device=dev)
    d_kept = torch.empty(n, dtype=torch.int32, device=dev)
    d_sum = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    nk = ctx.forward_device(d_pc.data_ptr(), d_feats.data_ptr(), [0, n], cfg, d_out.data_ptr(),
                            d_kept.data_ptr())
    ctx.sync_check()
    ctx._check(lib().fwa_b200_row_checksums(ctx._h, d_out.data_ptr(), nk, cfg.d_model, d_sum.data_ptr()))
    ctx.sync_check()
    out = d_out[:nk].cpu().numpy()
    kept = d_kept[:nk].cpu().numpy()
    coords = d_pc[:n].cpu().numpy()[kept]
    (comp, hit), drops = cache_and_drops(n, cfg)
    j = {"n_input": int(n), "n_kept": int(nk), "cache": {"computed": comp, "hits": hit},
         "dropped_per_block": drops, "config_digest": config_digest(cfg),
         "coords": coords.tolist(), "row_checksums": d_sum[:nk].cpu().numpy().tolist(),
         "feature_hash": fnv1a64_hex(out.tobytes())}
    if features_out:
        write_fwfb(features_out, out)
    return j
