"""`fwa bench` on the B200 path (reference tools/fwa_cli.cpp:249-281,
include/fwa/bench.hpp:15-143, 215-326): the reference's benchmark protocol and JSON result
with the GPU implementation under the clock.

    build_pipeline (fwa_cli.cpp:82-107): points file -> pillarize (GPU) -> params
    mode group         : the full backbone, run_backbone through the host API (bench.hpp:215-242)
    mode global        : one group holding every pillar, one block (bench.hpp:246-264)
    mode equal-window  : the padded SST-style baseline, block 0 (bench.hpp:271-326)
    protocol           : `warmup` untimed calls, `runs` wall-clock samples (steady clock around
                         each call, the device synchronised inside it), samples beyond 3x the
                         IQR excluded, mean / linear-interpolation p50 / p95 (bench.hpp:75-143)
    result JSON        : name, n_points, config_digest, wall_time_ms {mean, p50, p95},
                         outliers_excluded, runs, warmup, stage_ms (bench.hpp:33-43)

stage_ms (group mode) reports this implementation's own stages (schedule, positional
embedding, fused block kernels, host<->device copies; CUDA events), not the reference's
sort/group/gather/attention/ffn/scatter split: here gather, attention, FFN and scatter are
one kernel per block.
"""
from __future__ import annotations

import math
import time
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import ConfigError, Context, FwaConfig, init_backbone_params, pillar_params


# ----------------------------------------------------------------------------- protocol
def percentile(sorted_samples: Sequence[float], q: float) -> float:
    """Linear-interpolation percentile of a sorted sample (bench.hpp:75-83)."""
    n = len(sorted_samples)
    if n == 0:
        return 0.0
    if n == 1:
        return float(sorted_samples[0])
    pos = q * (n - 1)
    lo = int(math.floor(pos))
    hi = min(lo + 1, n - 1)
    frac = pos - lo
    return float(sorted_samples[lo] + frac * (sorted_samples[hi] - sorted_samples[lo]))


def exclude_outliers(samples: Sequence[float]) -> Tuple[List[float], int]:
    """Drop samples beyond 3x the interquartile range (bench.hpp:86-106)."""
    if len(samples) < 4:
        return list(samples), 0
    s = sorted(samples)
    q1, q3 = percentile(s, 0.25), percentile(s, 0.75)
    lo, hi = q1 - 3.0 * (q3 - q1), q3 + 3.0 * (q3 - q1)
    kept = [x for x in samples if lo <= x <= hi]
    return kept, len(samples) - len(kept)


def summarize(name: str, n_points: int, digest: str, samples: Sequence[float], runs: int, warmup: int) -> dict:
    """BenchResult (bench.hpp:124-143) as its JSON document (bench.hpp:33-43)."""
    kept, excluded = exclude_outliers(samples)
    s = sorted(kept)
    mean = sum(kept) / len(kept) if kept else 0.0
    return {"name": name, "n_points": int(n_points), "config_digest": digest,
            "wall_time_ms": {"mean": mean, "p50": percentile(s, 0.5), "p95": percentile(s, 0.95)},
            "outliers_excluded": excluded, "runs": runs, "warmup": warmup, "stage_ms": {}}


def measure(runs: int, warmup: int, fn: Callable[[], None]) -> List[float]:
    """bench.hpp:108-122: steady-clock milliseconds around each call (fn synchronises)."""
    if runs < 1:
        raise ConfigError("bench: runs must be >= 1")
    if warmup < 0:
        raise ConfigError("bench: warmup must be >= 0")
    for _ in range(warmup):
        fn()
    out = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        out.append((time.perf_counter() - t0) * 1e3)
    return out


# ----------------------------------------------------------------------------- modes
DEFAULT_BUCKETS = (16, 32, 64, 128, 256)  # workload::default_bucket_edges


def _pillars(ctx: Context, input_path: str, cfg: FwaConfig, seed: int):
    """build_pipeline's pillarization (fwa_cli.cpp:82-90) on the GPU; returns host arrays."""
    import torch

    from .attend import ingest_points
    xy, feats = ingest_points(input_path)
    n_pts, f_in = xy.shape[0], feats.shape[1]
    dev = torch.device("cuda", ctx.device)
    w = torch.from_numpy(pillar_params(f_in, cfg.d_model, seed)).to(dev)
    d_xy = torch.from_numpy(np.ascontiguousarray(xy)).to(dev)
    d_f = torch.from_numpy(np.ascontiguousarray(feats if f_in else np.zeros((n_pts, 1)))).to(dev)
    d_pc = torch.empty((max(n_pts, 1), 2), dtype=torch.float64, device=dev)
    d_pf = torch.empty((max(n_pts, 1), cfg.d_model), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    n = ctx.pillarize_device(d_xy.data_ptr(), d_f.data_ptr(), n_pts, f_in, cfg.resolution, w.data_ptr(), 0,
                             cfg.d_model, d_pc.data_ptr(), d_pf.data_ptr(), n_pts)
    ctx.sync_check()
    return d_pc[:n].cpu().numpy(), d_pf[:n].cpu().numpy()


def bench(ctx: Context, input_path: str, cfg: Optional[FwaConfig] = None, mode: str = "group", runs: int = 50,
          warmup: int = 10, buckets: Sequence[int] = (), name: str = "", params_path: Optional[str] = None,
          seed: int = 42) -> dict:
    """cmd_bench (fwa_cli.cpp:249-281)."""
    import torch

    from . import PillarSet
    from .attend import config_digest
    cfg = cfg or FwaConfig()
    if runs < 1:
        raise ConfigError("--runs must be >= 1")
    if warmup < 0:
        raise ConfigError("--warmup must be >= 0")
    buckets = tuple(buckets) or DEFAULT_BUCKETS
    digest = config_digest(cfg)
    coords, feats = _pillars(ctx, input_path, cfg, seed)
    n = coords.shape[0]
    if params_path:
        with open(params_path, "rb") as fh:
            blob = fh.read()
    else:
        blob = init_backbone_params(cfg, seed)
    ctx.load_params(cfg, blob)
    if mode == "group":
        ps = PillarSet(coords, feats)
        samples = measure(runs, warmup, lambda: ctx.run_backbone(ps, cfg))
        r = summarize("group", n, digest, samples, runs, warmup)
        ctx.set_profiling(True)  # the stage split, one more profiled pass of each run
        for _ in range(runs):
            ctx.run_backbone(ps, cfg)
        prof = ctx.profile()
        ctx.set_profiling(False)
        r["stage_ms"] = {k: v / max(1, runs) for k, (v, c) in prof.items() if c}
        return r
    dev = torch.device("cuda", ctx.device)
    if mode == "global":
        if n == 0:
            raise ConfigError("bench: empty input")
        # one group of every pillar, block 0 (bench.hpp:246-264): features cast, PE computed
        f = feats.astype(np.float32)
        pe = ctx.positional_embedding(coords, cfg.d_model)
        record = blob[:16 + 4 * _record_floats(cfg)]
        samples = measure(runs, warmup, lambda: ctx.fwa_block_forward(f, pe, record, 1))
        return summarize("global", n, digest, samples, runs, warmup)
    if mode == "equal-window":
        d_coords = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
        d_feats = torch.from_numpy(feats.astype(np.float32)).to(dev)
        d_out = torch.empty((max(n, 1), cfg.d_model), dtype=torch.float32, device=dev)

        def one():
            ctx.equal_window_forward(d_coords.data_ptr(), d_feats.data_ptr(), n, cfg, d_out.data_ptr(), buckets)
            torch.cuda.synchronize(dev)

        samples = measure(runs, warmup, one)
        return summarize("equal-window", n, digest, samples, runs, warmup)
    raise ConfigError(f"unknown mode '{mode}'")


def _record_floats(cfg: FwaConfig) -> int:
    d, f = cfg.d_model, cfg.d_ff
    return 4 * d * d + 3 * d + d + 4 * d + 2 * d * f + f + d
