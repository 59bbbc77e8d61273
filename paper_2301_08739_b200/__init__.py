"""B200-native FlatFormer backbone forward (flattened window attention).

Python mirror of the reference library's hot-path API (paths relative to
/root/reference/proj/include/fwa):

    FwaConfig, validate            backbone.hpp:22-47
    PillarSet                      geometry.hpp:46-52
    BackboneOutput / RunStats      backbone.hpp:104-135
    run_backbone(pillars, cfg, params, n_threads)   backbone.hpp:159-334
    sort / group / block_schedule  flatten.hpp:97-161
    positional_embedding           kernels.hpp:364-393
    fwa_block_forward              kernels.hpp:636-650
    init_backbone_params           backbone.hpp:83-102 (FWAP bytes, kernels.hpp:149-175)
    generate_synthetic+pillarize   geometry.hpp:246-386

Every numeric call goes through the C ABI of ``libfwa_b200.so`` (include/fwa_b200.h):
hand-written sm_100a CUDA kernels.  There is no CPU fallback — if the library or a
GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FWA_B200_LIB") or os.path.join(HERE, "libfwa_b200.so")  # override: A/B builds

EXPORTS = [
    "fwa_b200_ctx_create", "fwa_b200_ctx_destroy", "fwa_b200_last_error", "fwa_b200_set_precision",
    "fwa_b200_kernel_launches", "fwa_b200_fast_path", "fwa_b200_load_params",
    "fwa_b200_set_profiling", "fwa_b200_get_profile", "fwa_b200_sync_check",
    "fwa_b200_backbone_forward", "fwa_b200_backbone_forward_batch", "fwa_b200_backbone_forward_frames",
    "fwa_b200_backbone_forward_device", "fwa_b200_sort_plan", "fwa_b200_block_forward",
    "fwa_b200_positional_embedding", "fwa_b200_positional_embedding_f16", "fwa_b200_generate_pillars", "fwa_b200_init_params",
    "fwa_b200_split_begin", "fwa_b200_split_block", "fwa_b200_split_scatter", "fwa_b200_split_plan",
    "fwa_b200_split_plan_device",
    "fwa_b200_pillarize", "fwa_b200_pillarize_device", "fwa_b200_generate_points", "fwa_b200_pillar_params",
    "fwa_b200_row_checksums", "fwa_b200_fnv1a64", "fwa_b200_equal_window_forward", "fwa_b200_block_backward",
    "fwa_b200_load_input_proj", "fwa_b200_init_params_fin", "fwa_b200_current_device",
    "fwa_b200_split_p2p_setup", "fwa_b200_split_block_p2p", "fwa_b200_alloc", "fwa_b200_free",
    "fwa_b200_ipc_handle", "fwa_b200_ipc_open", "fwa_b200_ipc_close",
]

PREC_BF16, PREC_FP32, PREC_BF16_3K = 0, 1, 2
_PREC = {"bf16": PREC_BF16, "fp32": PREC_FP32, "bf16_3k": PREC_BF16_3K}


# ----------------------------------------------------------------------------- errors (error.hpp)

class FwaError(RuntimeError):
    code = 7


class ConfigError(FwaError):
    code = 1


class ParseError(FwaError):
    code = 2


class SchemaError(FwaError):
    code = 3


class ShapeError(FwaError):
    code = 4


class NumericError(FwaError):
    code = 5


class ContractError(FwaError):
    code = 6


class CudaError(FwaError):
    code = 8


_ERRS = {c.code: c for c in (ConfigError, ParseError, SchemaError, ShapeError, NumericError,
                             ContractError, FwaError, CudaError)}


# ----------------------------------------------------------------------------- C structs

class _Cfg(C.Structure):
    _fields_ = [("resolution", C.c_double), ("window_px", C.c_int32), ("window_py", C.c_int32),
                ("group_size", C.c_int32), ("n_blocks", C.c_int32), ("d_model", C.c_int32),
                ("n_heads", C.c_int32), ("d_ff", C.c_int32)]


class _Out(C.Structure):
    _fields_ = [("features", C.c_void_p), ("kept_indices", C.c_void_p), ("dropped_ids", C.c_void_p),
                ("dropped_per_block", C.c_void_p), ("block_perms", C.c_void_p),
                ("n_kept", C.c_int64), ("cache_computed", C.c_int32), ("cache_hits", C.c_int32),
                ("stage_ms", C.c_double * 6)]


class _FrameStats(C.Structure):
    _fields_ = [("n_kept", C.c_int64), ("n_dropped", C.c_int32), ("cache_computed", C.c_int32),
                ("cache_hits", C.c_int32)]


STAGES = ("sort", "group", "gather", "attention", "ffn", "scatter")  # StageTimes order (backbone.hpp:109-126)


class _EwReport(C.Structure):
    _fields_ = [("n_windows", C.c_int64), ("max_occ", C.c_int32), ("min_nonzero_occ", C.c_int32),
                ("padding_factor", C.c_double), ("rows_padded", C.c_int64), ("n_buckets", C.c_int32),
                ("bucket_edge", C.c_int32 * 8), ("bucket_pad", C.c_int32 * 8), ("bucket_windows", C.c_int64 * 8)]


class _Scene(C.Structure):
    _fields_ = [("n_clusters", C.c_int32), ("points_per_cluster_min", C.c_int32),
                ("points_per_cluster_max", C.c_int32), ("cluster_sigma", C.c_double),
                ("extent_x", C.c_double), ("extent_y", C.c_double), ("n_background", C.c_int32),
                ("f_in", C.c_int32)]


_lib_handle = None


def lib():
    """Load libfwa_b200.so (fails loudly when it has not been built)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.fwa_b200_ctx_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
        L.fwa_b200_ctx_destroy.argtypes = [vp]
        L.fwa_b200_last_error.argtypes = [vp]
        L.fwa_b200_last_error.restype = C.c_char_p
        L.fwa_b200_set_precision.argtypes = [vp, C.c_int]
        L.fwa_b200_kernel_launches.argtypes = [vp]
        L.fwa_b200_kernel_launches.restype = i64
        L.fwa_b200_fast_path.argtypes = [vp, C.POINTER(_Cfg)]
        L.fwa_b200_set_profiling.argtypes = [vp, C.c_int]
        L.fwa_b200_sync_check.argtypes = [vp]
        L.fwa_b200_get_profile.argtypes = [vp, vp, vp]
        L.fwa_b200_load_params.argtypes = [vp, C.POINTER(_Cfg), vp, C.c_size_t]
        L.fwa_b200_load_input_proj.argtypes = [vp, i32, i32, vp, vp]
        L.fwa_b200_backbone_forward.argtypes = [vp, vp, vp, C.c_int, i64, C.POINTER(_Cfg),
                                                C.POINTER(_Out)]
        L.fwa_b200_backbone_forward_frames.argtypes = [vp, C.c_int, vp, vp, C.c_int, vp, C.POINTER(_Cfg),
                                                       C.POINTER(_Out)]
        L.fwa_b200_backbone_forward_batch.argtypes = [vp, vp, vp, C.c_int, vp, C.c_int,
                                                      C.POINTER(_Cfg), C.POINTER(_Out), vp]
        L.fwa_b200_backbone_forward_device.argtypes = [vp, vp, vp, vp, C.c_int, C.POINTER(_Cfg),
                                                       vp, vp, C.POINTER(i64)]
        L.fwa_b200_sort_plan.argtypes = [vp, vp, i64, C.c_double, C.c_double, C.c_int, C.c_int, vp]
        L.fwa_b200_block_forward.argtypes = [vp, vp, vp, i64, i32, vp, C.c_size_t, vp]
        L.fwa_b200_positional_embedding.argtypes = [vp, vp, i64, i32, vp]
        L.fwa_b200_positional_embedding_f16.argtypes = [vp, vp, i64, i32, vp]
        L.fwa_b200_generate_pillars.argtypes = [C.POINTER(_Scene), C.c_uint64, C.c_double, i32,
                                                C.c_uint64, vp, vp]
        L.fwa_b200_generate_pillars.restype = i64
        L.fwa_b200_split_begin.argtypes = [vp, vp, i64, C.POINTER(_Cfg), C.POINTER(i64)]
        L.fwa_b200_split_block.argtypes = [vp, C.c_int, i64, i64, vp, vp]
        L.fwa_b200_split_scatter.argtypes = [vp, C.c_int, vp, vp]
        L.fwa_b200_split_plan.argtypes = [vp, C.c_int, vp]
        L.fwa_b200_split_plan_device.argtypes = [vp, C.c_int, vp]
        L.fwa_b200_split_p2p_setup.argtypes = [vp, C.c_int, C.c_int, vp, vp]
        L.fwa_b200_split_block_p2p.argtypes = [vp, C.c_int, vp]
        L.fwa_b200_alloc.argtypes = [vp, C.c_size_t]
        L.fwa_b200_alloc.restype = vp
        L.fwa_b200_free.argtypes = [vp, vp]
        L.fwa_b200_free.restype = None
        L.fwa_b200_ipc_handle.argtypes = [vp, vp, vp]
        L.fwa_b200_ipc_open.argtypes = [vp, vp, C.POINTER(vp)]
        L.fwa_b200_ipc_close.argtypes = [vp, vp]
        L.fwa_b200_init_params.argtypes = [C.POINTER(_Cfg), C.c_uint64, vp, C.c_size_t]
        L.fwa_b200_init_params.restype = i64
        L.fwa_b200_init_params_fin.argtypes = [C.POINTER(_Cfg), i32, C.c_uint64, vp, C.c_size_t, vp]
        L.fwa_b200_init_params_fin.restype = i64
        L.fwa_b200_pillarize.argtypes = [vp, vp, vp, i64, i32, C.c_double, vp, vp, i32, vp, vp, C.POINTER(i64)]
        L.fwa_b200_pillarize_device.argtypes = [vp, vp, vp, i64, i32, C.c_double, vp, vp, i32, vp, vp, i64,
                                                C.POINTER(i64)]
        L.fwa_b200_generate_points.argtypes = [C.POINTER(_Scene), C.c_uint64, vp, vp]
        L.fwa_b200_generate_points.restype = i64
        L.fwa_b200_pillar_params.argtypes = [i32, i32, C.c_uint64, vp]
        L.fwa_b200_pillar_params.restype = i64
        L.fwa_b200_row_checksums.argtypes = [vp, vp, i64, i32, vp]
        L.fwa_b200_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.fwa_b200_fnv1a64.restype = C.c_uint64
        L.fwa_b200_block_backward.argtypes = [vp, vp, vp, i64, i32, vp, C.c_size_t, vp, vp, vp]
        L.fwa_b200_equal_window_forward.argtypes = [vp, vp, vp, i64, C.POINTER(_Cfg), vp, i32, vp,
                                                     C.POINTER(_EwReport)]
        _lib_handle = L
    return _lib_handle


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------- reference types

@dataclass
class FwaConfig:
    """fwa::backbone::FwaConfig (backbone.hpp:22-34)."""
    resolution: float = 0.32
    window_px: int = 9
    window_py: int = 9
    group_size: int = 69
    n_blocks: int = 8
    d_model: int = 128
    n_heads: int = 8
    d_ff: int = 256

    def window_x_m(self) -> float:
        return self.window_px * self.resolution

    def window_y_m(self) -> float:
        return self.window_py * self.resolution

    def c(self) -> _Cfg:
        return _Cfg(self.resolution, self.window_px, self.window_py, self.group_size,
                    self.n_blocks, self.d_model, self.n_heads, self.d_ff)

    def to_json(self) -> dict:
        return {"resolution": self.resolution, "window": [self.window_px, self.window_py],
                "group_size": self.group_size, "n_blocks": self.n_blocks,
                "d_model": self.d_model, "n_heads": self.n_heads, "d_ff": self.d_ff}

    @classmethod
    def from_json(cls, j: dict) -> "FwaConfig":
        """backbone.hpp:59-70 (missing keys take the defaults)."""
        w = j.get("window", [9, 9])
        return cls(j.get("resolution", 0.32), int(w[0]), int(w[1]), j.get("group_size", 69),
                   j.get("n_blocks", 8), j.get("d_model", 128), j.get("n_heads", 8),
                   j.get("d_ff", 256))


def validate(cfg: FwaConfig) -> None:
    """backbone.hpp:36-47."""
    if not cfg.resolution > 0.0:
        raise ConfigError("config: resolution must be > 0")
    if cfg.window_px < 1 or cfg.window_py < 1:
        raise ConfigError("config: window dims must be >= 1")
    if cfg.group_size < 1:
        raise ConfigError("config: group_size must be >= 1")
    if cfg.n_blocks < 1:
        raise ConfigError("config: n_blocks must be >= 1")
    if cfg.d_model < 4 or cfg.d_model % 4:
        raise ConfigError("config: d_model must be divisible by 4")
    if cfg.n_heads < 1 or cfg.d_model % cfg.n_heads:
        raise ConfigError("config: d_model must be divisible by n_heads")
    if cfg.d_ff < 1:
        raise ConfigError("config: d_ff must be >= 1")


@dataclass
class PillarSet:
    """geometry::PillarSet: coords N x 2 f64 (cell centres), features N x D f64."""
    coords: np.ndarray
    features: np.ndarray
    resolution: float = 0.32

    def size(self) -> int:
        return int(self.coords.shape[0])


@dataclass
class CacheStats:
    computed: int = 0
    hits: int = 0


@dataclass
class StageTimes:
    """backbone.hpp:109-126: milliseconds per stage of one call (device time, CUDA events;
    the fused block kernel's time apportioned by its per-phase SM-clock counters)."""
    sort_ms: float = 0.0
    group_ms: float = 0.0
    gather_ms: float = 0.0
    attention_ms: float = 0.0
    ffn_ms: float = 0.0
    scatter_ms: float = 0.0

    def total(self) -> float:
        return self.sort_ms + self.group_ms + self.gather_ms + self.attention_ms + self.ffn_ms + self.scatter_ms

    @classmethod
    def from_c(cls, a) -> "StageTimes":
        return cls(*[float(a[i]) for i in range(6)])


@dataclass
class RunStats:
    cache: CacheStats = field(default_factory=CacheStats)
    dropped_per_block: List[int] = field(default_factory=list)
    stages: StageTimes = field(default_factory=StageTimes)


@dataclass
class BackboneOutput:
    """backbone.hpp:128-135 (+ optional per-block plans, the parity hook)."""
    features: np.ndarray
    coords: np.ndarray
    kept_indices: np.ndarray
    dropped_indices: List[np.ndarray]
    stats: RunStats
    n_input: int
    block_perms: Optional[List[np.ndarray]] = None


@dataclass
class WindowSpec:
    """flatten::WindowSpec (flatten.hpp:22-29)."""
    w_x: float = 1.0
    w_y: float = 1.0
    shift: bool = False
    major_axis: str = "X"


def block_schedule(n_blocks: int, w_x: float, w_y: float) -> List[WindowSpec]:
    """flatten.hpp:150-161: axis X iff i % 4 < 2, shift iff i odd."""
    if n_blocks < 1:
        raise ConfigError("n_blocks must be >= 1")
    return [WindowSpec(w_x, w_y, i % 2 == 1, "X" if i % 4 < 2 else "Y") for i in range(n_blocks)]


# ----------------------------------------------------------------------------- device context

class Context:
    """One CUDA device + stream; owns device workspace and resident parameters."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, precision: str = "bf16"):
        L = lib()
        h = C.c_void_p()
        rc = L.fwa_b200_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h))
        if rc:
            raise _ERRS.get(rc, FwaError)(f"fwa_b200_ctx_create failed ({rc}) on device {device}")
        self._h = h
        self.device = device
        self.set_precision(precision)

    def close(self):
        if getattr(self, "_h", None):
            lib().fwa_b200_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            msg = lib().fwa_b200_last_error(self._h).decode()
            raise _ERRS.get(rc, FwaError)(msg)

    def set_precision(self, precision: str):
        if precision not in _PREC:
            raise ValueError(f"precision must be one of {sorted(_PREC)}")
        self._check(lib().fwa_b200_set_precision(self._h, _PREC[precision]))
        self.precision = precision

    @property
    def kernel_launches(self) -> int:
        return int(lib().fwa_b200_kernel_launches(self._h))

    PROF_SLOTS = ("schedule", "pe", "ln1_qkv", "attention", "outproj_ffn", "h2d", "d2h", "block_fused")

    def set_profiling(self, enable: bool = True):
        self._check(lib().fwa_b200_set_profiling(self._h, int(enable)))

    def profile(self) -> dict:
        """{slot: (total_ms, calls)} accumulated since set_profiling()."""
        ms = np.zeros(len(self.PROF_SLOTS), np.float64)
        n = np.zeros(len(self.PROF_SLOTS), np.int64)
        self._check(lib().fwa_b200_get_profile(self._h, _ptr(ms), _ptr(n)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.PROF_SLOTS)}

    def fast_path(self, cfg: FwaConfig) -> bool:
        c = cfg.c()
        return bool(lib().fwa_b200_fast_path(self._h, C.byref(c)))

    def load_params(self, cfg: FwaConfig, fwap: bytes):
        c = cfg.c()
        buf = np.frombuffer(fwap, np.uint8)
        self._check(lib().fwa_b200_load_params(self._h, C.byref(c), _ptr(buf), len(fwap)))
        self._params_key = (id(fwap), len(fwap))

    def run_backbone(self, pillars: PillarSet, cfg: FwaConfig, want_block_perms=False) -> BackboneOutput:
        coords = np.ascontiguousarray(pillars.coords, np.float64)
        feats = pillars.features
        f64 = 1 if feats.dtype == np.float64 else 0
        feats = np.ascontiguousarray(feats, np.float64 if f64 else np.float32)
        n = coords.shape[0]
        self._check_width(feats, n, cfg)
        out_f = np.empty((n, cfg.d_model), np.float32)
        kept = np.empty(n, np.int32)
        dropped = np.empty(max(n, 1), np.int32)
        dpb = np.zeros(cfg.n_blocks, np.int32)
        perms = np.full((cfg.n_blocks, n), -1, np.int32) if want_block_perms else None
        o = _Out(_ptr(out_f).value, _ptr(kept).value, _ptr(dropped).value, _ptr(dpb).value,
                 _ptr(perms).value if perms is not None else None, 0, 0, 0)
        c = cfg.c()
        self._check(lib().fwa_b200_backbone_forward(self._h, _ptr(coords), _ptr(feats), f64, n,
                                                    C.byref(c), C.byref(o)))
        k = int(o.n_kept)
        dropped_lists, w = [], 0
        for b in range(cfg.n_blocks):
            dropped_lists.append(dropped[w:w + dpb[b]].copy())
            w += int(dpb[b])
        bp = None
        if want_block_perms:
            bp = []
            for b in range(cfg.n_blocks):
                n_act = n if (b == 0 or w == 0) else k
                bp.append(perms[b, :n_act].copy())
        return BackboneOutput(features=out_f[:k], coords=coords[kept[:k]], kept_indices=kept[:k],
                              dropped_indices=dropped_lists,
                              stats=RunStats(CacheStats(int(o.cache_computed), int(o.cache_hits)),
                                             [int(x) for x in dpb], StageTimes.from_c(o.stage_ms)),
                              n_input=n, block_perms=bp)

    def _check_width(self, feats, n, cfg):
        w = self._proj_in or cfg.d_model
        if feats.ndim != 2 or feats.shape[0] != n:
            raise ShapeError("backbone: features must be N x width")
        if feats.shape[1] != w:
            raise ShapeError("backbone: input projection width mismatch" if self._proj_in else
                             "backbone: pillar width != d_model and no input projection")

    _proj_in = 0

    def load_input_proj(self, weight: Optional[np.ndarray], bias: Optional[np.ndarray] = None):
        """BackboneParams::input_proj (backbone.hpp:74-81): weight d_model x f_in, bias d_model
        (None = zeros); None removes it.  Projected on the device, bit-exact."""
        if weight is None:
            self._check(lib().fwa_b200_load_input_proj(self._h, 0, 0, None, None))
            self._proj_in = 0
            return
        w = np.ascontiguousarray(weight, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        self._check(lib().fwa_b200_load_input_proj(self._h, w.shape[0], w.shape[1], _ptr(w),
                                                     _ptr(b) if b is not None else None))
        self._proj_in = int(w.shape[1])

    def run_backbone_ptrs(self, coords_ptr: int, feats_ptr: int, feats_is_f64: bool, n: int,
                          cfg: FwaConfig, out_features_ptr: int, kept_ptr: int = 0,
                          dropped_ptr: int = 0, dropped_per_block_ptr: int = 0):
        """run_backbone on caller-owned HOST buffers given as raw pointers (e.g. pinned
        torch tensors): coords N x 2 f64, feats N x D (f64 or f32).  Returns
        (n_kept, (cache_computed, cache_hits))."""
        o = _Out(out_features_ptr, kept_ptr or None, dropped_ptr or None,
                 dropped_per_block_ptr or None, None, 0, 0, 0)
        c = cfg.c()
        self._check(lib().fwa_b200_backbone_forward(self._h, C.c_void_p(coords_ptr),
                                                    C.c_void_p(feats_ptr), int(feats_is_f64), n,
                                                    C.byref(c), C.byref(o)))
        return int(o.n_kept), (int(o.cache_computed), int(o.cache_hits))

    def run_frames(self, frames: Sequence[PillarSet], cfg: FwaConfig) -> List[BackboneOutput]:
        """run_backbone over a sequence of frames with the PCIe copies pipelined against
        the compute (fwa_b200_backbone_forward_frames); output i == run_backbone(frames[i])."""
        keep, bufs = [], []
        f64 = None
        for ps in frames:
            coords = np.ascontiguousarray(ps.coords, np.float64)
            is64 = ps.features.dtype == np.float64
            if f64 is None:
                f64 = is64
            elif f64 != is64:
                raise ShapeError("frames: mixed feature dtypes")
            feats = np.ascontiguousarray(ps.features, np.float64 if is64 else np.float32)
            n = coords.shape[0]
            self._check_width(feats, n, cfg)
            out_f = np.empty((n, cfg.d_model), np.float32)
            kept = np.empty(max(n, 1), np.int32)
            dropped = np.empty(max(n, 1), np.int32)
            dpb = np.zeros(cfg.n_blocks, np.int32)
            keep.append((coords, feats, out_f, kept, dropped, dpb))
        ptrs = [(k[0].ctypes.data, k[1].ctypes.data, k[0].shape[0], k[2].ctypes.data, k[3].ctypes.data,
                 k[4].ctypes.data, k[5].ctypes.data) for k in keep]
        stats = self.run_frames_ptrs(ptrs, bool(f64), cfg, stages=True)
        outs = []
        for (coords, _, out_f, kept, dropped, dpb), (k, cache, stg) in zip(keep, stats):
            dropped_lists, w = [], 0
            for b in range(cfg.n_blocks):
                dropped_lists.append(dropped[w:w + dpb[b]].copy())
                w += int(dpb[b])
            outs.append(BackboneOutput(features=out_f[:k], coords=coords[kept[:k]], kept_indices=kept[:k],
                                       dropped_indices=dropped_lists,
                                       stats=RunStats(CacheStats(*cache), [int(x) for x in dpb], stg),
                                       n_input=coords.shape[0], block_perms=None))
        return outs

    def run_frames_ptrs(self, frames, feats_is_f64: bool, cfg: FwaConfig, stages: bool = False):
        """fwa_b200_backbone_forward_frames on caller-owned HOST buffers: `frames` is a list
        of (coords_ptr, feats_ptr, n, out_features_ptr, kept_ptr, dropped_ptr,
        dropped_per_block_ptr) (0 = not wanted).  Returns [(n_kept, (computed, hits))]."""
        F = len(frames)
        cp = (C.c_void_p * F)(*[f[0] for f in frames])
        fp = (C.c_void_p * F)(*[f[1] for f in frames])
        ns = (C.c_int64 * F)(*[int(f[2]) for f in frames])
        outs = (_Out * F)(*[_Out(f[3], f[4] or None, f[5] or None, f[6] or None, None, 0, 0, 0) for f in frames])
        c = cfg.c()
        self._check(lib().fwa_b200_backbone_forward_frames(self._h, F, cp, fp, int(feats_is_f64), ns, C.byref(c),
                                                           outs))
        if stages:
            return [(int(o.n_kept), (int(o.cache_computed), int(o.cache_hits)), StageTimes.from_c(o.stage_ms))
                    for o in outs]
        return [(int(o.n_kept), (int(o.cache_computed), int(o.cache_hits))) for o in outs]

    def run_batch(self, coords: np.ndarray, feats: np.ndarray, frame_offsets: Sequence[int],
                  cfg: FwaConfig):
        """Frame-parallel forward (BASELINE config 3): frames concatenated along rows."""
        coords = np.ascontiguousarray(coords, np.float64)
        f64 = 1 if feats.dtype == np.float64 else 0
        feats = np.ascontiguousarray(feats, np.float64 if f64 else np.float32)
        off = np.ascontiguousarray(frame_offsets, np.int64)
        n = coords.shape[0]
        nf = len(off) - 1
        out_f = np.empty((n, cfg.d_model), np.float32)
        kept = np.empty(n, np.int32)
        dropped = np.empty(max(n, 1), np.int32)
        dpb = np.zeros(cfg.n_blocks, np.int32)
        fs = (_FrameStats * nf)()
        o = _Out(_ptr(out_f).value, _ptr(kept).value, _ptr(dropped).value, _ptr(dpb).value, None, 0, 0, 0)
        c = cfg.c()
        self._check(lib().fwa_b200_backbone_forward_batch(self._h, _ptr(coords), _ptr(feats), f64,
                                                          _ptr(off), nf, C.byref(c), C.byref(o), fs))
        k = int(o.n_kept)
        frame_stats = [dict(n_kept=int(x.n_kept), n_dropped=int(x.n_dropped),
                            cache=(int(x.cache_computed), int(x.cache_hits)),
                            dropped_per_block=[int(x.n_dropped)] + [0] * (cfg.n_blocks - 1)) for x in fs]
        return dict(features=out_f[:k], kept=kept[:k], dropped=dropped[:int(dpb.sum())],
                    kept_per_frame=np.array([x["n_kept"] for x in frame_stats], np.int64),
                    frame_stats=frame_stats, cache=(int(o.cache_computed), int(o.cache_hits)),
                    stages=StageTimes.from_c(o.stage_ms))

    def forward_device(self, d_coords: int, d_feats: int, frame_offsets: Sequence[int],
                       cfg: FwaConfig, d_out: int, d_kept: Optional[int] = None) -> int:
        """Device-resident forward: raw device pointers (e.g. torch tensor data_ptr())."""
        off = np.ascontiguousarray(frame_offsets, np.int64)
        c = cfg.c()
        nk = C.c_int64()
        self._check(lib().fwa_b200_backbone_forward_device(
            self._h, C.c_void_p(d_coords), C.c_void_p(d_feats), _ptr(off), len(off) - 1,
            C.byref(c), C.c_void_p(d_out), C.c_void_p(d_kept) if d_kept else None, C.byref(nk)))
        return int(nk.value)

    # ---- group-range split (BASELINE config 4), see paper_2301_08739_b200/split.py
    def split_begin(self, d_coords: int, n: int, cfg: FwaConfig) -> int:
        c = cfg.c()
        k = C.c_int64()
        self._check(lib().fwa_b200_split_begin(self._h, C.c_void_p(d_coords), n, C.byref(c), C.byref(k)))
        return int(k.value)

    def split_block(self, b: int, g0: int, g1: int, d_x: int, d_y: int):
        self._check(lib().fwa_b200_split_block(self._h, b, g0, g1, C.c_void_p(d_x), C.c_void_p(d_y)))

    def split_scatter(self, b: int, d_y: int, d_dst: int):
        self._check(lib().fwa_b200_split_scatter(self._h, b, C.c_void_p(d_y), C.c_void_p(d_dst)))

    def split_p2p_setup(self, world: int, rank: int, x_ptrs: Sequence[int], out_ptrs: Sequence[int]):
        """Peer-memory split: `world` device pointers of every rank's x buffer (N x D f32) and
        output buffer (K x D f32), valid in this process."""
        xp = (C.c_void_p * world)(*x_ptrs)
        op = (C.c_void_p * world)(*out_ptrs)
        self._check(lib().fwa_b200_split_p2p_setup(self._h, world, rank, xp, op))

    def split_block_p2p(self, b: int, d_x: int):
        self._check(lib().fwa_b200_split_block_p2p(self._h, b, C.c_void_p(d_x)))

    def alloc(self, nbytes: int) -> int:
        """cudaMalloc'd device memory (shareable by CUDA IPC)."""
        p = lib().fwa_b200_alloc(self._h, nbytes)
        if not p:
            raise CudaError(lib().fwa_b200_last_error(self._h).decode())
        return int(p)

    def free(self, ptr: int):
        lib().fwa_b200_free(self._h, C.c_void_p(ptr))

    def ipc_handle(self, ptr: int) -> bytes:
        h = (C.c_uint8 * 64)()
        self._check(lib().fwa_b200_ipc_handle(self._h, C.c_void_p(ptr), h))
        return bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        p = C.c_void_p()
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        self._check(lib().fwa_b200_ipc_open(self._h, h, C.byref(p)))
        return int(p.value)

    def ipc_close(self, ptr: int):
        self._check(lib().fwa_b200_ipc_close(self._h, C.c_void_p(ptr)))

    def split_plan_device(self, b: int, d_ids: int):
        self._check(lib().fwa_b200_split_plan_device(self._h, b, C.c_void_p(d_ids)))

    def split_plan(self, b: int, K: int) -> np.ndarray:
        ids = np.empty(K, np.int32)
        self._check(lib().fwa_b200_split_plan(self._h, b, _ptr(ids)))
        return ids

    def sync_check(self):
        """Wait for the stream; raise deferred device-side errors of forward_device."""
        self._check(lib().fwa_b200_sync_check(self._h))

    def sort(self, coords: np.ndarray, spec: WindowSpec) -> np.ndarray:
        coords = np.ascontiguousarray(coords, np.float64)
        perm = np.empty(coords.shape[0], np.int32)
        self._check(lib().fwa_b200_sort_plan(self._h, _ptr(coords), coords.shape[0], spec.w_x,
                                             spec.w_y, int(spec.shift),
                                             int(spec.major_axis == "Y"), _ptr(perm)))
        return perm

    def positional_embedding(self, coords: np.ndarray, d_model: int) -> np.ndarray:
        coords = np.ascontiguousarray(coords, np.float64)
        out = np.empty((coords.shape[0], d_model), np.float32)
        self._check(lib().fwa_b200_positional_embedding(self._h, _ptr(coords), coords.shape[0],
                                                        d_model, _ptr(out)))
        return out

    def positional_embedding_f16(self, coords: np.ndarray, d_model: int) -> np.ndarray:
        """The bf16 fast path's fp16 PE rows (fp32 range-reduced sincospi on the device)."""
        coords = np.ascontiguousarray(coords, np.float64)
        out = np.empty((coords.shape[0], d_model), np.float16)
        self._check(lib().fwa_b200_positional_embedding_f16(self._h, _ptr(coords), coords.shape[0],
                                                            d_model, _ptr(out)))
        return out

    def pillarize(self, xy: np.ndarray, feats: np.ndarray, resolution: float, weight: np.ndarray,
                  bias: Optional[np.ndarray] = None) -> "PillarSet":
        """geometry::pillarize (geometry.hpp:246-300) on the GPU."""
        xy = np.ascontiguousarray(xy, np.float64)
        feats = np.ascontiguousarray(feats, np.float64)
        weight = np.ascontiguousarray(weight, np.float64)
        n, f_in = xy.shape[0], (feats.shape[1] if feats.ndim == 2 else 0)
        d_out = weight.shape[0]
        b = None if bias is None else np.ascontiguousarray(bias, np.float64)
        np_ = C.c_int64(0)
        coords = np.empty((max(n, 1), 2), np.float64)
        out = np.empty((max(n, 1), d_out), np.float64)
        self._check(lib().fwa_b200_pillarize(self._h, _ptr(xy), _ptr(feats), n, f_in, resolution, _ptr(weight),
                                              _ptr(b), d_out, _ptr(coords), _ptr(out), C.byref(np_)))
        p = np_.value
        return PillarSet(coords[:p].copy(), out[:p].copy(), resolution)

    def pillarize_device(self, d_xy: int, d_feats: int, n: int, f_in: int, resolution: float, d_weight: int,
                         d_bias: int, d_out: int, d_coords: int, d_out_feats: int, capacity: int) -> int:
        """Device-pointer pillarize (the pillars stay in HBM for forward_device); returns P."""
        np_ = C.c_int64(0)
        self._check(lib().fwa_b200_pillarize_device(self._h, d_xy, d_feats, n, f_in, resolution, d_weight,
                                                     d_bias or None, d_out, d_coords, d_out_feats, capacity,
                                                     C.byref(np_)))
        return np_.value

    def fwa_block_backward(self, f: np.ndarray, pe: np.ndarray, record: bytes, n_groups: int,
                           grad_out: np.ndarray):
        """kernels.hpp:660-765 on the GPU: (grad_f, parameter gradients as one FWAP record)."""
        f = np.ascontiguousarray(f, np.float32)
        pe = np.ascontiguousarray(pe, np.float32)
        go = np.ascontiguousarray(grad_out, np.float32)
        gf = np.empty_like(f)
        gr = np.empty(len(record), np.uint8)
        rb = np.frombuffer(record, np.uint8)
        self._check(lib().fwa_b200_block_backward(self._h, _ptr(f), _ptr(pe), f.shape[0], n_groups, _ptr(rb),
                                                   len(record), _ptr(go), _ptr(gf), _ptr(gr)))
        return gf, gr.tobytes()

    def equal_window_forward(self, d_coords: int, d_feats: int, n: int, cfg: FwaConfig, d_out: int,
                             bucket_edges=(16, 32, 64, 128, 256)) -> dict:
        """The equal-window padded baseline (bench.hpp:266-326) on device buffers: block 0 of
        the loaded params over windows padded to their occupancy bucket's maximum."""
        e = np.ascontiguousarray(bucket_edges, np.int32)
        r = _EwReport()
        c = cfg.c()
        self._check(lib().fwa_b200_equal_window_forward(self._h, C.c_void_p(d_coords), C.c_void_p(d_feats), n,
                                                         C.byref(c), _ptr(e), len(e), C.c_void_p(d_out),
                                                         C.byref(r)))
        nb = r.n_buckets
        return {"n_windows": r.n_windows, "max_occ": r.max_occ, "min_nonzero_occ": r.min_nonzero_occ,
                "padding_factor": r.padding_factor, "rows_padded": r.rows_padded,
                "buckets": [{"edge": r.bucket_edge[b], "pad": r.bucket_pad[b], "windows": r.bucket_windows[b]}
                            for b in range(nb)]}

    def fwa_block_forward(self, f: np.ndarray, pe: np.ndarray, record: bytes, n_groups: int) -> np.ndarray:
        f = np.ascontiguousarray(f, np.float32)
        pe = np.ascontiguousarray(pe, np.float32)
        if f.shape != pe.shape:
            raise ShapeError("group_attention: pe shape mismatch")
        out = np.empty_like(f)
        buf = np.frombuffer(record, np.uint8)
        self._check(lib().fwa_b200_block_forward(self._h, _ptr(f), _ptr(pe), f.shape[0], n_groups,
                                                 _ptr(buf), len(record), _ptr(out)))
        return out


_default_ctx = {}


def default_context(device: int = 0, precision: str = "bf16") -> Context:
    key = (device, precision)
    if key not in _default_ctx:
        _default_ctx[key] = Context(device, precision=precision)
    return _default_ctx[key]


# ----------------------------------------------------------------------------- reference-shaped API

def run_backbone(pillars: PillarSet, cfg: FwaConfig, params, n_threads: int = 1, *,
                 device: int = 0, precision: str = "bf16", want_block_perms=False,
                 input_proj=None) -> BackboneOutput:
    """backbone.hpp:159-325.  `params` = FWAP bytes (n_blocks records) or an int seed
    (the seed overload, backbone.hpp:328-334: with pillar width != d_model it also draws
    the input projection).  `input_proj` = (weight d_model x f_in, bias or None), the
    optional BackboneParams::input_proj.  `n_threads` is accepted for API parity; the
    GPU path's results do not depend on it."""
    validate(cfg)
    if isinstance(params, (int, np.integer)):
        params, w = init_backbone_params_fin(cfg, int(pillars.features.shape[1]), int(params))
        if w is not None:
            input_proj = (w, None)
    ctx = default_context(device, precision)
    ctx.load_params(cfg, params)
    ctx.load_input_proj(*(input_proj or (None,)))
    return ctx.run_backbone(pillars, cfg, want_block_perms=want_block_perms)


def sort(coords: np.ndarray, spec: WindowSpec, *, device: int = 0) -> np.ndarray:
    """flatten::sort (flatten.hpp:97-120): the window-sort permutation."""
    if spec.w_x <= 0.0 or spec.w_y <= 0.0:
        raise ConfigError("window dims must be positive")
    return default_context(device).sort(coords, spec)


def group(perm: np.ndarray, g: int):
    """flatten::group (flatten.hpp:134-146): (member_indices [n_groups x g], dropped)."""
    if g < 1:
        raise ConfigError("group size must be >= 1")
    n_groups = len(perm) // g
    return perm[:n_groups * g].reshape(n_groups, g), perm[n_groups * g:]


def positional_embedding(coords: np.ndarray, d_model: int, *, device: int = 0) -> np.ndarray:
    return default_context(device).positional_embedding(coords, d_model)


def fwa_block_forward(f, pe, record: bytes, n_groups: int, *, device: int = 0, precision="bf16"):
    return default_context(device, precision).fwa_block_forward(f, pe, record, n_groups)


def init_backbone_params(cfg: FwaConfig, seed: int) -> bytes:
    """init_backbone_params(cfg, f_in=d_model, seed) as FWAP records."""
    c = cfg.c()
    n = lib().fwa_b200_init_params(C.byref(c), seed, None, 0)
    if n < 0:
        raise _ERRS.get(-n, FwaError)("init_backbone_params failed")
    buf = np.empty(n, np.uint8)
    lib().fwa_b200_init_params(C.byref(c), seed, _ptr(buf), n)
    return buf.tobytes()


def init_backbone_params_fin(cfg: FwaConfig, f_in: int, seed: int):
    """init_backbone_params(cfg, f_in, seed) (backbone.hpp:83-102): (FWAP bytes, input
    projection weight d_model x f_in or None when f_in == d_model)."""
    c = cfg.c()
    n = lib().fwa_b200_init_params_fin(C.byref(c), f_in, seed, None, 0, None)
    if n < 0:
        raise _ERRS.get(-n, FwaError)("init_backbone_params failed")
    buf = np.empty(n, np.uint8)
    w = np.empty((cfg.d_model, f_in), np.float32) if f_in != cfg.d_model else None
    r = lib().fwa_b200_init_params_fin(C.byref(c), f_in, seed, _ptr(buf), n, _ptr(w) if w is not None else None)
    if r < 0:
        raise _ERRS.get(-r, FwaError)("init_backbone_params failed")
    return buf.tobytes(), w


@dataclass
class SceneSpec:
    """geometry::SceneSpec (geometry.hpp:310-319)."""
    n_clusters: int = 0
    points_per_cluster_min: int = 1
    points_per_cluster_max: int = 1
    cluster_sigma: float = 1.0
    extent_x: float = 100.0
    extent_y: float = 100.0
    n_background: int = 0
    f_in: int = 1


# SURVEY.md §8(d) frames (seed 42): F10 9,975 / F30 30,212 / F60 60,897 / F250 255,066 pillars
SCENES = {
    "F10": SceneSpec(32, 200, 400, 2.0, 150.0, 150.0, 3200, 2),
    "F30": SceneSpec(100, 200, 400, 2.0, 150.0, 150.0, 10000, 2),
    "PINNED": SceneSpec(80, 200, 280, 1.3, 200.0, 200.0, 10000, 2),
    "F60": SceneSpec(220, 200, 400, 2.0, 150.0, 150.0, 22000, 2),
    "F100": SceneSpec(330, 200, 400, 2.0, 150.0, 150.0, 33000, 2),
    "F200": SceneSpec(660, 200, 400, 2.5, 300.0, 300.0, 66000, 2),
    "F250": SceneSpec(870, 200, 400, 2.5, 300.0, 300.0, 87000, 2),
}


def make_pillars(scene: SceneSpec, seed: int, d_out: int = 128, param_seed: Optional[int] = None,
                 resolution: float = 0.32) -> PillarSet:
    """generate_synthetic(scene, seed) -> pillarize(., resolution,
    random_pillar_params(f_in, d_out, param_seed)) — bit-identical to the reference."""
    s = _scene_c(scene)
    ps = seed if param_seed is None else param_seed
    n = lib().fwa_b200_generate_pillars(C.byref(s), seed, resolution, d_out, ps, None, None)
    if n < 0:
        raise _ERRS.get(-n, FwaError)("generate_synthetic/pillarize failed")
    coords = np.empty((n, 2), np.float64)
    feats = np.empty((n, d_out), np.float64)
    lib().fwa_b200_generate_pillars(C.byref(s), seed, resolution, d_out, ps, _ptr(coords), _ptr(feats))
    return PillarSet(coords, feats, resolution)


def _scene_c(scene: SceneSpec):
    return _Scene(scene.n_clusters, scene.points_per_cluster_min, scene.points_per_cluster_max,
                  scene.cluster_sigma, scene.extent_x, scene.extent_y, scene.n_background, scene.f_in)


def generate_points(scene: SceneSpec, seed: int):
    """generate_synthetic(scene, seed) (geometry.hpp:355-386): (xy n x 2, features n x f_in),
    bit-identical to the reference's point cloud."""
    s = _scene_c(scene)
    n = lib().fwa_b200_generate_points(C.byref(s), seed, None, None)
    if n < 0:
        raise _ERRS.get(-n, FwaError)("generate_synthetic failed")
    xy = np.empty((n, 2), np.float64)
    f = np.empty((n, scene.f_in), np.float64)
    lib().fwa_b200_generate_points(C.byref(s), seed, _ptr(xy), _ptr(f))
    return xy, f


def pillar_params(f_in: int, d_out: int, seed: int) -> np.ndarray:
    """random_pillar_params (geometry.hpp:71-79): weight d_out x f_in ~ N(0, 0.5^2), bias 0."""
    w = np.empty((d_out, f_in), np.float64)
    n = lib().fwa_b200_pillar_params(f_in, d_out, seed, _ptr(w))
    if n < 0:
        raise _ERRS.get(-n, FwaError)("random_pillar_params failed")
    return w


def fnv1a64_hex(b: bytes) -> str:
    """bench.hpp:62-72 (feature_hash / config_digest of the CLI `attend` output)."""
    return f"0x{lib().fwa_b200_fnv1a64(b, len(b)):016x}"
