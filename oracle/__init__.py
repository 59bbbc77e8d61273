"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this package.  It exposes three independent CPU oracles for the
FlatFormer backbone hot path (reference = /root/reference/proj):

* ``ref``  — the UNMODIFIED reference headers compiled in place
             (``oracle/_ref/libfwa_ref.so``, built by ``make -C oracle ref`` here;
             the .so travels to the GPU box, /root/reference does not).
* ``port`` — ``oracle/fwa_oracle.c``: a plain-C restatement of the reference
             loops in the same floating-point order (bit-exact vs ``ref``).
* ``np_sort`` — a NumPy restatement of the window sort (flatten.hpp:49-120)
             via ``np.lexsort`` over separately computed fp64 keys.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfwa_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libfwa_oracle.so")

ERR_NAMES = {1: "config_error", 2: "parse_error", 3: "schema_error", 4: "shape_error",
             5: "numeric_error", 6: "contract_error", 7: "error"}


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


class CfgC(C.Structure):
    _fields_ = [("resolution", C.c_double), ("window_px", C.c_int32), ("window_py", C.c_int32),
                ("group_size", C.c_int32), ("n_blocks", C.c_int32), ("d_model", C.c_int32),
                ("n_heads", C.c_int32), ("d_ff", C.c_int32)]


def make_cfg(resolution=0.32, window=(9, 9), group_size=69, n_blocks=8, d_model=128, n_heads=8,
             d_ff=256):
    """FwaConfig defaults (backbone.hpp:22-34)."""
    return CfgC(resolution, window[0], window[1], group_size, n_blocks, d_model, n_heads, d_ff)


def _p(a, t=C.c_void_p):
    return None if a is None else a.ctypes.data_as(t)


_ref = None
_port = None


def build(ref=True):
    """Compile the C restatement (always) and the reference shim (when the
    reference sources are present, i.e. in the build container)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_make_pillars.restype = C.c_void_p
        lib.ref_make_pillars.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_double,
                                         C.c_int, C.c_uint64, C.POINTER(C.c_int64)]
        lib.ref_pillars_get.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_pillars_free.argtypes = [C.c_void_p]
        lib.ref_generate_points.restype = C.c_int64
        lib.ref_generate_points.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                            C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_void_p,
                                            C.c_int64]
        lib.ref_config_json.restype = C.c_int64
        lib.ref_config_json.argtypes = [C.POINTER(CfgC), C.c_char_p, C.c_int64]
        lib.ref_fnv1a64_hex.argtypes = [C.c_void_p, C.c_int64, C.c_char_p]
        lib.ref_bench_summarize.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p]
        lib.ref_write_points.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_uint64, C.c_char_p, C.c_int]
        lib.ref_block_backward.restype = C.c_int64
        lib.ref_block_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p,
                                           C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        lib.ref_init_params_fwap.restype = C.c_int64
        lib.ref_init_params_fwap.argtypes = [C.POINTER(CfgC), C.c_int64, C.c_uint64, C.c_void_p,
                                             C.c_int64]
        lib.ref_zero_params_fwap.restype = C.c_int64
        lib.ref_zero_params_fwap.argtypes = [C.POINTER(CfgC), C.c_void_p, C.c_int64]
        lib.ref_run_backbone.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                         C.POINTER(CfgC), C.c_void_p, C.c_int64, C.c_int,
                                         C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_run_backbone_seeded.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                                C.POINTER(CfgC), C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                                C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p]
        lib.ref_block_plans.argtypes = [C.c_void_p, C.c_int64, C.POINTER(CfgC), C.c_void_p,
                                        C.c_void_p]
        for fn in (lib.ref_sort, lib.ref_oracle_sort):
            fn.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_int,
                           C.c_void_p]
        lib.ref_sort_key.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                     C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_positional_embedding.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        lib.ref_block_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                          C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        lib.ref_oracle_block.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                         C.c_void_p, C.c_int64, C.c_void_p]
        _ref = lib
    return _ref


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = C.CDLL(PORT_SO)
        lib.orc_sort.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_int,
                                 C.c_void_p]
        lib.orc_positional_embedding.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        lib.orc_block_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p,
                                          C.c_int64, C.c_void_p]
        lib.orc_run_backbone.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(CfgC),
                                         C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        _port = lib
    return _port


def _check_ref(rc):
    if rc != 0:
        raise OracleError(rc, ref().ref_last_error().decode())


# ----------------------------------------------------------------------------- reference (_ref)

def ref_make_pillars(scene, seed, d_out=128, param_seed=None, resolution=0.32):
    """generate_synthetic + pillarize(random_pillar_params(f_in, d_out, param_seed))."""
    lib = ref()
    n = C.c_int64()
    h = lib.ref_make_pillars(scene["n_clusters"], scene["ppc_min"], scene["ppc_max"],
                             scene["sigma"], scene["ext_x"], scene["ext_y"], scene["n_bg"],
                             scene["f_in"], seed, resolution, d_out,
                             seed if param_seed is None else param_seed, C.byref(n))
    if not h:
        raise OracleError(-n.value, lib.ref_last_error().decode())
    coords = np.empty((n.value, 2), np.float64)
    feats = np.empty((n.value, d_out), np.float64)
    lib.ref_pillars_get(h, _p(coords), _p(feats))
    lib.ref_pillars_free(h)
    return coords, feats


def ref_init_params(cfg, f_in, seed):
    lib = ref()
    n = lib.ref_init_params_fwap(C.byref(cfg), f_in, seed, None, 0)
    if n < 0:
        raise OracleError(-n, lib.ref_last_error().decode())
    buf = np.empty(n, np.uint8)
    lib.ref_init_params_fwap(C.byref(cfg), f_in, seed, _p(buf), n)
    return buf.tobytes()


def ref_zero_params(cfg):
    lib = ref()
    n = lib.ref_zero_params_fwap(C.byref(cfg), None, 0)
    buf = np.empty(n, np.uint8)
    lib.ref_zero_params_fwap(C.byref(cfg), _p(buf), n)
    return buf.tobytes()


def ref_run_backbone(coords, feats64, cfg, blob, n_threads=1):
    lib = ref()
    coords = np.ascontiguousarray(coords, np.float64)
    feats64 = np.ascontiguousarray(feats64, np.float64)
    n, d_in = feats64.shape
    out = np.empty((n, cfg.d_model), np.float32)
    kept = np.empty(n, np.int32)
    dropped = np.empty(n, np.int32)
    dpb = np.empty(cfg.n_blocks, np.int32)
    cache = np.empty(2, np.int32)
    stages = np.empty(6, np.float64)
    nk = C.c_int64()
    bb = np.frombuffer(blob, np.uint8)
    _check_ref(lib.ref_run_backbone(_p(coords), _p(feats64), n, d_in, C.byref(cfg), _p(bb),
                                    len(blob), n_threads, _p(out), _p(kept), C.byref(nk),
                                    _p(dropped), _p(dpb), _p(cache), _p(stages)))
    k = nk.value
    return dict(features=out[:k].copy(), kept=kept[:k].copy(),
                dropped=dropped[:int(dpb.sum())].copy(), dropped_per_block=dpb,
                cache=(int(cache[0]), int(cache[1])), stage_ms=stages)


def ref_run_backbone_seeded(coords, feats64, cfg, seed, n_threads=1):
    """The seed overload run_backbone(ps, cfg, seed) (backbone.hpp:328-334): draws the input
    projection when the pillar width != d_model.  Returns the outputs + that weight."""
    lib = ref()
    coords = np.ascontiguousarray(coords, np.float64)
    feats64 = np.ascontiguousarray(feats64, np.float64)
    n, d_in = feats64.shape
    out = np.empty((n, cfg.d_model), np.float32)
    kept = np.empty(n, np.int32)
    dropped = np.empty(n, np.int32)
    dpb = np.empty(cfg.n_blocks, np.int32)
    cache = np.empty(2, np.int32)
    w = np.zeros((cfg.d_model, d_in), np.float32)
    nk = C.c_int64()
    _check_ref(lib.ref_run_backbone_seeded(_p(coords), _p(feats64), n, d_in, C.byref(cfg), seed, n_threads,
                                           _p(out), _p(kept), C.byref(nk), _p(dropped), _p(dpb), _p(cache), _p(w)))
    k = nk.value
    return dict(features=out[:k].copy(), kept=kept[:k].copy(), dropped=dropped[:int(dpb.sum())].copy(),
                dropped_per_block=dpb, cache=(int(cache[0]), int(cache[1])), proj_weight=w)


def ref_block_plans(coords, cfg):
    lib = ref()
    coords = np.ascontiguousarray(coords, np.float64)
    n = coords.shape[0]
    perms = np.full((cfg.n_blocks, n), -1, np.int32)
    n_act = np.empty(cfg.n_blocks, np.int32)
    _check_ref(lib.ref_block_plans(_p(coords), n, C.byref(cfg), _p(perms), _p(n_act)))
    return [perms[b, :n_act[b]].copy() for b in range(cfg.n_blocks)]


def ref_sort(coords, w_x, w_y, shift, axis_y, brute=False):
    lib = ref()
    coords = np.ascontiguousarray(coords, np.float64)
    perm = np.empty(coords.shape[0], np.int32)
    fn = lib.ref_oracle_sort if brute else lib.ref_sort
    _check_ref(fn(_p(coords), coords.shape[0], w_x, w_y, int(shift), int(axis_y), _p(perm)))
    return perm


def ref_sort_key(x, y, w_x, w_y, shift, axis_y):
    win = np.empty(2, np.int64)
    loc = np.empty(2, np.float64)
    ref().ref_sort_key(x, y, w_x, w_y, int(shift), int(axis_y), _p(win), _p(loc))
    return (int(win[0]), int(win[1]), float(loc[0]), float(loc[1]))


def ref_positional_embedding(coords, d):
    coords = np.ascontiguousarray(coords, np.float64)
    out = np.empty((coords.shape[0], d), np.float32)
    _check_ref(ref().ref_positional_embedding(_p(coords), coords.shape[0], d, _p(out)))
    return out


def ref_block_forward(f, pe, n_groups, record, n_threads=1):
    f = np.ascontiguousarray(f, np.float32)
    pe = np.ascontiguousarray(pe, np.float32)
    out = np.empty_like(f)
    bb = np.frombuffer(record, np.uint8)
    _check_ref(ref().ref_block_forward(_p(f), _p(pe), f.shape[0], f.shape[1], n_groups, _p(bb),
                                       len(record), n_threads, _p(out)))
    return out


def ref_oracle_block(f, pe, n_groups, record):
    f = np.ascontiguousarray(f, np.float64)
    pe = np.ascontiguousarray(pe, np.float64)
    out = np.empty_like(f)
    bb = np.frombuffer(record, np.uint8)
    _check_ref(ref().ref_oracle_block(_p(f), _p(pe), f.shape[0], f.shape[1], n_groups, _p(bb),
                                      len(record), _p(out)))
    return out


# ----------------------------------------------------------------------------- C restatement

def port_sort(coords, w_x, w_y, shift, axis_y):
    coords = np.ascontiguousarray(coords, np.float64)
    perm = np.empty(coords.shape[0], np.int32)
    rc = port().orc_sort(_p(coords), coords.shape[0], w_x, w_y, int(shift), int(axis_y), _p(perm))
    if rc:
        raise OracleError(rc)
    return perm


def port_positional_embedding(coords, d):
    coords = np.ascontiguousarray(coords, np.float64)
    out = np.empty((coords.shape[0], d), np.float32)
    rc = port().orc_positional_embedding(_p(coords), coords.shape[0], d, _p(out))
    if rc:
        raise OracleError(rc)
    return out


def port_block_forward(f, pe, n_groups, record):
    f = np.ascontiguousarray(f, np.float32)
    pe = np.ascontiguousarray(pe, np.float32)
    out = np.empty_like(f)
    bb = np.frombuffer(record, np.uint8)
    rc = port().orc_block_forward(_p(f), _p(pe), f.shape[0], n_groups, _p(bb), len(record),
                                  _p(out))
    if rc:
        raise OracleError(rc)
    return out


def port_run_backbone(coords, feats32, cfg, blob, want_perms=False):
    coords = np.ascontiguousarray(coords, np.float64)
    feats32 = np.ascontiguousarray(feats32, np.float32)
    n = coords.shape[0]
    out = np.empty((n, cfg.d_model), np.float32)
    kept = np.empty(n, np.int32)
    dropped = np.empty(n, np.int32)
    dpb = np.zeros(cfg.n_blocks, np.int32)
    cache = np.empty(2, np.int32)
    perms = np.full((cfg.n_blocks, n), -1, np.int32) if want_perms else None
    nk = C.c_int64()
    bb = np.frombuffer(blob, np.uint8)
    rc = port().orc_run_backbone(_p(coords), _p(feats32), n, C.byref(cfg), _p(bb), len(blob),
                                 _p(out), _p(kept), C.byref(nk), _p(dropped), _p(dpb), _p(cache),
                                 _p(perms))
    if rc:
        raise OracleError(rc)
    k = nk.value
    res = dict(features=out[:k].copy(), kept=kept[:k].copy(),
               dropped=dropped[:int(dpb.sum())].copy(), dropped_per_block=dpb,
               cache=(int(cache[0]), int(cache[1])))
    if want_perms:
        res["block_perms"] = perms
    return res


# ----------------------------------------------------------------------------- NumPy restatement

def np_sort_keys(coords, w_x, w_y, shift, axis_y):
    """flatten.hpp:49-69 in vectorised fp64 (each op separately rounded)."""
    c = np.asarray(coords, np.float64)
    cx, cy = c[:, 0].copy(), c[:, 1].copy()
    if shift:
        cx = cx + w_x / 2.0
        cy = cy + w_y / 2.0
    cm, cn = (cy, cx) if axis_y else (cx, cy)
    wm, wn = (w_y, w_x) if axis_y else (w_x, w_y)
    win_m = np.floor(cm / wm).astype(np.int64)
    win_n = np.floor(cn / wn).astype(np.int64)
    loc_m = cm - win_m.astype(np.float64) * wm
    loc_n = cn - win_n.astype(np.float64) * wn
    return win_m, win_n, loc_m, loc_n


def np_sort(coords, w_x, w_y, shift, axis_y):
    """flatten.hpp:97-120 — lexsort is stable, so index order breaks ties."""
    wm, wn, lm, ln = np_sort_keys(coords, w_x, w_y, shift, axis_y)
    # -0.0 == +0.0 for the comparator; lexsort on floats already treats them equal.
    return np.lexsort((ln, lm, wn, wm)).astype(np.int32)


def max_rel_err(got, want):
    """Normwise error of the reference tests (tests/test_kernels.cpp:25-33)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want)) / max(float(np.max(np.abs(want))), 1e-30))


def _pairwise_sum(v):
    """dense.hpp:84-94: <= 8 values summed left to right from 0.0, else the two halves."""
    if len(v) <= 8:
        s = 0.0
        for x in v:
            s += x
        return s
    h = len(v) // 2
    return _pairwise_sum(v[:h]) + _pairwise_sum(v[h:])


def np_pillarize(xy, feats, resolution, weight, bias=None):
    """Pure-Python restatement of geometry::pillarize (geometry.hpp:246-300) for small
    clouds: cells (floor(x / res), floor(y / res)) in lexicographic order (std::map),
    members in ingestion order, pairwise mean pooling, gelu(bias + W pooled) in fp64
    with libm erf (math.erf), coords (cell + 0.5) * res.  Returns (coords, features)."""
    import math
    xy = np.asarray(xy, np.float64)
    feats = np.asarray(feats, np.float64).reshape(xy.shape[0], -1)
    weight = np.asarray(weight, np.float64)
    d_out, f_in = weight.shape
    cells = {}
    for i in range(xy.shape[0]):
        key = (int(math.floor(xy[i, 0] / resolution)), int(math.floor(xy[i, 1] / resolution)))
        cells.setdefault(key, []).append(i)
    coords, out = [], []
    for key in sorted(cells):
        mem = cells[key]
        pooled = [_pairwise_sum([float(feats[m, c]) for m in mem]) / float(len(mem)) for c in range(f_in)]
        row = []
        for o in range(d_out):
            acc = 0.0 if bias is None else float(bias[o])
            for c in range(f_in):
                acc += float(weight[o, c]) * pooled[c]
            row.append(0.5 * acc * (1.0 + math.erf(acc / 1.4142135623730951)))
        out.append(row)
        coords.append(((key[0] + 0.5) * resolution, (key[1] + 0.5) * resolution))
    return (np.array(coords, np.float64).reshape(-1, 2), np.array(out, np.float64).reshape(-1, d_out))


def ref_config_json(cfg):
    """nlohmann::json(FwaConfig).dump() of the reference (backbone.hpp:49-57)."""
    buf = C.create_string_buffer(4096)
    n = ref().ref_config_json(C.byref(cfg), buf, 4096)
    _check_ref(0 if n >= 0 else -n)
    return buf.value.decode()


def ref_bench_summarize(samples, runs, warmup):
    """bench::summarize (bench.hpp:124-143): (mean, p50, p95, outliers_excluded)."""
    v = np.ascontiguousarray(samples, np.float64)
    out = np.zeros(4, np.float64)
    _check_ref(ref().ref_bench_summarize(_p(v), v.size, runs, warmup, _p(out)))
    return float(out[0]), float(out[1]), float(out[2]), int(out[3])


def ref_fnv1a64_hex(b: bytes) -> str:
    """bench.hpp:62-72."""
    out = C.create_string_buffer(32)
    ref().ref_fnv1a64_hex(b, len(b), out)
    return out.value.decode()


def ref_write_points(scene, seed, path, binary):
    """generate_synthetic + write_binary / write_csv (geometry.hpp:202-237)."""
    _check_ref(ref().ref_write_points(scene["n_clusters"], scene["ppc_min"], scene["ppc_max"], scene["sigma"],
                                      scene["ext_x"], scene["ext_y"], scene["n_bg"], scene["f_in"], seed,
                                      path.encode(), int(binary)))


def np_equal_window_forward(coords, feats32, record, w_x, w_y, edges=(16, 32, 64, 128, 256)):
    """bench_equal_window (bench.hpp:266-326) computed: windows of
    partition_equal_window (workload.hpp:44-68: floor(x / w_x), floor(y / w_y),
    lexicographic, members in ingestion order), bucketed by occupancy, padded with zero
    feature / zero PE rows to the bucket's largest occupancy, then the reference block
    (port) per bucket.  Returns the real rows' outputs in input order."""
    c = np.asarray(coords, np.float64)
    f = np.asarray(feats32, np.float32)
    n, d = f.shape
    wm, wn, _, _ = np_sort_keys(c, w_x, w_y, 0, 0)
    order = np.lexsort((np.arange(n), wn, wm))
    key = np.stack([wm[order], wn[order]], 1)
    starts = np.flatnonzero(np.r_[True, np.any(key[1:] != key[:-1], axis=1)])
    ends = np.r_[starts[1:], n]
    occ = ends - starts
    bucket = np.searchsorted(np.asarray(edges), occ, side="left")
    pe = port_positional_embedding(c, d)
    out = np.zeros_like(f)
    for b in range(len(edges)):
        wins = np.flatnonzero(bucket == b)
        if wins.size == 0:
            continue
        pad = int(occ[wins].max())
        bf = np.zeros((wins.size * pad, d), np.float32)
        bp = np.zeros_like(bf)
        ids = []
        for j, w in enumerate(wins):
            mem = order[starts[w]:ends[w]]
            bf[j * pad:j * pad + mem.size] = f[mem]
            bp[j * pad:j * pad + mem.size] = pe[mem]
            ids.append((j * pad, mem))
        o = port_block_forward(bf, bp, wins.size, record)
        for r0, mem in ids:
            out[mem] = o[r0:r0 + mem.size]
    return out


def ref_block_backward(f, pe, n_groups, record, grad_out):
    """fwa_block_forward (cached) + fwa_block_backward (kernels.hpp:636-765) of the
    reference: (grad_f rows x d, parameter gradients as one FWAP record)."""
    f = np.ascontiguousarray(f, np.float32)
    pe = np.ascontiguousarray(pe, np.float32)
    g = np.ascontiguousarray(grad_out, np.float32)
    gf = np.empty_like(f)
    out = np.empty(len(record), np.uint8)
    bb = np.frombuffer(record, np.uint8)
    n = ref().ref_block_backward(_p(f), _p(pe), f.shape[0], f.shape[1], n_groups, _p(bb), len(record), _p(g),
                                 _p(gf), _p(out), len(record))
    _check_ref(0 if n >= 0 else -n)
    return gf, out[:n].tobytes()
