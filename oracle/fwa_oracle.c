/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path, used
 * as the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Never linked into, or called by, the product library.
 *
 * Plain C restatement of FlatFormer's flattened-window-attention backbone
 * forward as implemented by the reference (paths relative to
 * /root/reference/proj).  Every floating-point operation is written in the same
 * order as the reference's scalar loops so that, compiled with
 * -ffp-contract=off, results are bit-identical to the reference's own build
 * (pinned in tests/test_oracle.py against oracle/_ref and tests/golden/).
 *
 *   orc_sort_key            include/fwa/flatten.hpp:49-69   (make_sort_key)
 *   orc_key_less            include/fwa/flatten.hpp:41-47   (key_less)
 *   orc_sort                include/fwa/flatten.hpp:97-120  (sort, no cache)
 *   orc_positional_embedding include/fwa/kernels.hpp:364-393
 *   orc_block_forward       include/fwa/kernels.hpp:447-650 (group_attention_forward
 *                           + ffn_forward, normalize_row 235-249, softmax_row 251-262,
 *                           matmul_nt dense.hpp:50-64, gelu dense.hpp:67-72)
 *   orc_run_backbone        include/fwa/backbone.hpp:159-325 (block loop, plan cache,
 *                           drop bookkeeping, active-order output)
 *
 * Parameters are taken as FWAP records (kernels.hpp:149-206): magic "FWAP",
 * u32 D, u32 H, u32 D_ff, then 12 f32 tensors in AttnParams field order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_CONFIG 1
#define ORC_ERR_PARSE 2
#define ORC_ERR_SHAPE 4
#define ORC_ERR_NUMERIC 5

typedef struct {
    int64_t win_major, win_minor;
    double loc_major, loc_minor;
    int32_t idx;
} orc_key;

/* flatten.hpp:49-69 */
void orc_sort_key(double x, double y, double w_x, double w_y, int shift, int axis_y, int32_t idx,
                  orc_key* k) {
    double cx = x, cy = y;
    if (shift) {
        cx += w_x / 2.0;
        cy += w_y / 2.0;
    }
    const double cm = axis_y ? cy : cx, cn = axis_y ? cx : cy;
    const double wm = axis_y ? w_y : w_x, wn = axis_y ? w_x : w_y;
    k->win_major = (int64_t)floor(cm / wm);
    k->win_minor = (int64_t)floor(cn / wn);
    k->loc_major = cm - (double)k->win_major * wm;
    k->loc_minor = cn - (double)k->win_minor * wn;
    k->idx = idx;
}

/* flatten.hpp:41-47 */
static int orc_key_less(const orc_key* a, const orc_key* b) {
    if (a->win_major != b->win_major) return a->win_major < b->win_major;
    if (a->win_minor != b->win_minor) return a->win_minor < b->win_minor;
    if (a->loc_major != b->loc_major) return a->loc_major < b->loc_major;
    if (a->loc_minor != b->loc_minor) return a->loc_minor < b->loc_minor;
    return a->idx < b->idx;
}

static void merge_sort(int32_t* a, int32_t* tmp, int64_t n, const orc_key* keys) {
    if (n < 2) return;
    const int64_t h = n / 2;
    merge_sort(a, tmp, h, keys);
    merge_sort(a + h, tmp, n - h, keys);
    int64_t i = 0, j = h, w = 0;
    while (i < h && j < n) {
        if (orc_key_less(&keys[a[j]], &keys[a[i]])) tmp[w++] = a[j++];
        else tmp[w++] = a[i++];
    }
    while (i < h) tmp[w++] = a[i++];
    while (j < n) tmp[w++] = a[j++];
    memcpy(a, tmp, (size_t)n * sizeof(int32_t));
}

/* flatten.hpp:97-120: the key order is total (ends in orig index), so any
 * correct comparison sort yields the reference's permutation. */
int orc_sort(const double* coords, int64_t n, double w_x, double w_y, int shift, int axis_y,
             int32_t* perm) {
    if (w_x <= 0.0 || w_y <= 0.0) return ORC_ERR_CONFIG;
    orc_key* keys = (orc_key*)malloc(sizeof(orc_key) * (size_t)(n ? n : 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        orc_sort_key(coords[2 * i], coords[2 * i + 1], w_x, w_y, shift, axis_y, (int32_t)i, &keys[i]);
        perm[i] = (int32_t)i;
    }
    merge_sort(perm, tmp, n, keys);
    free(keys);
    free(tmp);
    return ORC_OK;
}

/* kernels.hpp:364-393 */
int orc_positional_embedding(const double* coords, int64_t n, int d, float* out) {
    if (d < 4 || d % 4 != 0) return ORC_ERR_CONFIG;
    const int nf = d / 4;
    double* freq = (double*)malloc(sizeof(double) * (size_t)nf);
    const double f_min = 1.0 / 10000.0, f_max = 1.0;
    for (int k = 0; k < nf; ++k)
        freq[k] = nf == 1 ? f_min : f_min * pow(f_max / f_min, (double)k / (double)(nf - 1));
    for (int64_t i = 0; i < n; ++i) {
        float* row = out + i * d;
        for (int axis = 0; axis < 2; ++axis) {
            const double c = coords[2 * i + axis];
            float* blk = row + axis * (d / 2);
            for (int k = 0; k < nf; ++k) {
                const double phase = 6.283185307179586 * freq[k] * c;
                blk[2 * k] = (float)sin(phase);
                blk[2 * k + 1] = (float)cos(phase);
            }
        }
    }
    free(freq);
    return ORC_OK;
}

/* One FWAP record (kernels.hpp:149-206), tensors pointing into the blob. */
typedef struct {
    int d, h, dff;
    const float *w_qkv, *b_qkv, *w_out, *b_out, *ln1_g, *ln1_b, *ln2_g, *ln2_b, *w1, *b1, *w2, *b2;
} orc_params;

static int64_t parse_record(const uint8_t* p, int64_t len, orc_params* o) {
    if (len < 16 || memcmp(p, "FWAP", 4) != 0) return -1;
    uint32_t d, h, f;
    memcpy(&d, p + 4, 4);
    memcpy(&h, p + 8, 4);
    memcpy(&f, p + 12, 4);
    const int64_t nfl = 3LL * d * d + 3LL * d + (int64_t)d * d + d + 4LL * d + (int64_t)f * d + f +
                        (int64_t)d * f + d;
    if (len < 16 + 4 * nfl) return -1;
    const float* t = (const float*)(p + 16);
    o->d = (int)d;
    o->h = (int)h;
    o->dff = (int)f;
    o->w_qkv = t; t += 3LL * d * d;
    o->b_qkv = t; t += 3LL * d;
    o->w_out = t; t += (int64_t)d * d;
    o->b_out = t; t += d;
    o->ln1_g = t; t += d;
    o->ln1_b = t; t += d;
    o->ln2_g = t; t += d;
    o->ln2_b = t; t += d;
    o->w1 = t; t += (int64_t)f * d;
    o->b1 = t; t += f;
    o->w2 = t; t += (int64_t)d * f;
    o->b2 = t;
    return 16 + 4 * nfl;
}

/* kernels.hpp:235-249 */
static float normalize_row(const float* x, int n, float* xhat) {
    float mean = 0.0f;
    for (int i = 0; i < n; ++i) mean += x[i];
    mean /= (float)n;
    float var = 0.0f;
    for (int i = 0; i < n; ++i) {
        const float dd = x[i] - mean;
        var += dd * dd;
    }
    var /= (float)n;
    const float inv_std = 1.0f / sqrtf(var + (float)1e-5);
    for (int i = 0; i < n; ++i) xhat[i] = (x[i] - mean) * inv_std;
    return inv_std;
}

/* dense.hpp:67-72 */
static float gelu_f(float x) {
    return 0.5f * x * (1.0f + (float)erf((double)x / 1.4142135623730951));
}

static int all_finite(const float* a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite((double)a[i])) return 0;
    return 1;
}

/* kernels.hpp:447-570 then 575-633 (fwa_block_forward 636-650). */
static int block_forward(const float* f, const float* pe, int64_t rows, int n_groups,
                         const orc_params* p, float* out) {
    const int d = p->d, dff = p->dff, heads = p->h;
    if (d < 1 || heads < 1 || dff < 1) return ORC_ERR_CONFIG;
    if (d % heads) return ORC_ERR_CONFIG;
    if (n_groups == 0 && rows == 0) return ORC_OK;
    if (n_groups < 1 || rows % n_groups) return ORC_ERR_SHAPE;
    if (!all_finite(f, rows * d) || !all_finite(pe, rows * d)) return ORC_ERR_NUMERIC;
    const int64_t gs = rows / n_groups;
    const int hd = d / heads;
    const float scale = 1.0f / (float)sqrt((double)hd);

    float* h = (float*)malloc(sizeof(float) * (size_t)(rows * d));
    float* q = (float*)malloc(sizeof(float) * (size_t)(rows * d));
    float* k = (float*)malloc(sizeof(float) * (size_t)(rows * d));
    float* v = (float*)malloc(sizeof(float) * (size_t)(rows * d));
    float* cat = (float*)calloc((size_t)(rows * d), sizeof(float));
    float* mid = (float*)malloc(sizeof(float) * (size_t)(rows * d));
    float* logits = (float*)malloc(sizeof(float) * (size_t)gs);
    float* xhat = (float*)malloc(sizeof(float) * (size_t)d);
    float* ln = (float*)malloc(sizeof(float) * (size_t)d);
    float* act = (float*)malloc(sizeof(float) * (size_t)dff);

    for (int64_t r = 0; r < rows; ++r) normalize_row(f + r * d, d, h + r * d);
    for (int64_t r = 0; r < rows; ++r)
        for (int i = 0; i < d; ++i)
            h[r * d + i] = p->ln1_g[i] * h[r * d + i] + p->ln1_b[i] + pe[r * d + i];

    /* packed QKV: matmul_nt (k innermost) then + bias split (kernels.hpp:488-500) */
    for (int64_t r = 0; r < rows; ++r) {
        const float* hr = h + r * d;
        for (int j = 0; j < 3 * d; ++j) {
            const float* wj = p->w_qkv + (int64_t)j * d;
            float acc = 0.0f;
            for (int c = 0; c < d; ++c) acc += hr[c] * wj[c];
            if (j < d) q[r * d + j] = acc + p->b_qkv[j];
            else if (j < 2 * d) k[r * d + (j - d)] = acc + p->b_qkv[j];
            else v[r * d + (j - 2 * d)] = acc + p->b_qkv[j];
        }
    }

    for (int64_t g = 0; g < n_groups; ++g) {
        const int64_t base = g * gs;
        for (int head = 0; head < heads; ++head) {
            const int off = head * hd;
            for (int64_t i = 0; i < gs; ++i) {
                const float* qi = q + (base + i) * d + off;
                for (int64_t j = 0; j < gs; ++j) {
                    const float* kj = k + (base + j) * d + off;
                    float acc = 0.0f;
                    for (int c = 0; c < hd; ++c) acc += qi[c] * kj[c];
                    logits[j] = acc * scale;
                }
                float mx = logits[0];
                for (int64_t j = 1; j < gs; ++j) mx = logits[j] > mx ? logits[j] : mx;
                float sum = 0.0f;
                for (int64_t j = 0; j < gs; ++j) {
                    logits[j] = expf(logits[j] - mx);
                    sum += logits[j];
                }
                const float inv = 1.0f / sum;
                for (int64_t j = 0; j < gs; ++j) logits[j] *= inv;
                float* oi = cat + (base + i) * d + off;
                for (int c = 0; c < hd; ++c) oi[c] = 0.0f;
                for (int64_t j = 0; j < gs; ++j) {
                    const float w = logits[j];
                    const float* vj = v + (base + j) * d + off;
                    for (int c = 0; c < hd; ++c) oi[c] += w * vj[c];
                }
            }
        }
    }

    /* out-proj + residual (kernels.hpp:550-560): o = f + proj + b_out */
    for (int64_t r = 0; r < rows; ++r) {
        const float* cr = cat + r * d;
        for (int j = 0; j < d; ++j) {
            const float* wj = p->w_out + (int64_t)j * d;
            float acc = 0.0f;
            for (int c = 0; c < d; ++c) acc += cr[c] * wj[c];
            mid[r * d + j] = f[r * d + j] + acc + p->b_out[j];
        }
    }

    /* ffn_forward (kernels.hpp:595-623) */
    for (int64_t r = 0; r < rows; ++r) {
        normalize_row(mid + r * d, d, xhat);
        for (int i = 0; i < d; ++i) ln[i] = p->ln2_g[i] * xhat[i] + p->ln2_b[i];
        for (int j = 0; j < dff; ++j) {
            const float* w = p->w1 + (int64_t)j * d;
            float acc = p->b1[j];
            for (int i = 0; i < d; ++i) acc += w[i] * ln[i];
            act[j] = gelu_f(acc);
        }
        for (int i = 0; i < d; ++i) {
            const float* w = p->w2 + (int64_t)i * dff;
            float acc = p->b2[i];
            for (int j = 0; j < dff; ++j) acc += w[j] * act[j];
            out[r * d + i] = mid[r * d + i] + acc;
        }
    }
    free(h); free(q); free(k); free(v); free(cat); free(mid);
    free(logits); free(xhat); free(ln); free(act);
    return ORC_OK;
}

int orc_block_forward(const float* f, const float* pe, int64_t rows, int n_groups,
                      const void* blob, int64_t blob_len, float* out) {
    orc_params p;
    if (parse_record((const uint8_t*)blob, blob_len, &p) < 0) return ORC_ERR_PARSE;
    return block_forward(f, pe, rows, n_groups, &p, out);
}

typedef struct {
    double resolution;
    int32_t window_px, window_py, group_size, n_blocks, d_model, n_heads, d_ff;
} orc_config;

/* backbone.hpp:159-325.  feats are the caller's f32 cast of PillarSet
 * features (backbone.hpp:195-196).  Outputs: features n_kept x D (active
 * order), kept ids, dropped ids (per block, concatenated in tail order),
 * dropped_per_block[n_blocks], cache[2] = {computed, hits}; optional
 * block_perms (n_blocks x n, local indices). */
int orc_run_backbone(const double* coords, const float* feats, int64_t n, const orc_config* c,
                     const void* blob, int64_t blob_len, float* out_feats, int32_t* out_kept,
                     int64_t* out_n_kept, int32_t* out_dropped, int32_t* out_dropped_per_block,
                     int32_t* out_cache, int32_t* block_perms) {
    if (c->resolution <= 0.0 || c->window_px < 1 || c->window_py < 1 || c->group_size < 1 ||
        c->n_blocks < 1 || c->d_model < 4 || c->d_model % 4 || c->n_heads < 1 ||
        c->d_model % c->n_heads || c->d_ff < 1)
        return ORC_ERR_CONFIG;
    const int d = c->d_model, G = c->group_size, nb = c->n_blocks;
    orc_params* params = (orc_params*)malloc(sizeof(orc_params) * (size_t)nb);
    const uint8_t* bp = (const uint8_t*)blob;
    int64_t left = blob_len;
    for (int b = 0; b < nb; ++b) {
        const int64_t used = parse_record(bp, left, &params[b]);
        if (used < 0) { free(params); return ORC_ERR_CONFIG; }
        if (params[b].d != d || params[b].h != c->n_heads || params[b].dff != c->d_ff) {
            free(params);
            return ORC_ERR_CONFIG;
        }
        bp += used;
        left -= used;
    }
    if (left != 0) { free(params); return ORC_ERR_CONFIG; }

    const double w_x = c->window_px * c->resolution, w_y = c->window_py * c->resolution;
    float* x = (float*)malloc(sizeof(float) * (size_t)(n * d));
    memcpy(x, feats, sizeof(float) * (size_t)(n * d));
    float* pe_all = (float*)malloc(sizeof(float) * (size_t)(n * d));
    orc_positional_embedding(coords, n, d, pe_all);
    int32_t* active = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    double* cur = (double*)malloc(sizeof(double) * (size_t)(2 * n));
    for (int64_t i = 0; i < n; ++i) active[i] = (int32_t)i;
    memcpy(cur, coords, sizeof(double) * (size_t)(2 * n));
    int64_t n_active = n;

    /* plan cache keyed by (axis==X, shift) (backbone.hpp:211, 224-234) */
    int32_t* cache_perm[4] = {0, 0, 0, 0};
    int64_t cache_n[4] = {0, 0, 0, 0};
    int computed = 0, hits = 0, rc = ORC_OK;
    int64_t n_dropped_total = 0;
    float* gath = (float*)malloc(sizeof(float) * (size_t)(n * d));
    float* pe = (float*)malloc(sizeof(float) * (size_t)(n * d));
    float* outb = (float*)malloc(sizeof(float) * (size_t)(n * d));

    for (int b = 0; b < nb && rc == ORC_OK; ++b) {
        const int axis_y = (b % 4) >= 2, shift = (b % 2) == 1; /* flatten.hpp:150-161 */
        if (n_active < G) { rc = ORC_ERR_NUMERIC; break; }
        const int slot = (axis_y ? 0 : 2) + shift;
        int32_t* perm;
        if (cache_perm[slot] && cache_n[slot] == n_active) {
            ++hits;
            perm = cache_perm[slot];
        } else {
            perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_active);
            orc_sort(cur, n_active, w_x, w_y, shift, axis_y, perm);
            ++computed;
            cache_perm[slot] = perm;
            cache_n[slot] = n_active;
        }
        if (block_perms) memcpy(block_perms + (int64_t)b * n, perm, sizeof(int32_t) * (size_t)n_active);
        const int64_t n_groups = n_active / G, rows = n_groups * G, n_drop = n_active - rows;
        for (int64_t r = 0; r < rows; ++r) {
            memcpy(gath + r * d, x + (int64_t)perm[r] * d, sizeof(float) * (size_t)d);
            memcpy(pe + r * d, pe_all + (int64_t)active[perm[r]] * d, sizeof(float) * (size_t)d);
        }
        rc = block_forward(gath, pe, rows, (int)n_groups, &params[b], outb);
        if (rc) break;
        for (int64_t r = 0; r < rows; ++r)
            memcpy(x + (int64_t)perm[r] * d, outb + r * d, sizeof(float) * (size_t)d);
        out_dropped_per_block[b] = (int32_t)n_drop;
        for (int64_t t = rows; t < n_active; ++t) out_dropped[n_dropped_total++] = active[perm[t]];
        if (n_drop) {
            uint8_t* keep = (uint8_t*)malloc((size_t)n_active);
            memset(keep, 1, (size_t)n_active);
            for (int64_t t = rows; t < n_active; ++t) keep[perm[t]] = 0;
            int64_t w = 0;
            for (int64_t i = 0; i < n_active; ++i) {
                if (!keep[i]) continue;
                active[w] = active[i];
                cur[2 * w] = cur[2 * i];
                cur[2 * w + 1] = cur[2 * i + 1];
                if (w != i) memcpy(x + w * d, x + i * d, sizeof(float) * (size_t)d);
                ++w;
            }
            n_active = w;
            free(keep);
            for (int s = 0; s < 4; ++s) { free(cache_perm[s]); cache_perm[s] = 0; }
        }
    }
    if (rc == ORC_OK) {
        memcpy(out_feats, x, sizeof(float) * (size_t)(n_active * d));
        memcpy(out_kept, active, sizeof(int32_t) * (size_t)n_active);
        *out_n_kept = n_active;
        out_cache[0] = computed;
        out_cache[1] = hits;
    }
    for (int s = 0; s < 4; ++s) free(cache_perm[s]);
    free(params); free(x); free(pe_all); free(active); free(cur);
    free(gath); free(pe); free(outb);
    return rc;
}
