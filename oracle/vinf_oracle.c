/* CPU restatement of the reference temporal-block path — TEST INFRASTRUCTURE ONLY.
 * See vinf_oracle.h for the contract and how it is pinned. Each function cites
 * the reference file:line it restates (paths relative to /root/reference/proj).
 * Loop order and f64/f32 conversions follow the reference so that results are
 * bitwise-identical to it on the same host (checked in tests/test_oracle.py). */
#include "vinf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ECONFIG 1
#define ORC_ERANGE 2

/* ---- rng.hpp ------------------------------------------------------------ */

uint64_t orc_splitmix_next(uint64_t* state) { /* rng.hpp:14-19 */
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

float orc_next_unit(uint64_t* state) { /* rng.hpp:23-26: exact in binary32 */
    const uint64_t top24 = orc_splitmix_next(state) >> 40;
    return (float)top24 * (2.0f / 16777216.0f) - 1.0f;
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) { /* rng.hpp:34-37 */
    uint64_t s = seed ^ (salt * 0xD1B54A32D192ED03ull);
    return orc_splitmix_next(&s);
}

void orc_fill_seeded(float* out, size_t n, uint64_t seed, uint64_t first_elem, float scale) {
    /* tensor.cpp:98-106 (scale == 1) and pipeline.cpp:26-31 draw() (first_elem == 0) */
    uint64_t s = seed + first_elem * 0x9E3779B97F4A7C15ull;
    for (size_t i = 0; i < n; ++i) {
        const float u = orc_next_unit(&s);
        out[i] = (scale == 1.0f) ? u : u * scale;
    }
}

/* ---- pipeline.cpp:14-67 -------------------------------------------------- */

enum { SLOT_STUB = 0, SLOT_CONVW = 1, SLOT_CONVB = 2, SLOT_GAMMA = 3, SLOT_BETA = 4,
       SLOT_WQ = 5, SLOT_WK = 6, SLOT_WV = 7, SLOT_WO = 8 };

int orc_build_block(uint32_t C, uint32_t taps, uint64_t weight_seed, uint32_t b, float* stub_a,
                    float* stub_c, float* conv_w, float* conv_b, float* gamma, float* beta,
                    float* wq, float* wk, float* wv, float* wo) {
    if (taps == 0 || taps % 2 == 0 || C == 0) return ORC_ECONFIG;
    const float mat = 1.0f / sqrtf((float)C);
#define SALT(slot) orc_mix_seed(weight_seed, (uint64_t)b * 16 + (slot))
    { /* ops.cpp:57-65 spatial_stub_coeffs: first C draws are a, next C are c */
        uint64_t s = SALT(SLOT_STUB);
        for (uint32_t i = 0; i < C; ++i) stub_a[i] = orc_next_unit(&s);
        for (uint32_t i = 0; i < C; ++i) stub_c[i] = orc_next_unit(&s);
    }
    orc_fill_seeded(conv_w, (size_t)taps * C * C, SALT(SLOT_CONVW), 0, mat);
    orc_fill_seeded(conv_b, C, SALT(SLOT_CONVB), 0, 1.0f);
    orc_fill_seeded(gamma, C, SALT(SLOT_GAMMA), 0, 1.0f);
    orc_fill_seeded(beta, C, SALT(SLOT_BETA), 0, 1.0f);
    orc_fill_seeded(wq, (size_t)C * C, SALT(SLOT_WQ), 0, mat);
    orc_fill_seeded(wk, (size_t)C * C, SALT(SLOT_WK), 0, mat);
    orc_fill_seeded(wv, (size_t)C * C, SALT(SLOT_WV), 0, mat);
    orc_fill_seeded(wo, (size_t)C * C, SALT(SLOT_WO), 0, mat);
#undef SALT
    return ORC_OK;
}

/* ---- ops.cpp:42-55 ------------------------------------------------------- */

void orc_spatial_affine_tanh(const float* v, size_t n, uint32_t C, const float* a, const float* c,
                             float* out) {
    for (size_t i = 0; i < n; ++i) {
        const uint32_t ch = (uint32_t)(i % C);
        out[i] = tanhf(a[ch] * v[i] + c[ch]);
    }
}

/* ---- ops.cpp:73-104 ------------------------------------------------------ */

int orc_conv_over_extended(const float* ext, uint32_t ext_f, uint32_t H, uint32_t W, uint32_t C,
                           uint32_t out_start, uint32_t out_len, uint32_t taps, const float* wts,
                           const float* bias, float* out) {
    if (taps == 0 || taps % 2 == 0) return ORC_ECONFIG;
    if (out_len == 0 || out_start > ext_f || out_len > ext_f - out_start) return ORC_ERANGE;
    const int halo = (int)((taps - 1) / 2);
    const size_t npos = (size_t)H * W;
    const size_t fe = npos * C;
    for (uint32_t f = 0; f < out_len; ++f) {
        for (size_t pos = 0; pos < npos; ++pos) {
            float* o = out + (size_t)f * fe + pos * C;
            for (uint32_t oc = 0; oc < C; ++oc) {
                double acc = (double)bias[oc];
                for (int j = -halo; j <= halo; ++j) {
                    const int64_t sf = (int64_t)out_start + f + j;
                    if (sf < 0 || sf >= (int64_t)ext_f) continue; /* video edge: zeros */
                    const float* in = ext + (size_t)sf * fe + pos * C;
                    const float* wr = wts + ((size_t)(j + halo) * C + oc) * C;
                    for (uint32_t ic = 0; ic < C; ++ic) acc += (double)wr[ic] * (double)in[ic];
                }
                o[oc] = (float)acc;
            }
        }
    }
    return ORC_OK;
}

/* ---- ops.cpp:112-173 ----------------------------------------------------- */

int orc_group_means(const float* v, size_t total, uint32_t C, uint32_t groups, double* means) {
    if (groups == 0 || C % groups != 0) return ORC_ECONFIG;
    const uint32_t gs = C / groups;
    for (uint32_t g = 0; g < groups; ++g) means[g] = 0.0;
    for (size_t i = 0; i < total; ++i) means[(i % C) / gs] += (double)v[i];
    const double count = (double)(total / groups);
    for (uint32_t g = 0; g < groups; ++g) means[g] /= count;
    return ORC_OK;
}

int orc_group_sqdev(const float* v, size_t total, uint32_t C, uint32_t groups,
                    const double* means, double* vars) {
    if (groups == 0 || C % groups != 0) return ORC_ECONFIG;
    const uint32_t gs = C / groups;
    for (uint32_t g = 0; g < groups; ++g) vars[g] = 0.0;
    for (size_t i = 0; i < total; ++i) {
        const uint32_t g = (uint32_t)(i % C) / gs;
        const double d = (double)v[i] - means[g];
        vars[g] += d * d;
    }
    const double count = (double)(total / groups);
    for (uint32_t g = 0; g < groups; ++g) vars[g] /= count;
    return ORC_OK;
}

int orc_normalize_with_stats(const float* v, size_t total, uint32_t C, uint32_t groups,
                             const float* gamma, const float* beta, float eps,
                             const double* means, const double* vars, float* out) {
    if (groups == 0 || C % groups != 0) return ORC_ECONFIG;
    if (!(eps > 0.0f)) return ORC_ECONFIG;
    const uint32_t gs = C / groups;
    double* inv = (double*)malloc(sizeof(double) * groups);
    for (uint32_t g = 0; g < groups; ++g) inv[g] = 1.0 / sqrt(vars[g] + (double)eps);
    for (size_t i = 0; i < total; ++i) {
        const uint32_t ch = (uint32_t)(i % C);
        const uint32_t g = ch / gs;
        out[i] = (float)((double)gamma[ch] * (((double)v[i] - means[g]) * inv[g]) +
                         (double)beta[ch]);
    }
    free(inv);
    return ORC_OK;
}

int orc_group_norm(const float* v, size_t total, uint32_t C, uint32_t groups, const float* gamma,
                   const float* beta, float eps, float* out) {
    if (groups == 0 || C % groups != 0) return ORC_ECONFIG;
    double* m = (double*)malloc(sizeof(double) * groups);
    double* s = (double*)malloc(sizeof(double) * groups);
    orc_group_means(v, total, C, groups, m);
    orc_group_sqdev(v, total, C, groups, m, s);
    const int rc = orc_normalize_with_stats(v, total, C, groups, gamma, beta, eps, m, s, out);
    free(m);
    free(s);
    return rc;
}

/* ---- ops.cpp:177-207 ----------------------------------------------------- */

int orc_build_local_window(uint32_t a, uint32_t frames, uint32_t n_local, uint32_t* out) {
    if (a >= frames) return -1;
    const uint32_t half = n_local / 2;
    const uint32_t lo = a > half ? a - half : 0;
    const uint32_t hi = (a + half < frames) ? a + half : frames - 1;
    int n = 0;
    for (uint32_t i = lo; i <= hi; ++i) out[n++] = i;
    return n;
}

int orc_build_global_index_set(uint32_t frames, uint32_t n_global, uint32_t* out) {
    if (n_global > frames) return -1;
    for (uint32_t j = 0; j < n_global; ++j)
        out[j] = (uint32_t)(((uint64_t)j * frames) / n_global);
    return (int)n_global;
}

void orc_project_vec(const float* w, const float* x, uint32_t dim, float* y) {
    for (uint32_t o = 0; o < dim; ++o) {
        double acc = 0.0;
        const float* row = w + (size_t)o * dim;
        for (uint32_t i = 0; i < dim; ++i) acc += (double)row[i] * (double)x[i];
        y[o] = (float)acc;
    }
}

/* ops.cpp:209-241 for one head: q/k/v rows have stride `ld`, the head uses
 * `dim` channels starting at the pointers given. */
static void attend_tokens(const float* q, const float* keys, const float* values, size_t ld,
                          const uint32_t* tokens, const uint8_t* biased, size_t n, float bias,
                          float scale, uint32_t dim, float* ctx, double* logits, double* acc,
                          double* row_sum) {
    double mx = -1e300;
    for (size_t i = 0; i < n; ++i) {
        const float* k = keys + (size_t)tokens[i] * ld;
        double dot = 0.0;
        for (uint32_t c = 0; c < dim; ++c) dot += (double)q[c] * (double)k[c];
        double l = (double)scale * dot;
        if (biased[i]) l += (double)bias;
        logits[i] = l;
        if (l > mx) mx = l;
    }
    double denom = 0.0;
    for (size_t i = 0; i < n; ++i) {
        logits[i] = exp(logits[i] - mx);
        denom += logits[i];
    }
    for (uint32_t c = 0; c < dim; ++c) acc[c] = 0.0;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double wgt = logits[i] / denom;
        sum += wgt;
        const float* v = values + (size_t)tokens[i] * ld;
        for (uint32_t c = 0; c < dim; ++c) acc[c] += wgt * (double)v[c];
    }
    for (uint32_t c = 0; c < dim; ++c) ctx[c] = (float)acc[c];
    if (row_sum) *row_sum = sum;
}

/* Shared core of attention_full / dual_scope_reference / attention_parallel:
 * for every position, project `rows` source frames to K/V (src_at(r)), the
 * query frames (q_src) to Q, attend over tokens[a], project through Wo. */
typedef struct {
    uint32_t n;          /* tokens for this query */
    uint32_t* tok;       /* row indices into the K/V row table */
    uint8_t* biased;
} TokenList;

static void attention_core(const float* const* kv_src, uint32_t rows, const float* const* q_src,
                           uint32_t nq, float* const* out_at, size_t npos, uint32_t C,
                           const float* wq, const float* wk, const float* wv, const float* wo,
                           float scale, uint32_t heads, const TokenList* lists, float bias,
                           double* row_sums) {
    const uint32_t d = C / heads;
    float* km = (float*)malloc(sizeof(float) * (size_t)rows * C);
    float* vm = (float*)malloc(sizeof(float) * (size_t)rows * C);
    float* qm = (float*)malloc(sizeof(float) * (size_t)nq * C);
    float* ctx = (float*)malloc(sizeof(float) * C);
    uint32_t maxn = 1;
    for (uint32_t a = 0; a < nq; ++a)
        if (lists[a].n > maxn) maxn = lists[a].n;
    double* logits = (double*)malloc(sizeof(double) * maxn);
    double* acc = (double*)malloc(sizeof(double) * d);
    size_t probe = 0;
    for (size_t pos = 0; pos < npos; ++pos) {
        for (uint32_t r = 0; r < rows; ++r) {
            const float* x = kv_src[r] + pos * C;
            orc_project_vec(wk, x, C, km + (size_t)r * C);
            orc_project_vec(wv, x, C, vm + (size_t)r * C);
        }
        for (uint32_t a = 0; a < nq; ++a)
            orc_project_vec(wq, q_src[a] + pos * C, C, qm + (size_t)a * C);
        for (uint32_t a = 0; a < nq; ++a) {
            for (uint32_t h = 0; h < heads; ++h) {
                double rs = 0.0;
                attend_tokens(qm + (size_t)a * C + (size_t)h * d, km + (size_t)h * d,
                              vm + (size_t)h * d, C, lists[a].tok, lists[a].biased, lists[a].n,
                              bias, scale, d, ctx + (size_t)h * d, logits, acc,
                              row_sums ? &rs : NULL);
                if (row_sums && h == 0) row_sums[probe++] = rs;
            }
            orc_project_vec(wo, ctx, C, out_at[a] + pos * C);
        }
    }
    free(km); free(vm); free(qm); free(ctx); free(logits); free(acc);
}

static void free_lists(TokenList* l, uint32_t n) {
    for (uint32_t a = 0; a < n; ++a) { free(l[a].tok); free(l[a].biased); }
    free(l);
}

int orc_attention_full(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                       const float* wq, const float* wk, const float* wv, const float* wo,
                       float scale, float* out, double* row_sums) {
    if (!(scale > 0.0f) || F == 0) return ORC_ECONFIG;
    const size_t npos = (size_t)H * W, fe = npos * C;
    TokenList* lists = (TokenList*)calloc(F, sizeof(TokenList));
    const float** src = (const float**)malloc(sizeof(float*) * F);
    float** dst = (float**)malloc(sizeof(float*) * F);
    for (uint32_t a = 0; a < F; ++a) {
        lists[a].n = F;
        lists[a].tok = (uint32_t*)malloc(sizeof(uint32_t) * F);
        lists[a].biased = (uint8_t*)calloc(F, 1);
        for (uint32_t i = 0; i < F; ++i) lists[a].tok[i] = i;
        src[a] = v + (size_t)a * fe;
        dst[a] = out + (size_t)a * fe;
    }
    /* ops.cpp:276-287 scans (h, w) then a; row_sums follow that order */
    attention_core(src, F, src, F, dst, npos, C, wq, wk, wv, wo, scale, 1, lists, 0.0f, row_sums);
    free_lists(lists, F);
    free(src); free(dst);
    return ORC_OK;
}

int orc_dual_scope(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C, double t,
                   const float* wq, const float* wk, const float* wv, const float* wo, float scale,
                   uint32_t heads, uint32_t n_local, uint32_t n_global, float bias, double t_star,
                   float* out, uint64_t* counters) {
    if (!(scale > 0.0f) || heads == 0 || C % heads != 0) return ORC_ECONFIG;
    if (n_global > F || F == 0) return ORC_ECONFIG;
    const size_t npos = (size_t)H * W, fe = npos * C;
    uint32_t* gset = (uint32_t*)malloc(sizeof(uint32_t) * (n_global + 1));
    orc_build_global_index_set(F, n_global, gset);
    const int bias_global = t > t_star; /* ops.cpp:298, strict */
    TokenList* lists = (TokenList*)calloc(F, sizeof(TokenList));
    uint32_t* win = (uint32_t*)malloc(sizeof(uint32_t) * (n_local + 2));
    const float** src = (const float**)malloc(sizeof(float*) * F);
    float** dst = (float**)malloc(sizeof(float*) * F);
    uint64_t entries = 0, maxt = 0;
    for (uint32_t a = 0; a < F; ++a) { /* ops.cpp:301-316: window first, then globals */
        const int nw = orc_build_local_window(a, F, n_local, win);
        const uint32_t n = (uint32_t)nw + n_global;
        lists[a].n = n;
        lists[a].tok = (uint32_t*)malloc(sizeof(uint32_t) * n);
        lists[a].biased = (uint8_t*)malloc(n);
        for (int i = 0; i < nw; ++i) {
            lists[a].tok[i] = win[i];
            lists[a].biased[i] = bias_global ? 0 : 1;
        }
        for (uint32_t j = 0; j < n_global; ++j) {
            lists[a].tok[nw + j] = gset[j];
            lists[a].biased[nw + j] = bias_global ? 1 : 0;
        }
        entries += n;
        if (n > maxt) maxt = n;
        src[a] = v + (size_t)a * fe;
        dst[a] = out + (size_t)a * fe;
    }
    attention_core(src, F, src, F, dst, npos, C, wq, wk, wv, wo, scale, heads, lists, bias, NULL);
    if (counters) { /* ops.cpp:326-333 */
        counters[0] += entries * npos;
        counters[1] += (uint64_t)F * npos;
        if (maxt > counters[2]) counters[2] = maxt;
    }
    free_lists(lists, F);
    free(gset); free(win); free(src); free(dst);
    return ORC_OK;
}

int orc_attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const float* v,
                           const float* pre, const float* post, const float* glob, uint32_t H,
                           uint32_t W, uint32_t C, double t, const float* wq, const float* wk,
                           const float* wv, const float* wo, float scale, uint32_t heads,
                           uint32_t n_local, uint32_t n_global, float bias, double t_star,
                           float* out) {
    uint32_t f_clip;
    if (orc_make_plan(frames, workers, &f_clip) != ORC_OK) return ORC_ECONFIG;
    if (!(scale > 0.0f) || heads == 0 || C % heads != 0) return ORC_ECONFIG;
    const uint32_t half = n_local / 2;
    const uint32_t npre = (worker > 0) ? half : 0;
    const uint32_t npost = (worker + 1 < workers) ? half : 0;
    if ((npre && !pre) || (npost && !post) || (n_global && !glob)) return ORC_ECONFIG;
    const size_t npos = (size_t)H * W, fe = npos * C;
    const uint32_t ext_f = npre + f_clip + npost;
    const uint32_t start = worker * f_clip, ext_start = start - npre;
    const int bias_global = t > t_star;
    /* clip_parallel.cpp:277-280: rows 0..ext_f-1 = [pre | v | post], then globals */
    const uint32_t rows = ext_f + n_global;
    const float** kv = (const float**)malloc(sizeof(float*) * rows);
    for (uint32_t r = 0; r < npre; ++r) kv[r] = pre + (size_t)r * fe;
    for (uint32_t r = 0; r < f_clip; ++r) kv[npre + r] = v + (size_t)r * fe;
    for (uint32_t r = 0; r < npost; ++r) kv[npre + f_clip + r] = post + (size_t)r * fe;
    for (uint32_t j = 0; j < n_global; ++j) kv[ext_f + j] = glob + (size_t)j * fe;
    TokenList* lists = (TokenList*)calloc(f_clip, sizeof(TokenList));
    uint32_t* win = (uint32_t*)malloc(sizeof(uint32_t) * (n_local + 2));
    const float** qs = (const float**)malloc(sizeof(float*) * f_clip);
    float** dst = (float**)malloc(sizeof(float*) * f_clip);
    int rc = ORC_OK;
    for (uint32_t a = 0; a < f_clip; ++a) { /* clip_parallel.cpp:285-305 */
        const int nw = orc_build_local_window(start + a, frames, n_local, win);
        const uint32_t n = (uint32_t)nw + n_global;
        lists[a].n = n;
        lists[a].tok = (uint32_t*)malloc(sizeof(uint32_t) * n);
        lists[a].biased = (uint8_t*)malloc(n);
        for (int i = 0; i < nw; ++i) {
            if (win[i] < ext_start || win[i] - ext_start >= ext_f) rc = ORC_ERANGE;
            lists[a].tok[i] = win[i] - ext_start;
            lists[a].biased[i] = bias_global ? 0 : 1;
        }
        for (uint32_t j = 0; j < n_global; ++j) {
            lists[a].tok[nw + j] = ext_f + j;
            lists[a].biased[nw + j] = bias_global ? 1 : 0;
        }
        qs[a] = v + (size_t)a * fe;
        dst[a] = out + (size_t)a * fe;
    }
    if (rc == ORC_OK)
        attention_core(kv, rows, qs, f_clip, dst, npos, C, wq, wk, wv, wo, scale, heads, lists,
                       bias, NULL);
    free_lists(lists, f_clip);
    free(kv); free(win); free(qs); free(dst);
    return rc;
}

/* ---- clip_parallel.cpp:54-91, 343-387 ------------------------------------ */

int orc_make_plan(uint32_t frames, uint32_t workers, uint32_t* f_clip) {
    if (workers == 0 || frames == 0 || frames % workers != 0) return ORC_ECONFIG;
    *f_clip = frames / workers;
    return ORC_OK;
}

int orc_global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start, uint32_t len,
                                uint32_t* out) {
    if (n_global > frames) return -1;
    int n = 0;
    for (uint32_t j = 0; j < n_global; ++j) {
        const uint32_t g = (uint32_t)(((uint64_t)j * frames) / n_global);
        if (g >= start && g < start + len) out[n++] = g - start;
    }
    return n;
}

int orc_predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo,
                             uint32_t global_frames, uint32_t worker, uint64_t frame_bytes,
                             uint64_t* out) {
    uint32_t f_clip;
    if (orc_make_plan(frames, workers, &f_clip) != ORC_OK) return ORC_ECONFIG;
    out[0] = out[1] = out[2] = 0;
    if (workers == 1) return ORC_OK;
    if (global_frames > 0) {
        uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (global_frames + 1));
        uint64_t total = 0, next = 0, mine = 0;
        for (uint32_t w = 0; w < workers; ++w) {
            const int k = orc_global_members_in_range(frames, global_frames, w * f_clip, f_clip, tmp);
            const uint64_t b = (uint64_t)k * frame_bytes;
            total += b;
            if (w == (worker + 1) % workers) next = b;
            if (w == worker) mine = b;
        }
        free(tmp);
        out[0] += total - next;
        out[1] += mine;
        out[2] += workers - 1;
    }
    if (halo > 0) {
        const uint64_t hb = (uint64_t)halo * frame_bytes;
        if (worker + 1 < workers) { out[0] += hb; out[1] += hb; out[2] += 1; }
        if (worker > 0) { out[0] += hb; out[1] += hb; out[2] += 1; }
    }
    return ORC_OK;
}

int orc_predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                                  uint32_t worker, uint64_t* out) {
    (void)worker;
    uint32_t f_clip;
    if (orc_make_plan(frames, workers, &f_clip) != ORC_OK) return ORC_ECONFIG;
    out[0] = out[1] = out[2] = 0;
    if (workers == 1) return ORC_OK;
    const uint64_t block = (uint64_t)groups * sizeof(double);
    out[0] = 2 * block * (workers - 1);
    out[1] = 2 * block;
    out[2] = 2 * (uint64_t)(workers - 1);
    return ORC_OK;
}

/* ---- pipeline.cpp:102-111, one block ------------------------------------- */

int orc_block_forward(const float* x, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                      uint32_t taps, uint32_t groups, double t, const float* stub_a,
                      const float* stub_c, const float* conv_w, const float* conv_b,
                      const float* gamma, const float* beta, float eps, const float* wq,
                      const float* wk, const float* wv, const float* wo, float scale,
                      uint32_t heads, uint32_t n_local, uint32_t n_global, float bias,
                      double t_star, float* out) {
    const size_t n = (size_t)F * H * W * C;
    float* u = (float*)malloc(sizeof(float) * n);
    float* tmp = (float*)malloc(sizeof(float) * n);
    int rc;
    orc_spatial_affine_tanh(x, n, C, stub_a, stub_c, u);
    rc = orc_conv_over_extended(u, F, H, W, C, 0, F, taps, conv_w, conv_b, tmp);
    if (rc) goto done;
    for (size_t i = 0; i < n; ++i) u[i] = u[i] + tmp[i]; /* pipeline.cpp:83-91 add */
    rc = orc_group_norm(u, n, C, groups, gamma, beta, eps, tmp);
    if (rc) goto done;
    rc = orc_dual_scope(tmp, F, H, W, C, t, wq, wk, wv, wo, scale, heads, n_local, n_global, bias,
                        t_star, out, NULL);
    if (rc) goto done;
    for (size_t i = 0; i < n; ++i) out[i] = tmp[i] + out[i];
done:
    free(u);
    free(tmp);
    return rc;
}
