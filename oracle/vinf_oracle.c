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

/* ---- speed without changing a bit --------------------------------------------------
 * The checker must finish the BASELINE configurations (up to 24 x 40x64 x C=640 and
 * C=1280 levels) in seconds on the GPU box's host, and stay bitwise equal to the
 * reference. Two devices do that:
 *   1. positions (and frames) are independent in every reduction the reference does
 *      per output, so they are split over pthreads (ORC_THREADS, default: all cores);
 *      each output is still computed by exactly one thread in the reference's order;
 *   2. the f64-accumulated dot products (ops.cpp:90-99, :200-207) are vectorised ACROSS
 *      outputs, never along the reduction: each output's accumulator sees the same
 *      sequence of additions as the reference's scalar loop. f32 x f32 products are exact
 *      in f64, so a fused or separate multiply-add rounds identically.
 * The GroupNorm statistics (one running sum per group over the whole tensor,
 * ops.cpp:112-142) are order-dependent and stay serial. */
#include <pthread.h>
#include <unistd.h>

typedef double orc_v4d __attribute__((vector_size(32)));
typedef float orc_v4f __attribute__((vector_size(16), aligned(4)));

static int orc_threads(void) {
    const char* e = getenv("ORC_THREADS");
    long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    if (n < 1) n = 1;
    if (n > 256) n = 256;
    return (int)n;
}

typedef void (*orc_range_fn)(void* ctx, size_t lo, size_t hi);
typedef struct { orc_range_fn fn; void* ctx; size_t lo, hi; } orc_job;
static void* orc_job_run(void* p) {
    orc_job* j = (orc_job*)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}
/* fn(ctx, lo, hi) over [0, n) in contiguous ranges, one per thread */
static void orc_parallel(size_t n, orc_range_fn fn, void* ctx) {
    int nt = orc_threads();
    if ((size_t)nt > n) nt = (int)(n ? n : 1);
    if (nt <= 1) { fn(ctx, 0, n); return; }
    pthread_t th[256];
    orc_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = n * (size_t)t / (size_t)nt;
        jobs[t].hi = n * (size_t)(t + 1) / (size_t)nt;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, orc_job_run, &jobs[t]);
    orc_job_run(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

/* Row micro-kernel. For nr <= 4 rows r and every output o < N:
 *   acc = init ? (double)init[o] : 0.0;
 *   for s in [0, nseg): for i in [0, K): acc += (double)wT[s][i*N + o] * (double)x[s][r][i];
 *   y[r][o] = (float)acc;
 * wT[s] is the TRANSPOSED weight matrix ([K][N]), so a step over i reads N contiguous
 * weights; x[s][r] points at row r's K inputs of segment s. */
#define ORC_MAXSEG 16
static void orc_rows(uint32_t nr, uint32_t nseg, const float* const* wT,
                     const float* const (*x)[4], uint32_t K, uint32_t N, const float* init,
                     float* const* y) {
    uint32_t o0 = 0;
    for (; o0 + 8 <= N; o0 += 8) {
        orc_v4d a[4][2];
        for (uint32_t r = 0; r < 4; ++r)
            for (int h = 0; h < 2; ++h)
                for (int k = 0; k < 4; ++k) a[r][h][k] = init ? (double)init[o0 + 4 * h + k] : 0.0;
        for (uint32_t s = 0; s < nseg; ++s) {
            const float* w = wT[s] + o0;
            const float* x0 = x[s][0];
            const float* x1 = x[s][nr > 1 ? 1 : 0];
            const float* x2 = x[s][nr > 2 ? 2 : 0];
            const float* x3 = x[s][nr > 3 ? 3 : 0];
            for (uint32_t i = 0; i < K; ++i, w += N) {
                const orc_v4d w0 = __builtin_convertvector(*(const orc_v4f*)w, orc_v4d);
                const orc_v4d w1 = __builtin_convertvector(*(const orc_v4f*)(w + 4), orc_v4d);
                const double v0 = (double)x0[i], v1 = (double)x1[i], v2 = (double)x2[i],
                             v3 = (double)x3[i];
                a[0][0] += w0 * v0; a[0][1] += w1 * v0;
                a[1][0] += w0 * v1; a[1][1] += w1 * v1;
                a[2][0] += w0 * v2; a[2][1] += w1 * v2;
                a[3][0] += w0 * v3; a[3][1] += w1 * v3;
            }
        }
        for (uint32_t r = 0; r < nr; ++r)
            for (int h = 0; h < 2; ++h)
                for (int k = 0; k < 4; ++k) y[r][o0 + 4 * h + k] = (float)a[r][h][k];
    }
    for (; o0 < N; ++o0) /* N % 8 tail (the reference's own tests use C = 3, 4) */
        for (uint32_t r = 0; r < nr; ++r) {
            double acc = init ? (double)init[o0] : 0.0;
            for (uint32_t s = 0; s < nseg; ++s)
                for (uint32_t i = 0; i < K; ++i)
                    acc += (double)wT[s][(size_t)i * N + o0] * (double)x[s][r][i];
            y[r][o0] = (float)acc;
        }
}

/* [rows][cols] -> [cols][rows] */
static float* orc_transpose(const float* w, uint32_t rows, uint32_t cols) {
    float* t = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < cols; ++c) t[(size_t)c * rows + r] = w[(size_t)r * cols + c];
    return t;
}

/* y_r = W x_r for nr rows through the micro-kernel (WT = W transposed, [dim][dim]) */
static void orc_project_rows(const float* WT, const float* const* xs, uint32_t nr, uint32_t dim,
                             float* const* ys) {
    for (uint32_t r0 = 0; r0 < nr; r0 += 4) {
        const uint32_t n = nr - r0 < 4 ? nr - r0 : 4;
        const float* xr[1][4];
        float* yr[4];
        for (uint32_t r = 0; r < 4; ++r) {
            xr[0][r] = xs[r0 + (r < n ? r : 0)];
            yr[r] = ys[r0 + (r < n ? r : 0)];
        }
        orc_rows(n, 1, &WT, (const float* const(*)[4])xr, dim, dim, NULL, yr);
    }
}

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

typedef struct { const float* v; uint32_t C; const float *a, *c; float* out; } orc_stub_job;
static void orc_stub_range(void* p, size_t lo, size_t hi) {
    const orc_stub_job* J = (const orc_stub_job*)p;
    for (size_t i = lo; i < hi; ++i) {
        const uint32_t ch = (uint32_t)(i % J->C);
        J->out[i] = tanhf(J->a[ch] * J->v[i] + J->c[ch]);
    }
}

void orc_spatial_affine_tanh(const float* v, size_t n, uint32_t C, const float* a, const float* c,
                             float* out) {
    orc_stub_job J = {v, C, a, c, out};
    orc_parallel(n, orc_stub_range, &J);
}

/* ---- ops.cpp:73-104 ------------------------------------------------------ */

typedef struct {
    const float* ext; uint32_t ext_f, C, taps, out_start;
    size_t npos, fe;
    const float* const* wT; /* [taps] transposed [C][C] tap matrices */
    const float* bias; float* out;
} orc_conv_job;

/* unit u = (output frame f, block of 4 positions) */
static void orc_conv_range(void* p, size_t lo, size_t hi) {
    const orc_conv_job* J = (const orc_conv_job*)p;
    const size_t nb = (J->npos + 3) / 4;
    const int halo = (int)((J->taps - 1) / 2);
    for (size_t u = lo; u < hi; ++u) {
        const uint32_t f = (uint32_t)(u / nb);
        const size_t p0 = (u % nb) * 4;
        const uint32_t nr = (uint32_t)(J->npos - p0 < 4 ? J->npos - p0 : 4);
        const float* wT[ORC_MAXSEG];
        const float* xs[ORC_MAXSEG][4];
        float* ys[4];
        uint32_t ns = 0;
        for (int j = -halo; j <= halo; ++j) { /* ops.cpp:91-99: taps in order, edges skipped */
            const int64_t sf = (int64_t)J->out_start + f + j;
            if (sf < 0 || sf >= (int64_t)J->ext_f) continue; /* video edge: zeros */
            wT[ns] = J->wT[j + halo];
            for (uint32_t r = 0; r < 4; ++r)
                xs[ns][r] = J->ext + (size_t)sf * J->fe + (p0 + (r < nr ? r : 0)) * J->C;
            ++ns;
        }
        for (uint32_t r = 0; r < 4; ++r)
            ys[r] = J->out + (size_t)f * J->fe + (p0 + (r < nr ? r : 0)) * J->C;
        orc_rows(nr, ns, wT, (const float* const(*)[4])xs, J->C, J->C, J->bias, ys);
    }
}

int orc_conv_over_extended(const float* ext, uint32_t ext_f, uint32_t H, uint32_t W, uint32_t C,
                           uint32_t out_start, uint32_t out_len, uint32_t taps, const float* wts,
                           const float* bias, float* out) {
    if (taps == 0 || taps % 2 == 0) return ORC_ECONFIG;
    if (out_len == 0 || out_start > ext_f || out_len > ext_f - out_start) return ORC_ERANGE;
    if (taps > ORC_MAXSEG) return ORC_ECONFIG;
    /* out[f,pos,oc] = b[oc] + sum_j sum_ic W[j][oc][ic] * ext[out_start+f+j, pos, ic],
     * accumulated in f64 in (j, ic) order, frames outside [0, ext_f) skipped */
    float* wT[ORC_MAXSEG];
    for (uint32_t j = 0; j < taps; ++j) wT[j] = orc_transpose(wts + (size_t)j * C * C, C, C);
    orc_conv_job J = {ext, ext_f, C, taps, out_start, (size_t)H * W, (size_t)H * W * C,
                      (const float* const*)wT, bias, out};
    orc_parallel((size_t)out_len * ((J.npos + 3) / 4), orc_conv_range, &J);
    for (uint32_t j = 0; j < taps; ++j) free(wT[j]);
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

typedef struct {
    const float* v; uint32_t C, gs; const float *gamma, *beta; const double *means, *inv; float* out;
} orc_norm_job;
static void orc_norm_range(void* p, size_t lo, size_t hi) {
    const orc_norm_job* J = (const orc_norm_job*)p;
    for (size_t i = lo; i < hi; ++i) {
        const uint32_t ch = (uint32_t)(i % J->C);
        const uint32_t g = ch / J->gs;
        J->out[i] = (float)((double)J->gamma[ch] * (((double)J->v[i] - J->means[g]) * J->inv[g]) +
                            (double)J->beta[ch]);
    }
}

int orc_normalize_with_stats(const float* v, size_t total, uint32_t C, uint32_t groups,
                             const float* gamma, const float* beta, float eps,
                             const double* means, const double* vars, float* out) {
    if (groups == 0 || C % groups != 0) return ORC_ECONFIG;
    if (!(eps > 0.0f)) return ORC_ECONFIG;
    const uint32_t gs = C / groups;
    double* inv = (double*)malloc(sizeof(double) * groups);
    for (uint32_t g = 0; g < groups; ++g) inv[g] = 1.0 / sqrt(vars[g] + (double)eps);
    orc_norm_job J = {v, C, gs, gamma, beta, means, inv, out};
    orc_parallel(total, orc_norm_range, &J);
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

typedef struct {
    const float* const* kv_src; uint32_t rows;
    const float* const* q_src; uint32_t nq;
    float* const* out_at; uint32_t C, heads;
    const float *wqT, *wkT, *wvT, *woT;
    float scale, bias;
    const TokenList* lists;
    double* row_sums;
} orc_attn_job;

static void orc_attn_range(void* p, size_t lo, size_t hi) {
    const orc_attn_job* J = (const orc_attn_job*)p;
    const uint32_t C = J->C, rows = J->rows, nq = J->nq, heads = J->heads;
    const uint32_t d = C / heads;
    float* km = (float*)malloc(sizeof(float) * (size_t)rows * C);
    float* vm = (float*)malloc(sizeof(float) * (size_t)rows * C);
    float* qm = (float*)malloc(sizeof(float) * (size_t)nq * C);
    float* cm = (float*)malloc(sizeof(float) * (size_t)nq * C);
    uint32_t maxn = 1;
    for (uint32_t a = 0; a < nq; ++a)
        if (J->lists[a].n > maxn) maxn = J->lists[a].n;
    double* logits = (double*)malloc(sizeof(double) * maxn);
    double* acc = (double*)malloc(sizeof(double) * d);
    const uint32_t nmax = rows > nq ? rows : nq;
    const float** xs = (const float**)malloc(sizeof(float*) * nmax);
    float** ys = (float**)malloc(sizeof(float*) * nmax);
    for (size_t pos = lo; pos < hi; ++pos) {
        /* ops.cpp:247-260 project_location: K and V of every row, Q of every query */
        for (uint32_t r = 0; r < rows; ++r) { xs[r] = J->kv_src[r] + pos * C; ys[r] = km + (size_t)r * C; }
        orc_project_rows(J->wkT, xs, rows, C, ys);
        for (uint32_t r = 0; r < rows; ++r) ys[r] = vm + (size_t)r * C;
        orc_project_rows(J->wvT, xs, rows, C, ys);
        for (uint32_t a = 0; a < nq; ++a) { xs[a] = J->q_src[a] + pos * C; ys[a] = qm + (size_t)a * C; }
        orc_project_rows(J->wqT, xs, nq, C, ys);
        for (uint32_t a = 0; a < nq; ++a) {
            for (uint32_t h = 0; h < heads; ++h) {
                double rs = 0.0;
                attend_tokens(qm + (size_t)a * C + (size_t)h * d, km + (size_t)h * d,
                              vm + (size_t)h * d, C, J->lists[a].tok, J->lists[a].biased,
                              J->lists[a].n, J->bias, J->scale, d, cm + (size_t)a * C + (size_t)h * d,
                              logits, acc, J->row_sums ? &rs : NULL);
                if (J->row_sums && h == 0) J->row_sums[pos * nq + a] = rs;
            }
        }
        /* ops.cpp:334: out = Wo ctx */
        for (uint32_t a = 0; a < nq; ++a) { xs[a] = cm + (size_t)a * C; ys[a] = J->out_at[a] + pos * C; }
        orc_project_rows(J->woT, xs, nq, C, ys);
    }
    free(km); free(vm); free(qm); free(cm); free(logits); free(acc); free(xs); free(ys);
}

static void attention_core(const float* const* kv_src, uint32_t rows, const float* const* q_src,
                           uint32_t nq, float* const* out_at, size_t npos, uint32_t C,
                           const float* wq, const float* wk, const float* wv, const float* wo,
                           float scale, uint32_t heads, const TokenList* lists, float bias,
                           double* row_sums) {
    float* wqT = orc_transpose(wq, C, C);
    float* wkT = orc_transpose(wk, C, C);
    float* wvT = orc_transpose(wv, C, C);
    float* woT = orc_transpose(wo, C, C);
    orc_attn_job J = {kv_src, rows, q_src, nq, out_at, C, heads, wqT, wkT, wvT, woT,
                      scale, bias, lists, row_sums};
    orc_parallel(npos, orc_attn_range, &J);
    free(wqT); free(wkT); free(wvT); free(woT);
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
