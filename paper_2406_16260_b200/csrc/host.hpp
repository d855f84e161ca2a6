// Internal C++ host layer: error taxonomy, clip plan / token sets, device parameter
// objects, GEMM dispatch, operator forms and the clip engine. The C ABI in capi.cpp is
// a thin guarded wrapper over these.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vinf_temporal.h"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace vinf {

// error.hpp:10-34 of the reference, carried as a status code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(VINF_ERR_CONFIG, m); }
[[noreturn]] inline void shape_error(const std::string& m) { throw Error(VINF_ERR_INVALID, m); }
[[noreturn]] inline void range_error(const std::string& m) { throw Error(VINF_ERR_INVALID, m); }
[[noreturn]] inline void protocol_error(const std::string& m) {
    throw Error(VINF_ERR_TRANSPORT, m);
}
void cuda_check(int err, const char* what);
extern int g_gemm_debug_flags;  // ORed into every GEMM's flags (diagnostics only)

// ---- plan.cpp (pure host) ----
std::vector<uint32_t> build_local_window(uint32_t a, uint32_t frames, uint32_t n_local);
std::vector<uint32_t> build_global_index_set(uint32_t frames, uint32_t n_global);
uint32_t make_plan(uint32_t frames, uint32_t workers);  // returns f_clip
std::vector<uint32_t> global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start,
                                              uint32_t len);
void predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo, uint32_t gframes,
                          uint32_t worker, uint64_t frame_bytes, uint64_t out[3]);
void predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups, uint64_t out[3]);

// Host token table for nq queries (kMaxTokens slots each): the reference's explicit
// token lists (window first, then globals; duplicates kept) plus, per block of kQBlock
// queries, the sorted distinct K/V frames they touch and each token's column in it.
struct HostTokens {
    std::vector<uint16_t> rows;
    std::vector<uint8_t> biased;
    std::vector<uint16_t> count;
    std::vector<uint8_t> col;
    std::vector<uint16_t> kv_frames;
    std::vector<uint16_t> kv_count;
    // Per-column form of the token lists (what the tensor-core cores use): query a's
    // window tokens are the contiguous columns [wlo[a], whi[a]] of its block's K/V list,
    // its global tokens put gmult[block][c] copies on column c; window / global tokens get
    // the bias iff wflag / gflag (uniform per table, checked).
    std::vector<uint16_t> nwin;
    std::vector<uint8_t> wlo, whi, gmult;
    std::vector<uint32_t> kv_box;  // TMA box program per block (TokenTable::kv_box)
    std::vector<uint16_t> kv_nbox, kv_load_rows;
    int wflag = 0, gflag = 0;
    uint32_t nq = 0, nqb = 0;
    bool kv_ok = true;
    void resize(uint32_t n) {
        nq = n;
        nqb = (n + kQBlock - 1) / kQBlock;
        rows.assign(size_t(n) * kMaxTokens, 0);
        biased.assign(size_t(n) * kMaxTokens, 0);
        count.assign(n, 0);
        col.assign(size_t(n) * kMaxTokens, 0);
        kv_frames.assign(size_t(nqb) * kKvMax, 0);
        kv_count.assign(nqb, 0);
        nwin.assign(n, 0);
        wlo.assign(n, 0);
        whi.assign(n, 0);
        gmult.assign(size_t(nqb) * kKvMax, 0);
        kv_box.assign(size_t(nqb) * kKvMax, 0);
        kv_nbox.assign(nqb, 0);
        kv_load_rows.assign(nqb, 0);
    }
    // Window tokens first, then (global = true) the sampled global tokens.
    void push(uint32_t a, uint32_t row, bool b, bool global = false) {
        const uint16_t k = count[a];
        if (k >= kMaxTokens) config_error("too many tokens per query (n_local + 1 + n_global)");
        if (!global && nwin[a] != k) config_error("window tokens must precede global tokens");
        if (row > 0xFFFFu)
            config_error("attention buffer exceeds 65535 frames (16-bit token rows)");
        rows[size_t(a) * kMaxTokens + k] = uint16_t(row);
        biased[size_t(a) * kMaxTokens + k] = b ? 1 : 0;
        count[a] = k + 1;
        if (!global) nwin[a] = k + 1;
    }
    // Builds the per-block K/V lists; call after all push()es. gather4: the attention core
    // may fetch runs of single frames four at a time (head dim a multiple of 64).
    void finalize(bool gather4 = false);
    // One device blob: rows | biased | col | count | kv_frames | kv_count.
    size_t blob_bytes() const;
    void pack(uint8_t* dst) const;
    TokenTable view(const uint8_t* dev_base) const;
};

// Device copy of a HostTokens table (one allocation).
struct DevTokens {
    void* buf = nullptr;
    TokenTable tt{};
    void upload(const HostTokens& h, cudaStream_t s);  // allocates on first use
    void release();
};

// Weight matrix [rows, K] as bf16 hi (= RN(w)) and lo (= RN(w - hi)) planes + fp32 copy.
struct DevMat {
    uint32_t rows = 0, K = 0;
    __nv_bfloat16* hi = nullptr;
    __nv_bfloat16* lo = nullptr;
    void alloc(uint32_t r, uint32_t k);
    void from_f32(const float* w_dev, cudaStream_t s);  // splits a device fp32 matrix
    void release();
};

// A GEMM operand: bf16 plane(s) over [rows, cols] with row stride ld (elements).
struct Operand {
    const __nv_bfloat16* hi = nullptr;
    const __nv_bfloat16* lo = nullptr;  // non-null -> fp32 (split) mode
    uint64_t rows = 0;
    uint32_t cols = 0;
    uint64_t ld = 0;
};

struct Epilogue {
    const float* bias = nullptr;
    const void* res = nullptr;
    const float* res_scale = nullptr;  // residual * scale per column (or identity)
    int64_t res_ld = 0;
    bool res_bf16 = false;
    void* out = nullptr;
    int64_t out_ld = 0;
    bool out_bf16 = false;
    float* colpart = nullptr;  // fused per-(32-row block, column) (sum, sum of squares)
    // fp32 output as split bf16 planes: out = hi plane, out_lo = lo plane (both bf16, out_ld)
    void* out_lo = nullptr;
};

// out[m, n] = sum_s A[m + a_rows[s]] . B[n + b_rows[s]] (+ bias, + res); M x N, K = A.cols.
// Split mode (A.lo && B.lo) expands each segment into hi*hi + hi*lo + lo*hi.
void gemm(const Operand& A, const std::vector<int64_t>& a_rows, const DevMat& B,
          const std::vector<int64_t>& b_rows, int64_t M, int64_t N, const Epilogue& ep, bool split,
          cudaStream_t s);

}  // namespace vinf

// Opaque handle types of the C ABI.
struct vinf_conv_kernel {
    uint32_t taps = 0, C = 0;
    vinf::DevMat w;       // [taps*C, C]
    float* bias = nullptr;  // [C]
};

struct vinf_attention_params {
    uint32_t C = 0, heads = 1;
    float scale = 0.f;
    vinf::DevMat wqkv;  // [3C, C] = Wq; Wk; Wv
    vinf::DevMat wo;    // [C, C]
};
