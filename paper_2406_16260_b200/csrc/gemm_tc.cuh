// Segmented-K tcgen05 GEMM used by every dense contraction of the temporal block:
//
//   D[m, n] = sum_s  A_s[m + a_row_s, :] . B_s[n + b_row_s, :]   (+ bias[n]) (+ R[m, n])
//
// Each segment s names one A and one B tensor map (bf16, K-major, [rows, K]) and a
// row offset into each. This single form covers
//   * the temporal conv as an implicit GEMM: one segment per tap j, A rows shifted
//     by j*H*W inside the halo-extended clip buffer (ops.cpp:87-102), B = W[j];
//   * the Q/K/V and O projections (ops.cpp:200-207): one segment;
//   * the fp32 mode ("bf16x3"): every segment becomes three, hi*hi + hi*lo + lo*hi,
//     with A = a_hi + a_lo and B = b_hi + b_lo split on the producer side.
// TMA zero-fills out-of-range rows (negative or past the end), which is exactly the
// reference's zero padding at the video boundary (ops.cpp:94).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace vinf {

constexpr int kGemmMaxSeg = 12;

struct GemmSeg {
    int32_t a_map;  // 0 or 1 (A hi / A lo)
    int32_t a_row;  // row offset added to the output row
    int32_t b_map;  // 0 or 1 (B hi / B lo)
    int32_t b_row;  // row offset added to the output column
};

struct GemmParams {
    int32_t M, N, K;
    int32_t nseg;
    GemmSeg seg[kGemmMaxSeg];
    const float* bias;  // [N] fp32 or null
    const void* res;    // residual [M, ld] or null
    const float* res_scale;  // optional per-column scale of the residual (16-byte aligned)
    int64_t res_ld;
    int32_t res_bf16;
    void* out;
    int64_t out_ld;
    int32_t out_bf16;
    int32_t flags;  // kGemmFlag* (diagnostics)
    // Optional per-column statistics of the stored output (GroupNorm fused into the
    // conv epilogue), partial rows each written exactly once (no atomics, deterministic):
    // colpart[(r*2 + 0)*N + n] = sum over the rows of partial r of out[m,n],
    // colpart[(r*2 + 1)*N + n] = sum of squares; fp32 [gemm_colpart_rows(M, N)][2][N].
    // Partial r is one (CTA group, TMEM quadrant) when every CTA keeps one column tile
    // (4 * gridDim / n_tiles rows), else one 32-row block (ceil(M / 32) rows).
    float* colpart;
    // fp32 accumulator stored as split bf16 planes (out_bf16 == 0): out = RN(y) and
    // out_lo = RN(y - RN(y)), both bf16 [M, out_ld]; the fp32-mode Q/K/V projection, whose
    // consumer (the attention core's bf16x3 mode) reads exactly these planes
    void* out_lo;
};

constexpr int32_t kGemmFlagNoStore = 1;  // benchmark-only: skip epilogue global traffic
constexpr int32_t kGemmFlagDiagNoTma = 16;  // diagnostics (TMA-store epilogue): stage, do not store
constexpr int32_t kGemmFlagDiagNoSts = 32;  // diagnostics (TMA-store epilogue): convert only
constexpr int32_t kGemmFlagDiagL2Out = 64;  // diagnostics (TMA-store epilogue): rows folded mod 1024
constexpr int32_t kGemmFlagTmaOut = 1 << 8;  // bf16 output leaves through TMA stores (maps.out)
// bf16 output + bf16 residual both through TMA (maps.out, maps.res); block_n % 32 == 0
constexpr int32_t kGemmFlagTmaRes = 1 << 9;

struct GemmMaps {
    CUtensorMap a[2];
    CUtensorMap b[2];
    CUtensorMap out;  // [M, N] bf16, box 32 x 32, 64B swizzle (with kGemmFlagTmaOut / TmaRes)
    CUtensorMap res;  // [M, N] bf16 residual, same box and swizzle (with kGemmFlagTmaRes)
};

// Host side: encode a 2D bf16 K-major tensor map over [rows, cols] with row stride
// ld_elems, box = 64 (K) x box_rows, 128B swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t ld_elems, uint32_t box_rows);
// The epilogue's output map: bf16 [rows, cols] (row stride ld_elems), box 32 x 32, 64B swizzle.
int make_tmap_out_bf16(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems);

// Launches the GEMM on `stream` with N tile block_n. Returns 0 or a cudaError_t.
int gemm_tc_launch(const GemmMaps& maps, const GemmParams& p, int block_n, cudaStream_t stream);

// Largest supported N tile for a given N (used to build B tensor maps).
int gemm_pick_block_n(int N);

// Partial rows the fused column statistics of an M x N GEMM occupy (see GemmParams::colpart);
// never more than 4 * ceil(M / 128), the size to allocate.
int gemm_colpart_rows(int64_t M, int N);

}  // namespace vinf
