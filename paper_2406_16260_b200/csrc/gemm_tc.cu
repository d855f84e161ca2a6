// Persistent, warp-specialised tcgen05 GEMM (sm_100a). See gemm_tc.cuh for the contract.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one thread issues
// tcgen05.mma), warp 2 = TMEM allocator, warps 4..11 = epilogue (TMEM -> registers ->
// bias/residual/convert -> global): two warps per TMEM lane quadrant, alternating
// 32-column chunks of each tile. Operand tiles are 128 x 64 (A) and BN x 64 (B) bf16,
// TMA-loaded with 128B swizzle into a STAGES-deep mbarrier ring. The fp32 accumulator
// lives in TMEM, double-buffered (2 x BN columns) so the epilogue of tile i overlaps
// the main loop of tile i+1.
//
// Epilogue: per 32-column chunk, tcgen05.ld gives each lane one accumulator row; the warp
// transposes the 32x32 block through padded shared memory (conflict-free 16 B accesses)
// so residual loads and output stores are row-coalesced (8 lanes x 4 columns per row,
// 4 rows per instruction). The next chunk's residual is prefetched (all 8 requests in
// flight) while the current chunk is stored. Interior tiles take a branch-free path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "gemm_tc.cuh"

namespace vinf {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr uint32_t kABytes = kBM * kBK * 2;
constexpr int kStgPitch = 36;  // floats per staged row (32 + 4 pad: conflict-free 16 B access)
constexpr uint32_t kStgBytes = kEpiWarps * 32 * kStgPitch * 4;  // a 32x32 fp32 block per epilogue warp

constexpr int kResSlots = 3;  // TMA residual ring depth per epilogue warp (32 x 32 bf16 boxes)

// RT: residual in through TMA and output out through TMA (bf16, no statistics): the
// epilogue needs no transpose block, only two 2 KB store-staging blocks and a residual ring
// per warp.
template <int BN, bool ST = false, bool RT = false, bool TMAO = false>
struct TileCfg {
    static constexpr uint32_t kBBytes = BN * kBK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    // staging per epilogue warp: RT stages its output boxes in the residual ring, the other
    // TMA-store epilogue uses two 2 KB boxes, the transposed epilogue a 32 x kStgPitch fp32 block
    static constexpr uint32_t kStgWarp = RT ? 0 : TMAO ? 4096 : 32 * kStgPitch * 4;
    static constexpr uint32_t kStg = kEpiWarps * kStgWarp;
    static constexpr uint32_t kRes = RT ? kEpiWarps * kResSlots * 2048 : 0;
    static constexpr int kStages =
        std::min<int>(8, (227 * 1024 - 1024 - 1024 - kStg - kRes) / kStageBytes);
    static constexpr uint32_t kAccStride = BN <= 128 ? 128 : 256;  // TMEM columns per buffer
    static constexpr uint32_t kTmemCols = 2 * kAccStride;
    static constexpr uint32_t kSmemBytes =
        kStages * kStageBytes + 1024 /*align*/ + 1024 /*bars*/ + kStg + kRes;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dev::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// Epilogue of one 128 x BN tile for the warp owning TMEM lane quadrant q (rows m0..m0+31).
//   OBF: output (and residual) bf16, else fp32.   RES: residual present.
// Each 32 x 32 accumulator chunk is transposed through the warp's padded smem block so a
// lane then owns 8 consecutive columns of 4 rows (rows tr + 8i): residual loads and output
// stores are 16-byte (bf16) row segments, 4 lanes covering a row's 64 bytes.
template <bool OBF>
struct EpiRes {
    static constexpr int W = OBF ? 4 : 8;  // 32-bit words of 8 residual values
    uint32_t w[4][W];
};

template <int BN, bool OBF, bool RES>
__device__ __forceinline__ void epi_load_res(const GemmParams& p, EpiRes<OBF>& rr, int lane, int m0,
                                             int n0, int c, bool full, int n_lim) {
    if (!RES) return;
    using T = typename std::conditional<OBF, __nv_bfloat16, float>::type;
    const T* res = static_cast<const T*>(p.res);
    const int tr = lane >> 2, n = n0 + c + (lane & 3) * 8;
    const bool store = !(p.flags & kGemmFlagNoStore);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = int64_t(m0) + tr + 8 * i;
        const bool ok = store && (full || (gm < p.M && n < n_lim)) && n < n_lim;
        const T* src = res + (ok ? gm * p.res_ld + n : 0);
        uint4 a = make_uint4(0u, 0u, 0u, 0u), b = a;
        if (ok) {
            a = __ldg(reinterpret_cast<const uint4*>(src));
            if (!OBF) b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
        }
        rr.w[i][0] = a.x;
        rr.w[i][1] = a.y;
        rr.w[i][2] = a.z;
        rr.w[i][3] = a.w;
        if (!OBF) {
            rr.w[i][4 % EpiRes<OBF>::W] = b.x;
            rr.w[i][5 % EpiRes<OBF>::W] = b.y;
            rr.w[i][6 % EpiRes<OBF>::W] = b.z;
            rr.w[i][7 % EpiRes<OBF>::W] = b.w;
        }
    }
}

// Per-column epilogue vectors of a lane's 8 columns in one chunk: bias, and the residual
// scale (GemmParams::res_scale, GroupNorm folding). Fetched one chunk ahead, like the
// residual, so their load latency is not exposed.
struct EpiCol {
    float b[8], s[8];
};
template <bool RES>
__device__ __forceinline__ void epi_load_col(const GemmParams& p, EpiCol& col, int lane, int n0, int c,
                                             int n_lim) {
    const int n = n0 + c + (lane & 3) * 8;
    const bool okb = p.bias && n < n_lim;
    const float4 b0 = okb ? __ldg(reinterpret_cast<const float4*>(p.bias + n)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b1 = okb ? __ldg(reinterpret_cast<const float4*>(p.bias + n) + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
    col.b[0] = b0.x; col.b[1] = b0.y; col.b[2] = b0.z; col.b[3] = b0.w;
    col.b[4] = b1.x; col.b[5] = b1.y; col.b[6] = b1.z; col.b[7] = b1.w;
    if (RES && p.res_scale) {
        const int nc = min(n, n_lim - 8);
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.res_scale + nc));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.res_scale + nc) + 1);
        col.s[0] = s0.x; col.s[1] = s0.y; col.s[2] = s0.z; col.s[3] = s0.w;
        col.s[4] = s1.x; col.s[5] = s1.y; col.s[6] = s1.z; col.s[7] = s1.w;
    }
}

// Column statistics accumulated per (CTA, epilogue warp) over all of the CTA's tiles, used
// when every CTA keeps one column tile (gridDim.x % n_tiles == 0): after the butterfly, lane
// l keeps column (l & 3) * 8 + (l >> 2) of each of its chunks (<= 4 per tile), in a fixed
// order, so the partial rows drop from M / 32 to 4 per CTA (the fold reads 13x less at the
// block's shapes) and stay deterministic.
struct CtaStats {
    float s[4], q[4];
};

template <int BN, bool OBF, bool RES, bool ST>
__device__ __forceinline__ void epilogue_tile(const GemmParams& p, uint32_t tmem_acc, int q, int lane,
                                              uint32_t stg, int m0, int n0, int half,
                                              EpiRes<OBF>& rr, EpiCol& col, CtaStats* cst = nullptr) {
    using T = typename std::conditional<OBF, __nv_bfloat16, float>::type;
    const int tr = lane >> 2;        // transposed: rows tr + 8i
    const int tc = (lane & 3) * 8;   // transposed: first of 8 columns
    const int n_lim = min(p.N, n0 + BN);
    const bool full = (m0 + 32 <= p.M) && (n0 + BN <= p.N);
    const bool store = !(p.flags & kGemmFlagNoStore);
    T* out = static_cast<T*>(p.out);
    // rr and col already hold this warp's first chunk (loaded before the accumulator was ready)
#pragma unroll 1
    for (int c = 32 * half; c < BN; c += 64) {
        const EpiCol cc = col;
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_acc + (uint32_t(q * 32) << 16) + c, r);
        dev::tmem_wait_ld();
        if (n0 + c >= n_lim) continue;  // warp-uniform: past the matrix edge
        const uint32_t srow = stg + uint32_t(lane * kStgPitch * 4);
#pragma unroll
        for (int j = 0; j < 8; ++j) sts128(srow + 16 * j, r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        __syncwarp();
        float cur[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t a = stg + uint32_t(((tr + 8 * i) * kStgPitch + tc) * 4);
            const float4 v0 = lds128(a), v1 = lds128(a + 16);
            cur[i][0] = v0.x; cur[i][1] = v0.y; cur[i][2] = v0.z; cur[i][3] = v0.w;
            cur[i][4] = v1.x; cur[i][5] = v1.y; cur[i][6] = v1.z; cur[i][7] = v1.w;
            if (RES) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    float r;
                    if (OBF) {
                        const uint32_t w = rr.w[i][k >> 1];
                        r = __uint_as_float((k & 1) ? (w & 0xFFFF0000u) : (w << 16));
                    } else {
                        r = __uint_as_float(rr.w[i][k % EpiRes<OBF>::W]);
                    }
                    cur[i][k] = p.res_scale ? fmaf(r, cc.s[k], cur[i][k]) : cur[i][k] + r;
                }
            }
        }
        __syncwarp();
        if (c + 64 < BN && n0 + c + 64 < n_lim) {  // next chunk
            epi_load_res<BN, OBF, RES>(p, rr, lane, m0, n0, c + 64, full, n_lim);
            epi_load_col<RES>(p, col, lane, n0, c + 64, n_lim);
        }
        if (!store) continue;
        const int n = n0 + c + tc;
        const float* b8 = cc.b;
        float cs[8], cq[8];  // column stats of the stored values
#pragma unroll
        for (int k = 0; k < 8; ++k) cs[k] = cq[k] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gm = int64_t(m0) + tr + 8 * i;
            if (!full && (gm >= p.M || n >= n_lim)) continue;
            // BN not a multiple of 32 (e.g. 240): the last chunk of an interior tile would
            // spill into the next tile's columns
            if (BN % 32 != 0 && n >= n_lim) continue;
            T* dst = out + gm * p.out_ld + n;
            float y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = cur[i][k] + b8[k];
            if (OBF) {
                uint32_t w[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * h], y[2 * h + 1]);
                    w[h] = *reinterpret_cast<const uint32_t*>(&b2);
                    if (ST) {  // statistics of the stored (rounded) values
                        y[2 * h] = __low2float(b2);
                        y[2 * h + 1] = __high2float(b2);
                    }
                }
                *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
            } else if (p.out_lo) {
                uint32_t wh[4], wl[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * h], y[2 * h + 1]);
                    const __nv_bfloat162 l2 = __floats2bfloat162_rn(y[2 * h] - __low2float(b2),
                                                                    y[2 * h + 1] - __high2float(b2));
                    wh[h] = *reinterpret_cast<const uint32_t*>(&b2);
                    wl[h] = *reinterpret_cast<const uint32_t*>(&l2);
                }
                const int64_t o = gm * p.out_ld + n;
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + o) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out_lo) + o) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            } else {
                *reinterpret_cast<float4*>(dst) = make_float4(y[0], y[1], y[2], y[3]);
                *reinterpret_cast<float4*>(dst + 4) = make_float4(y[4], y[5], y[6], y[7]);
            }
            if (ST) {  // statistics of the stored value minus the bias (groupnorm.cu colpart_entry)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float v = y[k] - b8[k];
                    cs[k] += v;
                    cq[k] = fmaf(v, v, cq[k]);
                }
            }
        }
        if (ST) {
            // lanes l ^ {4, 8, 16} hold the same 8 columns for the block's other rows
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[k] += __shfl_xor_sync(0xffffffffu, cs[k], 4);
                cs[k] += __shfl_xor_sync(0xffffffffu, cs[k], 8);
                cs[k] += __shfl_xor_sync(0xffffffffu, cs[k], 16);
                cq[k] += __shfl_xor_sync(0xffffffffu, cq[k], 4);
                cq[k] += __shfl_xor_sync(0xffffffffu, cq[k], 8);
                cq[k] += __shfl_xor_sync(0xffffffffu, cq[k], 16);
            }
            if (cst) {
                const int kk = lane >> 2;
                float ss = cs[0], sq = cq[0];
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (kk == k) {
                        ss = cs[k];
                        sq = cq[k];
                    }
                const int jc = (c - 32 * half) >> 6;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j == jc) {
                        cst->s[j] += ss;
                        cst->q[j] += sq;
                    }
            } else if (tr == 0 && n < n_lim && m0 < p.M) {  // this warp owns (row block, 8 columns)
                float* part = p.colpart + int64_t(m0 >> 5) * 2 * p.N + n;
                *reinterpret_cast<float4*>(part) = make_float4(cs[0], cs[1], cs[2], cs[3]);
                *reinterpret_cast<float4*>(part + 4) = make_float4(cs[4], cs[5], cs[6], cs[7]);
                *reinterpret_cast<float4*>(part + p.N) = make_float4(cq[0], cq[1], cq[2], cq[3]);
                *reinterpret_cast<float4*>(part + p.N + 4) = make_float4(cq[4], cq[5], cq[6], cq[7]);
            }
        }
    }
}

// TMA-store epilogue (bf16 output, no residual, no column statistics: the Q/K/V
// projections). A lane converts its accumulator row's 32 columns to bf16 and writes them
// (64 B) into the warp's staging block in the TMA box layout (32 x 32, 64B swizzle: 16 B
// chunk j of row r sits at chunk j ^ ((r >> 1) & 3), conflict-free); one lane then stores
// the block with cp.async.bulk.tensor. Half the smem traffic of the fp32 transpose, and
// full-line writes without per-lane store instructions. Two staging blocks per warp
// alternate; a block is rewritten only after its previous store has read it. A partial
// 16-column chunk (BN = 240) goes out as direct 16-byte row stores.
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t smem_src, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(smem_src)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int BN>
__device__ __forceinline__ void epilogue_tile_tma(const GemmParams& p, const CUtensorMap* omap,
                                                  uint32_t tmem_acc, int q, int lane, uint32_t stg,
                                                  int m0, int n0, int half, uint32_t& nstore) {
    const int n_lim = min(p.N, n0 + BN);
    const bool store = !(p.flags & kGemmFlagNoStore);
#pragma unroll 1
    for (int c = 32 * half; c < BN; c += 64) {
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_acc + (uint32_t(q * 32) << 16) + c, r);
        dev::tmem_wait_ld();
        const int nb = n0 + c;
        if (nb >= n_lim || !store) continue;  // warp-uniform
        float y[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) y[k] = __uint_as_float(r[k]);
        if (p.bias) {
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                if (nb + 4 * v < n_lim) {
                    const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + nb) + v);
                    y[4 * v] += b.x;
                    y[4 * v + 1] += b.y;
                    y[4 * v + 2] += b.z;
                    y[4 * v + 3] += b.w;
                }
            }
        }
        uint32_t w[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * h], y[2 * h + 1]);
            w[h] = *reinterpret_cast<const uint32_t*>(&b2);
        }
        if (BN % 32 != 0 && nb + 32 > n0 + BN) {
            // partial chunk of a 240-wide tile: 16 columns, direct row stores
            const int64_t gm = int64_t(m0) + lane;
            if (gm < p.M) {
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + gm * p.out_ld + nb;
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (nb + 8 * v < n_lim)
                        *reinterpret_cast<uint4*>(dst + 8 * v) =
                            make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
            }
            continue;
        }
        const uint32_t buf = stg + (nstore & 1) * 2048;
        if (p.flags & kGemmFlagDiagNoSts) {  // diagnostics: no staging, no store
            if (w[0] == 0x7fc17fc1u && w[15] == 0x7fc17fc1u) static_cast<uint32_t*>(p.out)[lane] = w[7];
            continue;
        }
        const bool tma = !(p.flags & kGemmFlagDiagNoTma);
        if (nstore >= 2 && tma) {  // the store that last used this block has finished reading it
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
        }
        const uint32_t row = buf + lane * 64, sw = (lane >> 1) & 3;
#pragma unroll
        for (int j = 0; j < 4; ++j) sts128(row + ((j ^ sw) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        dev::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && tma) {
            // diagnostics: kGemmFlagDiagL2Out folds the rows onto 1024 (output stays in L2)
            tma_store_2d(omap, buf, nb, (p.flags & kGemmFlagDiagL2Out) ? (m0 & 1023) : m0);
            dev::bulk_commit();
        }
        ++nstore;
    }
}

// Residual through TMA (RT flavour: bf16 output + bf16 residual, e.g. the O projection,
// whose epilogue moves two bytes of HBM traffic for every byte of A). Each epilogue warp
// streams the 32 x 32 residual boxes of its own (tile, chunk) sequence through a private
// kResSlots-deep ring (64B swizzle, the store staging's layout, so a lane reads its
// accumulator row's 32 values conflict-free without a transpose). Loads run kResSlots boxes
// ahead, across tile boundaries, and hold no registers.
struct ResRing {
    uint32_t base;   // smem address of slot 0 of this warp's ring
    uint64_t* bar;   // kResSlots mbarriers
    uint32_t ncons;  // boxes consumed
    uint32_t nload;  // boxes issued
    int lt, lc;      // next box to issue: tile, chunk column
    uint32_t lloc;   // lt's index among this CTA's tiles (its parity swaps the warp's chunks)
    int h0;          // the warp's chunk parity on its even tiles
    bool pend;       // the slot consumed last holds an output box still being stored
};

template <int BN>
__device__ __forceinline__ void res_seek(const GemmParams& p, ResRing& rg, int n_tiles, int num_tiles) {
    // move (lt, lc) to the first box at or after it that lies inside the matrix (chunk parity
    // h0 on the warp's even tiles, swapped on odd ones, as the epilogue takes them)
    while (rg.lt < num_tiles) {
        const int n0 = (rg.lt % n_tiles) * BN;
        if (rg.lc < BN && n0 + rg.lc < min(p.N, n0 + BN)) return;
        rg.lt += gridDim.x;
        ++rg.lloc;
        rg.lc = 32 * (rg.h0 ^ int(rg.lloc & 1));
    }
}

template <int BN>
__device__ __forceinline__ void res_issue(const GemmParams& p, const CUtensorMap* rmap, ResRing& rg,
                                          int n_tiles, int num_tiles, int q) {
    // lane 0 only
    if (rg.lt >= num_tiles) return;
    const uint32_t slot = rg.nload % kResSlots;
    const int m0 = (rg.lt / n_tiles) * kBM + q * 32, n0 = (rg.lt % n_tiles) * BN;
    dev::mbar_arrive_expect_tx(&rg.bar[slot], 2048);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(rg.base + slot * 2048),
        "l"(reinterpret_cast<uint64_t>(rmap)), "r"(n0 + rg.lc), "r"(m0), "r"(dev::smem_u32(&rg.bar[slot]))
        : "memory");
    ++rg.nload;
    rg.lc += 64;
    res_seek<BN>(p, rg, n_tiles, num_tiles);
}

template <int BN>
__device__ __forceinline__ void epilogue_tile_tma_res(const GemmParams& p, const CUtensorMap* omap,
                                                      const CUtensorMap* rmap, uint32_t tmem_acc, int q,
                                                      int lane, uint32_t stg, int m0, int n0, int half,
                                                      uint32_t& nstore, ResRing& rg, int n_tiles,
                                                      int num_tiles) {
    static_assert(BN % 32 == 0, "whole 32-column chunks");
    const int n_lim = min(p.N, n0 + BN);
    const bool store = !(p.flags & kGemmFlagNoStore);
    const uint32_t sw = (lane >> 1) & 3;
#pragma unroll 1
    for (int c = 32 * half; c < BN; c += 64) {
        const int nb = n0 + c;
        if (nb >= n_lim) break;  // warp-uniform; the ring holds only in-range boxes
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_acc + (uint32_t(q * 32) << 16) + c, r);
        // this chunk's residual box
        const uint32_t slot = rg.ncons % kResSlots;
        dev::mbar_wait(&rg.bar[slot], (rg.ncons / kResSlots) & 1);
        uint32_t rw[16];
        {
            const uint32_t row = rg.base + slot * 2048 + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 v = lds128(row + ((j ^ sw) << 4));
                rw[4 * j] = __float_as_uint(v.x);
                rw[4 * j + 1] = __float_as_uint(v.y);
                rw[4 * j + 2] = __float_as_uint(v.z);
                rw[4 * j + 3] = __float_as_uint(v.w);
            }
        }
        ++rg.ncons;
        __syncwarp();
        if (!store && lane == 0) {  // the slot is read: refill it with the box kResSlots ahead
            dev::fence_proxy_async_smem();
            res_issue<BN>(p, rmap, rg, n_tiles, num_tiles, q);
        }
        dev::tmem_wait_ld();
        float y[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            float4 b = make_float4(0.f, 0.f, 0.f, 0.f), sc = b;
            const bool okv = nb + 4 * v < n_lim;  // N % 8 == 0: a float4 is wholly in or out
            if (p.bias && okv) b = __ldg(reinterpret_cast<const float4*>(p.bias + nb) + v);
            if (p.res_scale && okv) sc = __ldg(reinterpret_cast<const float4*>(p.res_scale + nb) + v);
            const float bb[4] = {b.x, b.y, b.z, b.w}, ss[4] = {sc.x, sc.y, sc.z, sc.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * v + e;
                const uint32_t w = rw[k >> 1];
                const float rv = __uint_as_float((k & 1) ? (w & 0xFFFF0000u) : (w << 16));
                const float a = __uint_as_float(r[k]);
                // the transposed epilogue's arithmetic: (acc + res*scale) + bias
                const float cur = p.res_scale ? fmaf(rv, ss[e], a) : a + rv;
                y[k] = cur + bb[e];
            }
        }
        if (!store) continue;
        uint32_t w[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * h], y[2 * h + 1]);
            w[h] = *reinterpret_cast<const uint32_t*>(&b2);
        }
        // the output box is staged in the residual slot just read (same 64B-swizzled box
        // layout; every lane's reads are done at the __syncwarp above): no separate staging,
        // which leaves the operand ring a fourth stage. The slot is refilled one chunk later,
        // once this store has read it.
        const uint32_t row = rg.base + slot * 2048 + lane * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) sts128(row + ((j ^ sw) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        dev::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(omap, rg.base + slot * 2048, nb, m0);
            dev::bulk_commit();
            if (rg.pend) {  // the previous chunk's slot: its store has read it once <= 1 is pending
                bulk_wait_read<1>();
                res_issue<BN>(p, rmap, rg, n_tiles, num_tiles, q);
            }
        }
        rg.pend = true;
        ++nstore;
    }
}

template <int BN, bool OBF, bool RES, bool ST, bool TMAO = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ GemmParams p) {
    constexpr bool RT = TMAO && RES;  // residual through TMA (the RT flavour)
    using Cfg = TileCfg<BN, ST, RT, TMAO>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;   // [2]
    uint64_t* tempty = tfull + 2;  // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    uint64_t* rbar = full + 32;    // RT: [kEpiWarps][kResSlots] residual ring barriers

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const int n_tiles = (p.N + BN - 1) / BN;
    const int m_tiles = (p.M + kBM - 1) / kBM;
    const int num_tiles = n_tiles * m_tiles;
    const int kb_per_seg = (p.K + kBK - 1) / kBK;
    const int k_iters = kb_per_seg * p.nseg;

    if (warp == 0 && lane == 0) {
        dev::tma_prefetch_desc(&maps.a[0]);
        dev::tma_prefetch_desc(&maps.a[1]);
        dev::tma_prefetch_desc(&maps.b[0]);
        dev::tma_prefetch_desc(&maps.b[1]);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            dev::mbar_init(&full[s], 1);
            dev::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            dev::mbar_init(&tfull[i], 1);
            dev::mbar_init(&tempty[i], kEpiWarps);
        }
        if (RT)
            for (int i = 0; i < kEpiWarps * kResSlots; ++i) dev::mbar_init(&rbar[i], 1);
        dev::fence_barrier_init();
    }
    if (warp == 2) dev::tmem_alloc(tmem_holder, Cfg::kTmemCols);
    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // the prologue above overlaps the previous kernel's tail (programmatic launch)
    dev::pdl_wait();
    dev::pdl_trigger();

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m0 = (tile / n_tiles) * kBM;
                const int n0 = (tile % n_tiles) * BN;
                for (int k = 0; k < k_iters; ++k, ++it) {
                    const uint32_t s = it % S;
                    const uint32_t ph = (it / S) & 1;
                    dev::mbar_wait(&empty[s], ph ^ 1);
                    dev::mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
                    const GemmSeg& sg = p.seg[k / kb_per_seg];
                    const int kk = (k % kb_per_seg) * kBK;
                    dev::tma_load_2d(smem_a + s * kABytes, &maps.a[sg.a_map], &full[s], kk,
                                     m0 + sg.a_row);
                    dev::tma_load_2d(smem_b + s * Cfg::kBBytes, &maps.b[sg.b_map], &full[s], kk,
                                     n0 + sg.b_row);
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        constexpr uint32_t idesc = dev::idesc_bf16_f32(kBM, BN);
        uint32_t it = 0;
        uint32_t local = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const uint32_t acc = local & 1;
            dev::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
            dev::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * Cfg::kAccStride;
            for (int k = 0; k < k_iters; ++k, ++it) {
                const uint32_t s = it % S;
                const uint32_t ph = (it / S) & 1;
                dev::mbar_wait(&full[s], ph);
                dev::tc_fence_after();
                if (lane == 0) {
                    const uint64_t ad = dev::sw128_kmajor_desc(dev::smem_u32(smem_a + s * kABytes));
                    const uint64_t bd =
                        dev::sw128_kmajor_desc(dev::smem_u32(smem_b + s * Cfg::kBBytes));
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        // advance 16 bf16 = 32 bytes along K inside the 128B swizzle atom
                        dev::umma_bf16(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc,
                                       (k > 0 || kk > 0) ? 1u : 0u);
                    }
                    dev::umma_commit(&empty[s]);
                    if (k == k_iters - 1) dev::umma_commit(&tfull[acc]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ===== Epilogue =====
        const int q = warp & 3;            // TMEM lane quadrant this warp may access
        const int half = (warp - 4) >> 2;  // which alternate 32-column chunks it takes
        const uint32_t stg =
            dev::smem_u32(smem + S * Cfg::kStageBytes + 1024) + (warp - 4) * Cfg::kStgWarp;
        uint32_t local = 0, nstore = 0;
        EpiRes<OBF> rr;
        EpiCol col;
        ResRing rg;
        // ST: per-CTA column statistics when this CTA's column tile never changes
        const bool cta_stats = ST && (gridDim.x % n_tiles) == 0;
        CtaStats cst;
#pragma unroll
        for (int j = 0; j < 4; ++j) cst.s[j] = cst.q[j] = 0.f;
        if (RT) {
            rg.base = dev::smem_u32(smem + S * Cfg::kStageBytes + 1024 + Cfg::kStg) +
                      (warp - 4) * (kResSlots * 2048);
            rg.bar = rbar + (warp - 4) * kResSlots;
            rg.ncons = rg.nload = 0;
            rg.lt = blockIdx.x;
            rg.lloc = 0;
            rg.h0 = half;
            rg.lc = 32 * half;
            rg.pend = false;
            res_seek<BN>(p, rg, n_tiles, num_tiles);
            if (lane == 0) {
                dev::tma_prefetch_desc(&maps.res);
                for (int i = 0; i < kResSlots; ++i) res_issue<BN>(p, &maps.res, rg, n_tiles, num_tiles, q);
            }
        }
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const uint32_t acc = local & 1;
            const int m0 = (tile / n_tiles) * kBM + q * 32, n0 = (tile % n_tiles) * BN;
            if (!TMAO) {  // the residual does not depend on the accumulator: fetch it early
                const int n_lim = min(p.N, n0 + BN);
                const bool full = (m0 + 32 <= p.M) && (n0 + BN <= p.N);
                if (n0 + 32 * half < n_lim) {
                    epi_load_res<BN, OBF, RES>(p, rr, lane, m0, n0, 32 * half, full, n_lim);
                    epi_load_col<RES>(p, col, lane, n0, 32 * half, n_lim);
                }
            }
            dev::mbar_wait(&tfull[acc], (local >> 1) & 1);
            dev::tc_fence_after();
            // TMA epilogues: the two warps of a quadrant swap chunk parity every tile, so an odd
            // chunk count (BN = 160: 3 + 2, 224: 4 + 3) balances over two tiles (the accumulator
            // is double-buffered: the lighter warp runs ahead into the next tile)
            const int hsw = half ^ int(local & 1);
            if constexpr (RT)
                epilogue_tile_tma_res<BN>(p, &maps.out, &maps.res, tmem_base + acc * Cfg::kAccStride, q,
                                          lane, stg, m0, n0, hsw, nstore, rg, n_tiles, num_tiles);
            else if constexpr (TMAO)
                epilogue_tile_tma<BN>(p, &maps.out, tmem_base + acc * Cfg::kAccStride, q, lane, stg,
                                      m0, n0, hsw, nstore);
            else
                epilogue_tile<BN, OBF, RES, ST>(p, tmem_base + acc * Cfg::kAccStride, q, lane, stg, m0,
                                                n0, half, rr, col, cta_stats ? &cst : nullptr);
            dev::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (TMAO && lane == 0) bulk_wait_read<0>();  // staging must outlive the stores' reads
        if (cta_stats && !(p.flags & kGemmFlagNoStore)) {
            // partial row (CTA group, quadrant): the n_tiles CTAs of a group cover every column once
            const int n0 = (blockIdx.x % n_tiles) * BN, n_lim = min(p.N, n0 + BN);
            float* part = p.colpart + (int64_t(blockIdx.x / n_tiles) * 4 + q) * 2 * p.N;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + 32 * half + 64 * j + (lane & 3) * 8 + (lane >> 2);
                if (32 * half + 64 * j < BN && n < n_lim) {
                    part[n] = cst.s[j];
                    part[p.N + n] = cst.q[j];
                }
            }
        }
    }

    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    if (warp == 2) dev::tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

int g_num_sms = 0;

template <int BN, bool OBF, bool RES, bool ST = false, bool TMAO = false>
int launch_cfg(const GemmMaps& maps, const GemmParams& p, cudaStream_t stream) {
    using Cfg = TileCfg<BN, ST, TMAO && RES, TMAO>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, OBF, RES, ST, TMAO>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(Cfg::kSmemBytes));
        if (e != cudaSuccess) return int(e);
        attr_set = true;
    }
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    const int n_tiles = (p.N + BN - 1) / BN;
    const int tiles = n_tiles * ((p.M + kBM - 1) / kBM);
    int grid = std::max(1, std::min(tiles, g_num_sms));
    // column statistics: a grid that is a multiple of the column tiles keeps every CTA on
    // one column tile (per-CTA statistics, gemm_colpart_rows)
    if (ST && grid > n_tiles) grid -= grid % n_tiles;
    return int(launch_pdl(gemm_tc_kernel<BN, OBF, RES, ST, TMAO>, dim3(grid), dim3(kThreads),
                          Cfg::kSmemBytes, stream, maps, p));
}

template <int BN>
int launch(const GemmMaps& maps, const GemmParams& p, cudaStream_t stream) {
    const bool res = p.res != nullptr;
    if (res && p.res_bf16 != p.out_bf16) return int(cudaErrorInvalidValue);
    if (p.colpart) {  // fused GroupNorm statistics: the conv flavour (residual present)
        if (!res) return int(cudaErrorInvalidValue);
        return p.out_bf16 ? launch_cfg<BN, true, true, true>(maps, p, stream)
                          : launch_cfg<BN, false, true, true>(maps, p, stream);
    }
    if (p.out_bf16 && !res && (p.flags & kGemmFlagTmaOut))
        return launch_cfg<BN, true, false, false, true>(maps, p, stream);
    if constexpr (BN % 32 == 0) {
        if (p.out_bf16 && res && (p.flags & kGemmFlagTmaRes))
            return launch_cfg<BN, true, true, false, true>(maps, p, stream);
    }
    if (p.out_bf16) return res ? launch_cfg<BN, true, true>(maps, p, stream)
                               : launch_cfg<BN, true, false>(maps, p, stream);
    return res ? launch_cfg<BN, false, true>(maps, p, stream)
               : launch_cfg<BN, false, false>(maps, p, stream);
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t ld_elems, uint32_t box_rows) {
    auto fn = get_encode_fn();
    if (!fn) return int(cudaErrorNotSupported);
    cuuint64_t gdim[2] = {cols, rows};
    cuuint64_t gstride[1] = {ld_elems * 2};
    cuuint32_t box[2] = {uint32_t(kBK), box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim,
                    gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

int make_tmap_out_bf16(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems) {
    auto fn = get_encode_fn();
    if (!fn) return int(cudaErrorNotSupported);
    cuuint64_t gdim[2] = {cols, rows};
    cuuint64_t gstride[1] = {ld_elems * 2};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gdim, gstride, box, estride,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

int gemm_colpart_rows(int64_t M, int N) {
    const int bn = gemm_pick_block_n(N);
    const int64_t rb = (M + 31) / 32;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    const int64_t n_tiles = (N + bn - 1) / bn, tiles = n_tiles * ((M + kBM - 1) / kBM);
    int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, g_num_sms));
    if (grid > n_tiles) grid -= grid % n_tiles;  // as launch_cfg does for the statistics kernels
    return int(grid % n_tiles == 0 ? grid / n_tiles * 4 : rb);
}

int gemm_pick_block_n(int N) {
    // Wide tiles feed the tensor pipe best (more MMA work per operand byte and per
    // instruction: at M = 61440, K = 640 the main loop runs at ~1550 TFLOP/s with N = 240
    // against ~1200 with N = 160), so take the widest tile that pads N by less than 1/16;
    // otherwise the least padding. (N = 640: 224; N = 1920: 240; N = 1280: 256; N = 320: 160.)
    static const int cands[] = {256, 240, 224, 192, 160, 128, 64};
    static const int forced = env_int("VINF_GEMM_BN", 0);  // diagnostics
    for (int bn : cands)
        if (bn == forced) return bn;
    for (int bn : cands) {
        if (bn < 192) break;
        const long padded = long((N + bn - 1) / bn) * bn;
        if (16 * (padded - N) < padded) return bn;
    }
    int best = 64;
    long best_waste = -1;
    for (int bn : cands) {
        const long tiles = (N + bn - 1) / bn;
        const long waste = tiles * bn - N;
        if (best_waste < 0 || waste < best_waste) {
            best = bn;
            best_waste = waste;
        }
    }
    return best;
}

int gemm_tc_launch(const GemmMaps& maps, const GemmParams& p, int block_n, cudaStream_t stream) {
    if (p.M <= 0 || p.N <= 0 || p.N % 8 != 0 || p.K <= 0 || p.nseg <= 0 || p.nseg > kGemmMaxSeg)
        return int(cudaErrorInvalidValue);
    switch (block_n) {
        case 256: return launch<256>(maps, p, stream);
        case 240: return launch<240>(maps, p, stream);
        case 224: return launch<224>(maps, p, stream);
        case 192: return launch<192>(maps, p, stream);
        case 160: return launch<160>(maps, p, stream);
        case 128: return launch<128>(maps, p, stream);
        case 64: return launch<64>(maps, p, stream);
        default: return int(cudaErrorInvalidValue);
    }
}

}  // namespace vinf
