// Fused Q/K/V projection + dual-scope attention core (bf16 mode), for clips whose every
// K/V token is one of the clip's own frames (the single-worker layout: BASELINE configs[1]).
//
// The unfused path writes Q/K/V (3 x 79 MB at cfg2) to HBM in the projection GEMM and
// reads it back in the attention core. Here one CTA owns P spatial positions x F frames
// (P*F <= 128 rows): it keeps the normalised activations of those rows resident in shared
// memory (TMA 3D box {64 channels, P positions, F frames}, 128B swizzle) and streams the
// projection weights through a 4-deep ring; tcgen05 computes the projection 64 channels at
// a time (N = 128 for a [Q | K] chunk, N = 64 for a V chunk) into a double-buffered TMEM
// accumulator. Eight worker warps turn each chunk into bf16 in shared memory (the same
// rounding as the GEMM epilogue) and consume it with warp MMAs: S += Q_c K_c^T over the QK
// chunks (the lean kernel's k order), the token softmax, then ctx_c = P V_c per V chunk.
// Only ctx leaves the SM. Numerics are the unfused path's: bitwise equal outputs.
//
// The kernel runs on CTA pairs (cluster of 2, tcgen05 cta_group::2): each CTA keeps its own
// positions' rows resident, the pair's MMA has M = 256, and each CTA streams only half of
// every weight tile ([Q|K] chunk: CTA 0 the 64 Q rows, CTA 1 the 64 K rows; V chunk: 32
// rows each). Halving the weight bytes per SM doubles the ring depth the shared memory left
// by the resident rows can hold, which is what the projection needs to stay fed.
//
// Roles (384 threads per CTA): warp 0 TMA producer, warp 1 MMA issuer (leader CTA),
// warp 2 TMEM allocator, warps 4..11 workers (worker w: position w >> 1, query rows
// 16 (w & 1) .. +15 of its CTA's positions).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kFuThreads = 12 * 32;
constexpr int kFuWorkers = 8;
constexpr int kFuWStages = 8;
constexpr uint32_t kFuWStage = 64 * 128;   // this CTA's half of a W tile: <= 64 rows x 64 k
constexpr int kFuPmax = 4;                 // positions per CTA (2 workers each)
constexpr int kFuSP = 28;                  // fp32 pitch of S rows (24 key columns + pad)

struct FuLay {
    uint32_t arows, a_blk, nkb, a, w, x0, x1, bars, total;
    __host__ __device__ FuLay(uint32_t P, uint32_t F, uint32_t C) {
        arows = (P * F + 7) & ~7u;     // whole 8-row swizzle atoms
        a_blk = arows * 128;           // one 64-channel k-block of the resident rows
        nkb = C / 64;
        a = 0;
        w = (a + nkb * a_blk + 1023) & ~1023u;
        x0 = w + kFuWStages * kFuWStage;
        x1 = x0 + 128 * 128;
        bars = x1 + 128 * 128;
        // the last k-block's MMA reads 128 rows: keep the over-read inside the allocation
        total = bars + 256 + 1024;
    }
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(dev::smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dev::smem_u32(bar)) : "memory");
}
// byte offset of 16-byte chunk `c` of staging row `r` (128 B rows, XOR swizzle)
__device__ __forceinline__ uint32_t xsw(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

struct FuMaps {
    CUtensorMap u2;   // [af frames][HW][C] bf16, box {64, P, F}, SW128
    CUtensorMap w;    // [3C][C] bf16, box {64, 64 rows}, SW128
    CUtensorMap w32;  // [3C][C] bf16, box {64, 32 rows}, SW128
};
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const void* tmap, uint32_t bar_leader, int32_t c0,
                                                 int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_leader)
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFuThreads, 1)
    qkv_attention_fused_kernel(const __grid_constant__ FuMaps maps, uint32_t HW, uint32_t C, uint32_t F,
                               uint32_t P, uint32_t f_own0, TokenTable tt, float scale, float bias,
                               __nv_bfloat16* __restrict__ ctx, uint32_t stagger) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const FuLay L(P, F, C);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* empty = full + kFuWStages;
    uint64_t* tfull = empty + kFuWStages;  // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint64_t* abar = tempty + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(abar + 1);
    const uint32_t sbase = dev::smem_u32(sm);
    const uint32_t nch = C / 64, nchunks = 2 * nch;
    const uint32_t p0 = blockIdx.x * P;
    const uint32_t rank = dev::cluster_rank();
    const bool leader = rank == 0;
    // channel chunk processed at step j of each phase (rotated per CTA when staggering, so
    // concurrent CTAs stream different weight rows)
    const uint32_t rot = stagger ? blockIdx.x % nch : 0;
    auto chan = [&](uint32_t j) { return ((j < nch ? j : j - nch) + rot) % nch; };

    if (warp == 0 && lane == 0) {
        dev::tma_prefetch_desc(&maps.u2);
        dev::tma_prefetch_desc(&maps.w);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < kFuWStages; ++s) {
            dev::mbar_init(&full[s], 1);
            dev::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            dev::mbar_init(&tfull[i], 1);
            dev::mbar_init(&tempty[i], 2 * kFuWorkers);  // both CTAs' workers (leader's is used)
        }
        dev::mbar_init(abar, 1);
        dev::fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         dev::smem_u32(tmem_holder)),
                     "r"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    dev::tc_fence_before();
    dev::cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated in both
    dev::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    dev::pdl_wait();
    dev::pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            // resident rows: every k-block of this CTA's P positions x F own frames; both
            // CTAs' loads complete on the leader's barriers
            const uint32_t abar_l = dev::peer_addr(dev::smem_u32(abar), 0);
            if (leader) dev::mbar_arrive_expect_tx(abar, 2 * L.nkb * P * F * 128);
            for (uint32_t kb = 0; kb < L.nkb; ++kb)
                tma_load_3d_pair(sbase + L.a + kb * L.a_blk, &maps.u2, abar_l, int32_t(kb * 64), int32_t(p0),
                                 int32_t(f_own0));
            uint32_t it = 0;
            for (uint32_t j = 0; j < nchunks; ++j) {
                const bool qk = j < nch;
                for (uint32_t kb = 0; kb < L.nkb; ++kb, ++it) {
                    const uint32_t s = it % kFuWStages;
                    dev::mbar_wait(&empty[s], ((it / kFuWStages) & 1) ^ 1);
                    const uint32_t full_l = dev::peer_addr(dev::smem_u32(&full[s]), 0);
                    if (leader) dev::mbar_arrive_expect_tx(&full[s], qk ? 2 * 64 * 128 : 2 * 32 * 128);
                    const uint32_t wst = sbase + L.w + s * kFuWStage;
                    if (qk)  // [Q | K] chunk: CTA 0 streams the Q rows, CTA 1 the K rows
                        dev::tma_load_2d_pair(wst, &maps.w, full_l, int32_t(kb * 64),
                                              int32_t(rank * C + chan(j) * 64));
                    else     // V chunk: 32 rows each
                        dev::tma_load_2d_pair(wst, &maps.w32, full_l, int32_t(kb * 64),
                                              int32_t(2 * C + chan(j) * 64 + rank * 32));
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            dev::mbar_wait(abar, 0);
            uint32_t it = 0;
            for (uint32_t j = 0; j < nchunks; ++j) {
                const bool qk = j < nch;
                const uint32_t buf = j & 1;
                dev::mbar_wait(&tempty[buf], ((j >> 1) & 1) ^ 1);
                dev::tc_fence_after();
                const uint32_t idesc = qk ? dev::idesc_bf16_f32(256, 128) : dev::idesc_bf16_f32(256, 64);
                for (uint32_t kb = 0; kb < L.nkb; ++kb, ++it) {
                    const uint32_t s = it % kFuWStages;
                    dev::mbar_wait(&full[s], (it / kFuWStages) & 1);
                    dev::tc_fence_after();
                    if (lane == 0) {
                        const uint64_t ad = dev::sw128_kmajor_desc(sbase + L.a + kb * L.a_blk);
                        const uint64_t bd = dev::sw128_kmajor_desc(sbase + L.w + s * kFuWStage);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            dev::umma_bf16_pair(tmem_base + buf * 128, ad + 2 * kk, bd + 2 * kk, idesc,
                                                (kb > 0 || kk > 0) ? 1u : 0u);
                        dev::umma_commit_pair(&empty[s]);
                        if (kb == L.nkb - 1) dev::umma_commit_pair(&tfull[buf]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp >= 4) {
        // ===== workers =====
        const int w = warp - 4;
        const int q = warp & 3;             // TMEM lane quadrant (rows 32q .. 32q+31)
        const int half = w >> 2;            // conversion: which 64 (QK) / 32 (V) columns
        const uint32_t pp = uint32_t(w >> 1);  // attention: position of this worker
        const int mt = w & 1;               // attention: query rows 16 mt .. 16 mt + 15
        const bool active = pp < P;
        const int g = lane >> 2, t4 = lane & 3;
        const uint32_t r7 = lane & 7, hi = lane >> 4, b1 = (lane >> 3) & 1;
        const uint32_t x0 = sbase + L.x0, x1 = sbase + L.x1;
        // staging row of (frame f, position pp): the resident rows' order (frame-major)
        auto row_of = [&](uint32_t f) { return min(f, F - 1) * P + pp; };
        const uint32_t qa_row = row_of(uint32_t(mt * 16) + r7 + b1 * 8);
        float acc[3][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        uint32_t pa[2][4];
        float* sp = reinterpret_cast<float*>(sm + L.x0);  // S / P scratch (after the QK phase)
        __shared__ float zinv_s[kFuPmax][32];

        for (uint32_t j = 0; j < nchunks; ++j) {
            const bool qk = j < nch;
            const uint32_t buf = j & 1;
            // ---- TMEM -> bf16 staging (Q_c in X0, K_c in X1; V_c in X0) ----
            dev::mbar_wait(&tfull[buf], (j >> 1) & 1);
            dev::tc_fence_after();
            {
                const uint32_t ncol = qk ? 64 : 32;  // this warp's columns of the chunk
                const uint32_t c0 = half * ncol;
                const uint32_t row = uint32_t(q * 32 + lane);
                for (uint32_t cc = 0; cc < ncol; cc += 32) {
                    uint32_t r[32];
                    dev::tmem_ld_32x32b_x32(tmem_base + buf * 128 + (uint32_t(q * 32) << 16) + c0 + cc, r);
                    dev::tmem_wait_ld();
                    // destination: QK: cols 0..63 -> X0 (Q), 64..127 -> X1 (K); V: X0
                    const uint32_t col = c0 + cc;  // first column of these 32
                    const uint32_t dst = (qk && col >= 64) ? x1 : x0;
                    const uint32_t dcol = qk ? (col & 63) : col;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        uint32_t wv[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[8 * k + 2 * h]),
                                                                            __uint_as_float(r[8 * k + 2 * h + 1]));
                            wv[h] = *reinterpret_cast<const uint32_t*>(&b2);
                        }
                        const uint32_t chunk16 = (dcol >> 3) + uint32_t(k);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + xsw(row, chunk16)),
                                     "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                                     : "memory");
                    }
                }
            }
            dev::tc_fence_before();
            __syncwarp();
            if (lane == 0) dev::mbar_arrive_remote(dev::peer_addr(dev::smem_u32(&tempty[buf]), 0));
            dev::named_bar(1, kFuWorkers * 32);
            if (qk) {
                // ---- S += Q_c K_c^T (query rows 16 mt.., 24 key frames = 3 n8 tiles) ----
                if (active) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint32_t a[4];
                        ldsm_x4(x0 + xsw(qa_row, uint32_t(kk * 2) + hi), a[0], a[1], a[2], a[3]);
#pragma unroll
                        for (int nt = 0; nt < 3; ++nt) {
                            const uint32_t krow = row_of(uint32_t(nt * 8) + r7);
                            uint32_t bb0, bb1;
                            ldsm_x2(x1 + xsw(krow, uint32_t(kk * 2) + b1), bb0, bb1);
                            mma_bf16(acc[nt], a[0], a[1], a[2], a[3], bb0, bb1);
                        }
                    }
                }
                dev::named_bar(1, kFuWorkers * 32);
                if (j == nch - 1) {
                    // ---- token softmax per query row -> P (bf16 fragments in registers) ----
                    if (active) {
#pragma unroll
                        for (int nt = 0; nt < 3; ++nt) {
                            const int col = nt * 8 + t4 * 2;
                            float* r0p = sp + (pp * 32 + uint32_t(mt * 16 + g)) * kFuSP;
                            r0p[col] = acc[nt][0];
                            r0p[col + 1] = acc[nt][1];
                            r0p[8 * kFuSP + col] = acc[nt][2];
                            r0p[8 * kFuSP + col + 1] = acc[nt][3];
                        }
                    }
                    dev::named_bar(1, kFuWorkers * 32);
                    for (uint32_t rr = uint32_t(w); rr < P * 32; rr += kFuWorkers) {
                        const uint32_t pos = rr >> 5, a_ = rr & 31;
                        float* row = sp + rr * kFuSP;
                        // per-column token softmax, as in the lean kernel (same bits)
                        float pv[2] = {0.f, 0.f};
                        float zi = 0.f;
                        if (a_ < F) {
                            const int lo = tt.wlo[a_], hi = tt.whi[a_];
                            const float bw = tt.wflag ? bias : 0.f, bg = tt.gflag ? bias : 0.f;
                            float sv[2];
                            bool inw[2];
                            int ng[2];
                            float m = -INFINITY;
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                const int c = lane + 32 * k;
                                const bool ok = c < int(F);
                                sv[k] = ok ? scale * row[c] : 0.f;
                                inw[k] = ok && c >= lo && c <= hi;
                                ng[k] = ok ? tt.gmult[c] : 0;
                                if (inw[k]) m = fmaxf(m, sv[k] + bw);
                                if (ng[k]) m = fmaxf(m, sv[k] + bg);
                            }
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                            float z = 0.f;
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                float p = inw[k] ? expf(sv[k] + bw - m) : 0.f;
                                if (ng[k]) {
                                    const float e = expf(sv[k] + bg - m);
                                    for (int t = 0; t < ng[k]; ++t) p += e;
                                }
                                pv[k] = p;
                                z += p;
                            }
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
                            zi = 1.0f / z;
                        }
                        __syncwarp();
                        if (lane < kFuSP) row[lane] = pv[0];
                        if (lane == 0) zinv_s[pos][a_] = zi;
                    }
                    dev::named_bar(1, kFuWorkers * 32);
                    if (active) {
                        // A fragments of P for k16 steps kq = 0, 1 (key columns 0..31; >= 24 zero)
                        const uint32_t ra = pp * 32 + uint32_t(mt * 16 + g), rb = ra + 8;
                        const float za = zinv_s[pp][mt * 16 + g], zb = zinv_s[pp][mt * 16 + g + 8];
                        auto pv = [&](uint32_t r, float zi, int c) -> float {
                            return c < 24 ? sp[r * kFuSP + c] * zi : 0.f;
                        };
#pragma unroll
                        for (int kq = 0; kq < 2; ++kq) {
                            const int c = kq * 16 + t4 * 2;
                            __nv_bfloat162 v0 = __floats2bfloat162_rn(pv(ra, za, c), pv(ra, za, c + 1));
                            __nv_bfloat162 v1 = __floats2bfloat162_rn(pv(rb, zb, c), pv(rb, zb, c + 1));
                            __nv_bfloat162 v2 = __floats2bfloat162_rn(pv(ra, za, c + 8), pv(ra, za, c + 9));
                            __nv_bfloat162 v3 = __floats2bfloat162_rn(pv(rb, zb, c + 8), pv(rb, zb, c + 9));
                            pa[kq][0] = *reinterpret_cast<uint32_t*>(&v0);
                            pa[kq][1] = *reinterpret_cast<uint32_t*>(&v1);
                            pa[kq][2] = *reinterpret_cast<uint32_t*>(&v2);
                            pa[kq][3] = *reinterpret_cast<uint32_t*>(&v3);
                        }
                    }
                    dev::named_bar(1, kFuWorkers * 32);  // scratch dead: X0/X1 reusable
                }
            } else {
                // ---- ctx_c = P V_c (16 query rows x 64 channels), rows < F stored ----
                if (active) {
                    const uint32_t vc = chan(j);
                    float o[8][4];
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
#pragma unroll
                    for (int kq = 0; kq < 2; ++kq) {
                        const uint32_t vrow = row_of(uint32_t(kq * 16) + r7 + b1 * 8);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            uint32_t b[4];
                            ldsm_x4_t(x0 + xsw(vrow, uint32_t(2 * i) + hi), b[0], b[1], b[2], b[3]);
                            mma_bf16(o[2 * i], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[0], b[1]);
                            mma_bf16(o[2 * i + 1], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[2], b[3]);
                        }
                    }
                    const uint32_t fa = uint32_t(mt * 16 + g), fb = fa + 8;
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) {
                        const uint32_t col = vc * 64 + uint32_t(nt * 8 + t4 * 2);
                        if (fa < F)
                            *reinterpret_cast<__nv_bfloat162*>(ctx + (uint64_t(fa) * HW + p0 + pp) * C + col) =
                                __floats2bfloat162_rn(o[nt][0], o[nt][1]);
                        if (fb < F)
                            *reinterpret_cast<__nv_bfloat162*>(ctx + (uint64_t(fb) * HW + p0 + pp) * C + col) =
                                __floats2bfloat162_rn(o[nt][2], o[nt][3]);
                    }
                }
                dev::named_bar(1, kFuWorkers * 32);
            }
        }
    }
    dev::tc_fence_before();
    dev::cluster_sync_all();
    dev::tc_fence_after();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256)
                     : "memory");
}

}  // namespace

bool fused_attention_supported(uint32_t C, uint32_t heads, uint32_t F, uint32_t HW) {
    if (heads != 1 || C % 64 != 0 || F == 0 || F > 24) return false;  // 3 key n8 tiles
    uint32_t P = kFuPmax;
    while (P > 1 && FuLay(P, F, C).total > 226u * 1024u) --P;
    // Opt-in (VINF_FUSED_ATTN=1): bitwise equal to the unfused path but measured slower on
    // B200 at cfg2 (380 vs 208 us for projection + core): with one CTA pair per SM pair the
    // eight worker warps cannot hide the per-chunk conversion, softmax and barrier latencies,
    // and the tensor pipe idles (ncu: ~5% active). Kept as the starting point for a
    // deeper-pipelined version.
    return FuLay(P, F, C).total <= 226u * 1024u && P * F <= 128 && HW % P == 0 && (HW / P) % 2 == 0 &&
           getenv("VINF_FUSED_ATTN") != nullptr;
}

int launch_qkv_attention_fused(const void* u2, uint32_t af, uint32_t f_own0, uint32_t HW, uint32_t C,
                               uint32_t F, const void* wqkv, TokenTable tt, float scale, float bias,
                               void* ctx, cudaStream_t s) {
    uint32_t P = kFuPmax;
    while (P > 1 && FuLay(P, F, C).total > 226u * 1024u) --P;
    const FuLay L(P, F, C);
    FuMaps maps;
    {
        // 3D view of the attention operand: [af frames][HW positions][C channels]
        static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
        if (!fn) {
            cudaDriverEntryPointQueryResult q;
            void* f = nullptr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return int(cudaErrorNotSupported);
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        }
        cuuint64_t gdim[3] = {C, HW, af};
        cuuint64_t gstr[2] = {uint64_t(C) * 2, uint64_t(HW) * C * 2};
        cuuint32_t box[3] = {64, P, F};
        cuuint32_t es[3] = {1, 1, 1};
        if (fn(&maps.u2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(u2), gdim, gstr, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return int(cudaErrorInvalidValue);
    }
    int rc = make_tmap_bf16(&maps.w, wqkv, 3ull * C, C, C, 64);
    if (rc) return rc;
    rc = make_tmap_bf16(&maps.w32, wqkv, 3ull * C, C, C, 32);
    if (rc) return rc;
    static uint32_t attr = 0;  // (static smem counts against the opt-in limit too)
    if (attr < L.total) {
        const cudaError_t e = cudaFuncSetAttribute(qkv_attention_fused_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
        if (e != cudaSuccess) return int(e);
        attr = L.total;
    }
    const uint32_t stagger = 0;  // 1 rotates the channel-chunk order per CTA (measured: no gain)
    return int(launch_pdl(qkv_attention_fused_kernel, dim3(HW / P), dim3(kFuThreads), L.total, s, maps, HW, C,
                          F, P, f_own0, tt, scale, bias, static_cast<__nv_bfloat16*>(ctx), stagger));
}

}  // namespace vinf
