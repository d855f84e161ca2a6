// Tensor-core dual-scope attention core for the bf16 mode (mma.sync m16n8k16 bf16 ->
// fp32). Per spatial position p and block of 32 query frames:
//
//   S  = Q K^T            [32 x R]   over the head dim in 64-wide chunks
//   P  = token softmax    [32 x R]   the reference's explicit token list per query
//                                    (window then globals, duplicates kept, +bias on the
//                                    flagged side): p_r = sum_{i: col_i = r} e^{l_i - m} / Z
//   ctx = P V             [32 x d]   in 64-wide output chunks, staged through smem for
//                                    16-byte row stores
//
// R = the distinct K/V frames the block's queries touch (<= 64; window band + globals).
// The kernel is bound by reading Q/K/V once and writing ctx once, so the
// whole per-CTA load sequence (Q+K chunks of every head, then V chunks) streams through
// one kStages-deep cp.async ring with a fixed prefetch distance; the V loads of a head
// are in flight while its softmax runs. tcgen05 needs M >= 64 and this tile has M = 32
// queries (24 at the VideoCrafter2 clip), so S and PV use the warp-level tensor path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kDC = 64;        // head-dim chunk (one 128-byte swizzle row)
constexpr int kTcWarps = 8;
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kStages = 4;     // cp.async ring depth (prefetch distance kStages - 1)

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    // byte offset of 16B chunk `chunk` of a 128-byte row (XOR swizzle: ldmatrix conflict-free)
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
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

// Dynamic smem layout (bytes), RP = padded K/V rows (multiple of 16, <= kKvMax):
//   ring[kStages] : Q chunk (32 x 128 B) + K-or-V chunk (RP x 128 B)
//   pb            : P as bf16, 32 x 128 B (A operand of P V)
//   sp            : S, then P (fp32), 32 x (kKvMax + 4)
//   ost           : output staging 32 x 128 B
//   zinv[32], qrow[32], kvrow[kKvMax]
struct Lay {
    uint32_t stage, ring, pb, sp, ost, zinv, qrow, kvrow, total;
    __host__ __device__ explicit Lay(uint32_t RP) {
        stage = kQBlock * 128 + RP * 128;
        ring = 0;
        pb = ring + kStages * stage;
        sp = pb + kQBlock * 128;
        ost = sp + kQBlock * (kKvMax + 4) * 4;
        zinv = ost + kQBlock * 128;
        qrow = zinv + kQBlock * 4;
        kvrow = qrow + kQBlock * 4;
        total = kvrow + kKvMax * 4;
    }
};

__global__ void __launch_bounds__(kTcThreads)
    attention_core_tc_kernel(const __nv_bfloat16* __restrict__ qkv, uint32_t HW, uint32_t C,
                             uint32_t heads, uint32_t nq, uint32_t q_frame0, TokenTable tt,
                             float scale, float bias, __nv_bfloat16* __restrict__ ctx) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t p = blockIdx.x, qb = blockIdx.y;
    const uint32_t a0 = qb * kQBlock;
    const uint32_t nqh = min(uint32_t(kQBlock), nq - a0);
    const uint32_t R = tt.kv_count[qb];
    const uint32_t RP = (R + 15) & ~15u;  // padded K/V rows (multiple of 16)
    const Lay L(RP);
    const uint32_t d = C / heads;
    const uint32_t nch = d / kDC;          // chunks per head and phase
    const uint32_t nload = heads * 2 * nch;  // load sequence: per head, Q+K chunks then V chunks
    const uint64_t ld = 3ull * C;
    uint32_t* qrow = reinterpret_cast<uint32_t*>(sm + L.qrow);
    uint32_t* kvrow = reinterpret_cast<uint32_t*>(sm + L.kvrow);
    float* sp = reinterpret_cast<float*>(sm + L.sp);
    float* zinv = reinterpret_cast<float*>(sm + L.zinv);
    constexpr int SP = kKvMax + 4;  // fp32 pitch of S / P rows

    if (tid < kQBlock) qrow[tid] = (q_frame0 + a0 + min(uint32_t(tid), nqh - 1)) * HW + p;
    if (tid < kKvMax)
        kvrow[tid] = uint32_t(tt.kv_frames[qb * kKvMax + min(uint32_t(tid), R - 1)]) * HW + p;
    __syncthreads();

    const uint32_t sbase = dev::smem_u32(sm);
    // Each thread copies the same (row, 16 B chunk) of every Q / K / V chunk: Q is
    // 32 rows x 8 chunks = one item per thread; K/V has RP rows x 8 = up to two.
    static_assert(kQBlock * 8 == kTcThreads, "one Q item per thread");
    const uint32_t it_r = tid >> 3, it_c = tid & 7;
    const __nv_bfloat16* q_src = qkv + uint64_t(qrow[it_r]) * ld + it_c * 8;
    const uint32_t q_dst = swz(it_r, it_c);
    const bool kv0 = it_r < RP, kv1 = it_r + 32 < RP;  // never write past this CTA's RP rows
    const __nv_bfloat16* kv_src0 = qkv + uint64_t(kvrow[min(it_r, RP - 1)]) * ld + it_c * 8;
    const __nv_bfloat16* kv_src1 = qkv + uint64_t(kvrow[min(it_r + 32, RP - 1)]) * ld + it_c * 8;
    const uint32_t kv_dst0 = kQBlock * 128 + swz(it_r, it_c), kv_dst1 = kQBlock * 128 + swz(it_r + 32, it_c);
    auto issue = [&](uint32_t li) {  // load item li of the sequence into ring slot li % kStages
        if (li < nload) {
            const uint32_t h = li / (2 * nch), w = li % (2 * nch);
            const bool qk = w < nch;
            const uint32_t col = h * d + (qk ? w : w - nch) * kDC;
            const uint32_t st = sbase + L.ring + (li % kStages) * L.stage;
            if (qk) cp_async16(st + q_dst, q_src + col);
            const uint32_t kvc = (qk ? C : 2 * C) + col;
            if (kv0) cp_async16(st + kv_dst0, kv_src0 + kvc);
            if (kv1) cp_async16(st + kv_dst1, kv_src1 + kvc);
        }
        cp_commit();  // always commit (possibly empty) so group counting stays uniform
    };
    for (uint32_t li = 0; li < kStages - 1; ++li) issue(li);

    const int mt = warp & 1;              // S: 16-row m tile;  PV: 16-row m tile
    const int wq = warp >> 1;             // 0..3
    const int NT = int(RP) / 8;           // n8 tiles of S (2..8)
    uint32_t li = 0;
    for (uint32_t h = 0; h < heads; ++h) {
        // ---------------- phase 1: S = Q K^T ----------------
        // warp: m tile mt (16 queries) x n8 tiles wq and wq + 4 of the RP key columns
        float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        for (uint32_t ch = 0; ch < nch; ++ch, ++li) {
            issue(li + kStages - 1);
            cp_wait<kStages - 1>();
            __syncthreads();
            const uint32_t qa = sbase + L.ring + (li % kStages) * L.stage;
            const uint32_t ka = qa + kQBlock * 128;
#pragma unroll
            for (int kk = 0; kk < kDC / 16; ++kk) {
                uint32_t a[4];
                ldsm_x4(qa + swz(mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, kk * 2 + (lane >> 4)),
                        a[0], a[1], a[2], a[3]);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int nt = wq + 4 * j;
                    if (nt < NT) {
                        uint32_t b0, b1;
                        ldsm_x2(ka + swz(nt * 8 + (lane & 7), kk * 2 + ((lane >> 3) & 1)), b0, b1);
                        mma_bf16(acc[j], a[0], a[1], a[2], a[3], b0, b1);
                    }
                }
            }
            __syncthreads();
        }
        {
            const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int nt = wq + 4 * j;
                if (nt < NT) {
                    const int col = nt * 8 + t4 * 2;
                    sp[(mt * 16 + g) * SP + col] = acc[j][0];
                    sp[(mt * 16 + g) * SP + col + 1] = acc[j][1];
                    sp[(mt * 16 + g + 8) * SP + col] = acc[j][2];
                    sp[(mt * 16 + g + 8) * SP + col + 1] = acc[j][3];
                }
            }
        }
        __syncthreads();
        // ---------------- phase 2: token softmax -> P (in place over S) ----------------
        for (uint32_t a = warp; a < uint32_t(kQBlock); a += kTcWarps) {
            float* row = sp + a * SP;
            if (a < nqh) {
                const uint32_t qa = a0 + a;
                const int n = tt.count[qa];
                const uint8_t* cols = tt.col + size_t(qa) * kMaxTokens;
                const uint8_t* flg = tt.biased + size_t(qa) * kMaxTokens;
                // each lane holds up to kMaxTokens/32 = 5 token logits
                float lg[(kMaxTokens + 31) / 32];
                int cl[(kMaxTokens + 31) / 32];
                float m = -INFINITY;
                const int nk = (n + 31) >> 5;
#pragma unroll
                for (int k = 0; k < (kMaxTokens + 31) / 32; ++k) {
                    const int i = lane + 32 * k;
                    cl[k] = 0;
                    lg[k] = -INFINITY;
                    if (k < nk && i < n) {
                        cl[k] = int(cols[i]);
                        lg[k] = scale * row[cl[k]] + (flg[i] ? bias : 0.f);
                    }
                    m = fmaxf(m, lg[k]);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                float z = 0.f;
#pragma unroll
                for (int k = 0; k < (kMaxTokens + 31) / 32; ++k) {
                    lg[k] = (k < nk && lane + 32 * k < n) ? expf(lg[k] - m) : 0.f;
                    z += lg[k];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
                __syncwarp();
                for (int c = lane; c < kKvMax; c += 32) row[c] = 0.f;  // S row consumed
                // Duplicate tokens (a frame in both the window and the global set) add into
                // the same column. The window list and the global list are each duplicate-
                // free, so a column receives at most two additions onto 0, and fp32 addition
                // of two operands is commutative: the result is order-independent
                // (bitwise reproducible).
#pragma unroll
                for (int k = 0; k < (kMaxTokens + 31) / 32; ++k)
                    if (k < nk && lane + 32 * k < n) atomicAdd(&row[cl[k]], lg[k]);
                if (lane == 0) zinv[a] = 1.0f / z;
            } else {
                for (int c = lane; c < kKvMax; c += 32) row[c] = 0.f;
                if (lane == 0) zinv[a] = 0.f;
            }
        }
        __syncthreads();
        for (int i = tid; i < kQBlock * int(RP) / 8; i += kTcThreads) {
            const uint32_t r = i / (RP / 8), c = i % (RP / 8);  // 8 bf16 per 16B chunk
            const float zi = zinv[r];
            const float* src = sp + r * SP + c * 8;
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(src[2 * k] * zi, src[2 * k + 1] * zi);
                w[k] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            *reinterpret_cast<uint4*>(sm + L.pb + swz(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        __syncthreads();
        // ---------------- phase 3: ctx = P V ----------------
        // warp: m tile mt, n8 tiles 2wq, 2wq+1 of each 64-wide chunk; its P fragments
        // (A operand) are loaded once per head and reused for every V chunk.
        const uint32_t pb_s = sbase + L.pb;
        uint32_t pa[4][4];  // k16 steps of RP (<= 64)
#pragma unroll
        for (int kq = 0; kq < 4; ++kq)
            if (kq < int(RP / 16))
                ldsm_x4(pb_s + swz(mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, kq * 2 + (lane >> 4)),
                        pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3]);
        for (uint32_t ch = 0; ch < nch; ++ch, ++li) {
            issue(li + kStages - 1);
            cp_wait<kStages - 1>();
            __syncthreads();
            const uint32_t va = sbase + L.ring + (li % kStages) * L.stage + kQBlock * 128;
            float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) {
                if (kq < int(RP / 16)) {
                    uint32_t b[4];
                    // (k lo, tile 2wq), (k hi, tile 2wq), (k lo, tile 2wq+1), (k hi, tile 2wq+1)
                    ldsm_x4_t(va + swz(kq * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, 2 * wq + (lane >> 4)),
                              b[0], b[1], b[2], b[3]);
                    mma_bf16(o[0], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[0], b[1]);
                    mma_bf16(o[1], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[2], b[3]);
                }
            }
            {
                const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t col = (2 * wq + j) * 8 + t4 * 2;
                    const __nv_bfloat162 lo2 = __floats2bfloat162_rn(o[j][0], o[j][1]);
                    const __nv_bfloat162 hi2 = __floats2bfloat162_rn(o[j][2], o[j][3]);
                    const uint32_t r0 = mt * 16 + g;
                    *reinterpret_cast<__nv_bfloat162*>(sm + L.ost + swz(r0, col >> 3) + (col & 7) * 2) = lo2;
                    *reinterpret_cast<__nv_bfloat162*>(sm + L.ost + swz(r0 + 8, col >> 3) + (col & 7) * 2) = hi2;
                }
            }
            __syncthreads();
            const uint32_t c0 = h * d + ch * kDC;
            for (int i = tid; i < int(nqh) * 8; i += kTcThreads) {
                const uint32_t r = i >> 3, c = i & 7;
                const uint4 v = *reinterpret_cast<const uint4*>(sm + L.ost + swz(r, c));
                *reinterpret_cast<uint4*>(ctx + (uint64_t(a0 + r) * HW + p) * C + c0 + c * 8) = v;
            }
            // the ring slot just consumed is refilled by the next iteration's issue() only
            // after the __syncthreads at its top; the staging buffer likewise
        }
    }
    cp_wait<0>();
}

// ---------------------------------------------------------------------------------------
// Lean ring kernel (the default). Same load sequence, smem layout and arithmetic as the
// kernel above (so the same bits), restructured for instruction count, which is what bounds
// the kernel above (ncu: ~76% issue-slot utilisation, HMMA ~4% of instructions):
//   * the K/V row count is a template parameter (launch-wide max), so every S/PV tile loop
//     is unrolled without per-tile branches;
//   * ldmatrix addresses are per-lane constants plus immediates (the swizzle XOR depends
//     only on lane bits);
//   * the load sequence advances incrementally (no divisions), one barrier per chunk;
//   * Q rows past the block's queries and K/V pad rows are never loaded (pad rows of every
//     ring slot are zeroed once), and ctx staging is double-buffered.
template <int NTL, int NS>
struct LeanLay {
    static constexpr uint32_t RP = NTL * 8;
    static constexpr uint32_t SP = RP + 4;
    static constexpr uint32_t stage = kQBlock * 128 + RP * 128;
    static constexpr uint32_t pb = NS * stage;
    static constexpr uint32_t sp = pb + kQBlock * 128;
    // ctx staging (2 x 32 rows x 128 B) reuses the P / S scratch: P lives in registers
    // for the whole PV phase and S is dead by then
    static constexpr uint32_t ost = pb;
    static constexpr uint32_t scratch = kQBlock * 128 + kQBlock * SP * 4;
    static constexpr uint32_t zinv = pb + (scratch > 2 * kQBlock * 128 ? scratch : 2 * kQBlock * 128);
    static constexpr uint32_t total = zinv + kQBlock * 4;
    static constexpr int min_blocks = (NTL <= 4 && NS <= 5) ? 4 : 3;  // CTAs per SM the smem allows
};

template <int NTL, int NS>
__global__ void __launch_bounds__(kTcThreads, LeanLay<NTL, NS>::min_blocks)
    attention_core_lean_kernel(const __nv_bfloat16* __restrict__ qkv, uint32_t HW, uint32_t C,
                               uint32_t heads, uint32_t nq, uint32_t q_frame0, TokenTable tt,
                               float scale, float bias, __nv_bfloat16* __restrict__ ctx) {
    dev::pdl_wait();
    dev::pdl_trigger();
    using LL = LeanLay<NTL, NS>;
    constexpr uint32_t RP = LL::RP;
    constexpr int SP = int(LL::SP);
    static_assert(NTL % 2 == 0 && NTL <= 8, "K/V rows padded to a multiple of 16, at most 64");
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // query blocks of one position are adjacent in launch order: their shared K/V rows
    // (the sampled globals, the overlapping window bands) are re-read from L2, not HBM
    const uint32_t nqb = (nq + kQBlock - 1) / kQBlock;
    const uint32_t p = blockIdx.x / nqb, qb = blockIdx.x - p * nqb;
    const uint32_t a0 = qb * kQBlock;
    const uint32_t nqh = min(uint32_t(kQBlock), nq - a0);
    const uint32_t R = tt.kv_count[qb];
    const uint32_t d = C / heads, nch = d / kDC;
    const uint64_t ld = 3ull * C;
    const uint32_t sbase = dev::smem_u32(sm);
    float* sp = reinterpret_cast<float*>(sm + LL::sp);
    float* zinv = reinterpret_cast<float*>(sm + LL::zinv);

    // K/V pad rows [R, RP) of every slot are never loaded: zero them once (P is 0 there
    // and must meet finite V values)
    for (uint32_t i = tid; i < (RP - R) * 8; i += kTcThreads) {
        const uint32_t off = kQBlock * 128 + swz(R + (i >> 3), i & 7);
#pragma unroll
        for (int st = 0; st < NS; ++st)
            *reinterpret_cast<uint4*>(sm + st * LL::stage + off) = make_uint4(0, 0, 0, 0);
    }

    // this thread's 16-byte pieces of every Q / K / V chunk
    const uint32_t lr = tid >> 3, lp = tid & 7;
    const bool q_ok = lr < nqh, k0_ok = lr < R, k1_ok = NTL > 4 && lr + 32 < R;
    const uint16_t* kvf = tt.kv_frames + qb * kKvMax;
    const __nv_bfloat16* q_src = qkv + uint64_t((q_frame0 + a0 + min(lr, nqh - 1)) * HW + p) * ld + lp * 8;
    const __nv_bfloat16* k_src0 = qkv + uint64_t(uint32_t(kvf[min(lr, R - 1)]) * HW + p) * ld + lp * 8;
    const __nv_bfloat16* k_src1 =
        qkv + uint64_t(uint32_t(kvf[min(lr + 32, R - 1)]) * HW + p) * ld + lp * 8;
    const uint32_t q_dst = swz(lr, lp);
    const uint32_t kv_dst0 = kQBlock * 128 + swz(lr, lp);
    const uint32_t kv_dst1 = kQBlock * 128 + swz(lr + 32, lp);
    uint32_t ld_h = 0, ld_w = 0, ld_slot = 0;
    auto issue = [&]() {
        if (ld_h < heads) {
            const bool qk = ld_w < nch;
            const uint32_t col = ld_h * d + (qk ? ld_w : ld_w - nch) * kDC;
            const uint32_t st = sbase + ld_slot * LL::stage;
            if (qk && q_ok) cp_async16(st + q_dst, q_src + col);
            const uint32_t kc = (qk ? C : 2 * C) + col;
            if (k0_ok) cp_async16(st + kv_dst0, k_src0 + kc);
            if (NTL > 4 && k1_ok) cp_async16(st + kv_dst1, k_src1 + kc);
            if (++ld_w == 2 * nch) {
                ld_w = 0;
                ++ld_h;
            }
        }
        cp_commit();
        ld_slot = ld_slot + 1 == NS ? 0 : ld_slot + 1;
    };
#pragma unroll
    for (int i = 0; i < NS - 1; ++i) issue();

    // per-lane ldmatrix offsets: the XOR swizzle only involves lane bits
    const int mt = warp & 1, wq = warp >> 1;
    const uint32_t r7 = lane & 7, hi = lane >> 4, b1 = (lane >> 3) & 1;
    uint32_t a_off[4], b_off[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        a_off[kk] = (mt * 16 + r7 + b1 * 8) * 128 + (((kk * 2 + hi) ^ r7) << 4);
        b_off[kk] = kQBlock * 128 + r7 * 128 + (((kk * 2 + b1) ^ r7) << 4);
    }
    const uint32_t v_off = kQBlock * 128 + (r7 + b1 * 8) * 128 + (((2 * wq + hi) ^ r7) << 4);
    const int g = lane >> 2, t4 = lane & 3;

    uint32_t cslot = 0, och = 0;
    for (uint32_t h = 0; h < heads; ++h) {
        // ---------------- S = Q K^T ----------------
        float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        for (uint32_t ch = 0; ch < nch; ++ch) {
            cp_wait<NS - 2>();
            __syncthreads();
            issue();
            const uint32_t st = sbase + cslot * LL::stage;
            cslot = cslot + 1 == NS ? 0 : cslot + 1;
#pragma unroll
            for (int kk = 0; kk < kDC / 16; ++kk) {
                uint32_t a[4];
                ldsm_x4(st + a_off[kk], a[0], a[1], a[2], a[3]);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (4 * j < NTL && wq + 4 * j < NTL) {
                        uint32_t b0, b1r;
                        ldsm_x2(st + b_off[kk] + (wq + 4 * j) * 1024, b0, b1r);
                        mma_bf16(acc[j], a[0], a[1], a[2], a[3], b0, b1r);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int nt = wq + 4 * j;
            if (4 * j < NTL && nt < NTL) {
                const int col = nt * 8 + t4 * 2;
                *reinterpret_cast<float2*>(&sp[(mt * 16 + g) * SP + col]) = make_float2(acc[j][0], acc[j][1]);
                *reinterpret_cast<float2*>(&sp[(mt * 16 + g + 8) * SP + col]) = make_float2(acc[j][2], acc[j][3]);
            }
        }
        __syncthreads();
        // ---------------- softmax over the token lists, per column -> P (in place) ----------
        // The reference's token list (window, then globals, duplicates kept; ops.cpp:209-241)
        // in column form: column c carries the window token iff wlo <= c <= whi and
        // gmult[c] global tokens; p_c = [window] e^(l_w - m) + sum over its global tokens
        // e^(l_g - m). Each lane owns columns lane and lane + 32: no token-list walk, no
        // shared-memory atomics.
        for (uint32_t a = warp; a < uint32_t(kQBlock); a += kTcWarps) {
            float* row = sp + a * SP;
            float pv[2] = {0.f, 0.f};
            float zi = 0.f;
            if (a < nqh) {
                const uint32_t qa = a0 + a;
                const int lo = tt.wlo[qa], hi = tt.whi[qa];
                const uint8_t* gm = tt.gmult + size_t(qb) * kKvMax;
                const float bw = tt.wflag ? bias : 0.f, bg = tt.gflag ? bias : 0.f;
                float sv[2];
                bool inw[2];
                int ng[2];
                float m = -INFINITY;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int c = lane + 32 * k;
                    const bool ok = c < int(R);
                    sv[k] = ok ? scale * row[c] : 0.f;
                    inw[k] = ok && c >= lo && c <= hi;
                    ng[k] = ok ? gm[c] : 0;
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
            for (int c = lane; c < SP; c += 32) row[c] = c < 64 ? pv[c >> 5] : 0.f;
            if (lane == 0) zinv[a] = zi;
        }
        __syncthreads();
#pragma unroll
        for (int i0 = 0; i0 < int(kQBlock * RP / 8); i0 += kTcThreads) {
            const int i = i0 + tid;
            if (i < int(kQBlock * RP / 8)) {
                const uint32_t r = i / (RP / 8), c = i % (RP / 8);
                const float zi = zinv[r];
                const float4 s0 = *reinterpret_cast<const float4*>(sp + r * SP + c * 8);
                const float4 s1 = *reinterpret_cast<const float4*>(sp + r * SP + c * 8 + 4);
                const __nv_bfloat162 w0 = __floats2bfloat162_rn(s0.x * zi, s0.y * zi);
                const __nv_bfloat162 w1 = __floats2bfloat162_rn(s0.z * zi, s0.w * zi);
                const __nv_bfloat162 w2 = __floats2bfloat162_rn(s1.x * zi, s1.y * zi);
                const __nv_bfloat162 w3 = __floats2bfloat162_rn(s1.z * zi, s1.w * zi);
                *reinterpret_cast<uint4*>(sm + LL::pb + swz(r, c)) =
                    make_uint4(*reinterpret_cast<const uint32_t*>(&w0), *reinterpret_cast<const uint32_t*>(&w1),
                               *reinterpret_cast<const uint32_t*>(&w2), *reinterpret_cast<const uint32_t*>(&w3));
            }
        }
        __syncthreads();
        uint32_t pa[NTL / 2][4];
#pragma unroll
        for (int kq = 0; kq < NTL / 2; ++kq)
            ldsm_x4(sbase + LL::pb + (mt * 16 + r7 + b1 * 8) * 128 + (((kq * 2 + hi) ^ r7) << 4),
                    pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3]);
        // ---------------- ctx = P V ----------------
        for (uint32_t ch = 0; ch < nch; ++ch, ++och) {
            cp_wait<NS - 2>();
            __syncthreads();
            if (ch > 0) {  // chunk ch-1 is staged: row stores of this block's queries
                const uint8_t* ost = sm + LL::ost + ((och - 1) & 1) * (kQBlock * 128);
                const uint32_t c0 = h * d + (ch - 1) * kDC;
                if (tid < int(nqh) * 8) {
                    const uint32_t r = tid >> 3, c = tid & 7;
                    *reinterpret_cast<uint4*>(ctx + (uint64_t(a0 + r) * HW + p) * C + c0 + c * 8) =
                        *reinterpret_cast<const uint4*>(ost + swz(r, c));
                }
            }
            issue();
            const uint32_t st = sbase + cslot * LL::stage;
            cslot = cslot + 1 == NS ? 0 : cslot + 1;
            float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kq = 0; kq < NTL / 2; ++kq) {
                uint32_t b[4];
                ldsm_x4_t(st + v_off + kq * 2048, b[0], b[1], b[2], b[3]);
                mma_bf16(o[0], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[0], b[1]);
                mma_bf16(o[1], pa[kq][0], pa[kq][1], pa[kq][2], pa[kq][3], b[2], b[3]);
            }
            uint8_t* ost = sm + LL::ost + (och & 1) * (kQBlock * 128);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t col = (2 * wq + j) * 8 + t4 * 2;
                const uint32_t r0 = mt * 16 + g;
                *reinterpret_cast<__nv_bfloat162*>(ost + swz(r0, col >> 3) + (col & 7) * 2) =
                    __floats2bfloat162_rn(o[j][0], o[j][1]);
                *reinterpret_cast<__nv_bfloat162*>(ost + swz(r0 + 8, col >> 3) + (col & 7) * 2) =
                    __floats2bfloat162_rn(o[j][2], o[j][3]);
            }
        }
        __syncthreads();
        {
            const uint8_t* ost = sm + LL::ost + ((och - 1) & 1) * (kQBlock * 128);
            const uint32_t c0 = h * d + (nch - 1) * kDC;
            if (tid < int(nqh) * 8) {
                const uint32_t r = tid >> 3, c = tid & 7;
                *reinterpret_cast<uint4*>(ctx + (uint64_t(a0 + r) * HW + p) * C + c0 + c * 8) =
                    *reinterpret_cast<const uint4*>(ost + swz(r, c));
            }
        }
    }
    cp_wait<0>();
}

template <int NTL, int NS>
int launch_lean(const void* qkv, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
                uint32_t q_frame0, const TokenTable& tt, float scale, float bias, void* ctx,
                cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attention_core_lean_kernel<NTL, NS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(LeanLay<NTL, NS>::total));
        attr = true;
    }
    dim3 grid(HW * ((nq + kQBlock - 1) / kQBlock));
    return int(launch_pdl(attention_core_lean_kernel<NTL, NS>, grid, dim3(kTcThreads),
                          LeanLay<NTL, NS>::total, s, static_cast<const __nv_bfloat16*>(qkv), HW, C,
                          heads, nq, q_frame0, tt, scale, bias, static_cast<__nv_bfloat16*>(ctx)));
}

}  // namespace

int g_attn_variant = -1;  // -1: unread; 0 lean ring kernel (default); 1 original ring kernel

bool attention_tc_supported(uint32_t C, uint32_t heads, const TokenTable& tt) {
    return heads > 0 && C % heads == 0 && (C / heads) % kDC == 0 && tt.kv_ok;
}

int launch_attention_core_tc(const void* qkv, uint64_t qkv_rows, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
                             uint32_t q_frame0, TokenTable tt, float scale, float bias, void* ctx,
                             cudaStream_t s) {
    const uint32_t nqb = (nq + kQBlock - 1) / kQBlock;
    const uint32_t RPmax = (uint32_t(tt.max_kv) + 15) & ~15u;
    if (g_attn_variant < 0) {
        const char* v = getenv("VINF_ATTN_VARIANT");
        g_attn_variant = v ? atoi(v) : 0;
    }
    if (g_attn_variant != 1) {
        static int ns = -1;
        if (ns < 0) {
            const char* e = getenv("VINF_ATTN_STAGES");
            ns = e ? atoi(e) : 5;
        }
#define LEAN(NTL)                                                                                \
    (ns == 4   ? launch_lean<NTL, 4>(qkv, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, s)    \
     : ns == 5 ? launch_lean<NTL, 5>(qkv, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, s)    \
     : ns == 8 ? launch_lean<NTL, 8>(qkv, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, s)    \
               : launch_lean<NTL, 6>(qkv, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, s))
        switch (RPmax) {
            case 16: return LEAN(2);
            case 32: return LEAN(4);
            case 48: return LEAN(6);
            case 64: return LEAN(8);
            default: break;
        }
#undef LEAN
    }
    const size_t shm = Lay(RPmax).total;  // largest K/V list here
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attention_core_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Lay(kKvMax).total));
        attr = true;
    }
    dim3 grid(HW, nqb);
    attention_core_tc_kernel<<<grid, kTcThreads, shm, s>>>(
        static_cast<const __nv_bfloat16*>(qkv), HW, C, heads, nq, q_frame0, tt, scale, bias,
        static_cast<__nv_bfloat16*>(ctx));
    return int(cudaGetLastError());
}

}  // namespace vinf
