// Dual-scope attention core, cp.async ring (attend_tokens, ops.cpp:209-241, applied per
// spatial position as in dual_scope_reference ops.cpp:318-336 and attention_parallel
// clip_parallel.cpp:311-334): the feed launch_attention_core uses for wide K/V tiles (long
// clips, many sampled globals) and the split (fp32) mode; attention_core.cu's TMA ring feeds
// the narrow bf16 tiles. Same token rules and arithmetic:
//
//   * one CTA per (spatial position, block of 32 query frames); R = the distinct K/V frames the
//     block's queries touch (window band + sampled globals, <= kKvMax = 192);
//   * S = Q K^T [32 x R] over the head dim in 64-wide chunks, the reference's explicit token
//     softmax on S (window tokens then globals, duplicates kept, +bias on the flagged side)
//     in column form, then ctx = P V [32 x d] in 64-wide output chunks;
//   * mma.sync m16n8k16 bf16 -> fp32; any head dim d = C / heads with d % 8 == 0 (the last
//     64-wide chunk of a head is zero-filled past d, cp.async src-size 0);
//   * split mode: Q/K/V and ctx as two bf16 planes, every product hi*hi + hi*lo + lo*hi.
//
// Every thread streams 16-byte pieces of the Q/K/V chunks through one NS-deep cp.async ring
// with a fixed prefetch distance (NS - 1 chunks), so a head's V loads are in flight while its
// softmax runs; with four CTAs per SM the copies of many independent positions are in flight
// at once, which is what wide tiles need (see launch_attention_core).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kDC = 64;  // head-dim chunk (one 128-byte swizzle row of bf16)
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr uint32_t kSmemPerSm = 228 * 1024;

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    // byte offset of 16B chunk `chunk` of a 128-byte row (XOR swizzle: ldmatrix conflict-free)
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// 16-byte async copy; src_bytes = 0 zero-fills the destination (head-dim chunk past d)
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(g), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// hi = RN(x), lo = RN(x - hi), two values at a time
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = pack_bf16(a - __low2float(h), b - __high2float(h));
}

// Shared-memory layout (bytes). NTL = K/V rows / 8 (launch-wide max of the blocks' R,
// padded to 16); PL = bf16 planes per operand (2 in split mode).
//   ring[NS]  : stage = [Q hi | Q lo] (32 x 128 B each) + [K-or-V hi | lo] (RP x 128 B each)
//   pb        : P as bf16 (PL planes), 64-column blocks of 32 x 128 B
//   sp        : S, then P (fp32), 32 x SP
//   ost       : ctx staging, 2 buffers x PL planes x 32 x 128 B; aliases pb/sp when P lives
//               in registers for the PV phase (PREG), since S and the smem P are dead then
//   zinv[32]
template <int NTL, int NS, bool SPLIT>
struct CoreLay {
    static constexpr uint32_t RP = NTL * 8;
    static constexpr uint32_t SP = RP + 4;
    static constexpr uint32_t PL = SPLIT ? 2 : 1;
    static constexpr bool PREG = NTL <= 8;
    static constexpr uint32_t QT = kQBlock * 128;
    static constexpr uint32_t KT = RP * 128;
    static constexpr uint32_t stage = PL * (QT + KT);
    static constexpr uint32_t PB = ((RP + 63) / 64) * kQBlock * 128;
    static constexpr uint32_t pb = NS * stage;
    static constexpr uint32_t sp = pb + PL * PB;
    static constexpr uint32_t sp_end = sp + kQBlock * SP * 4;
    static constexpr uint32_t OST = 2 * PL * QT;
    static constexpr uint32_t ost = PREG ? pb : sp_end;
    static constexpr uint32_t zinv = PREG ? (sp_end > pb + OST ? sp_end : pb + OST) : sp_end + OST;
    static constexpr uint32_t total = zinv + kQBlock * 4;
    static constexpr int blocks = int(kSmemPerSm / (total + 1024)) > 4 ? 4 : int(kSmemPerSm / (total + 1024));
};

// D > 0: one head with head dim D fixed at compile time (the VideoCrafter2 levels' long clips)
template <int NTL, int NS, bool SPLIT, int D = 0>
__global__ void __launch_bounds__(kThreads, CoreLay<NTL, NS, SPLIT>::blocks)
    attention_core_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t qkv_lo, uint32_t HW, uint32_t C_,
                          uint32_t heads_, uint32_t nq, uint32_t q_frame0, TokenTable tt, float scale,
                          float bias, __nv_bfloat16* __restrict__ ctx, int64_t ctx_lo, const FuseO fo) {
    const uint32_t C = D > 0 ? uint32_t(D) : C_, heads = D > 0 ? 1u : heads_;
    dev::pdl_wait();
    dev::pdl_trigger();
    using LL = CoreLay<NTL, NS, SPLIT>;
    constexpr uint32_t RP = LL::RP;
    constexpr int SP = int(LL::SP);
    constexpr int KR = (int(RP) + 31) / 32;  // K/V rows per loading thread
    constexpr int KC = (int(RP) + 31) / 32;  // softmax columns per lane
    constexpr int NJ = (NTL + 3) / 4;         // S n8 tiles per warp
    static_assert(NTL % 2 == 0 && RP <= uint32_t(kKvMax), "K/V rows padded to a multiple of 16");
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // query blocks of one position are adjacent in launch order: their shared K/V rows
    // (the sampled globals, the overlapping window bands) are re-read from L2, not HBM
    const uint32_t nqb = (nq + kQBlock - 1) / kQBlock;
    const uint32_t p = blockIdx.x / nqb, qb = blockIdx.x - p * nqb;
    const uint32_t a0 = qb * kQBlock;
    const uint32_t nqh = min(uint32_t(kQBlock), nq - a0);
    const uint32_t R = tt.kv_count[qb];
    const uint32_t d = D > 0 ? uint32_t(D) : C / heads, nch = (d + kDC - 1) / kDC;
    const uint64_t ld = 3ull * C;
    const uint32_t sbase = dev::smem_u32(sm);
    float* sp = reinterpret_cast<float*>(sm + LL::sp);
    float* zinv = reinterpret_cast<float*>(sm + LL::zinv);

    // K/V pad rows [R, RP) of every slot and plane are never loaded: zero them once (P is 0
    // there and must meet finite V values)
    for (uint32_t i = tid; i < (RP - R) * 8; i += kThreads) {
        const uint32_t off = swz(R + (i >> 3), i & 7);
#pragma unroll
        for (int st = 0; st < NS; ++st)
#pragma unroll
            for (uint32_t pl = 0; pl < LL::PL; ++pl)
                *reinterpret_cast<uint4*>(sm + st * LL::stage + LL::PL * LL::QT + pl * LL::KT + off) =
                    make_uint4(0, 0, 0, 0);
    }

    // this thread's 16-byte pieces of every Q / K / V chunk: piece lp of row lr (Q) and of
    // rows lr + 32k (K/V)
    const uint32_t lr = tid >> 3, lp = tid & 7;
    const bool q_ok = lr < nqh;
    const uint16_t* kvf = tt.kv_frames + qb * kKvMax;
    const __nv_bfloat16* q_src = qkv + uint64_t((q_frame0 + a0 + min(lr, nqh - 1)) * HW + p) * ld + lp * 8;
    const __nv_bfloat16* k_src[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k)
        k_src[k] = qkv + uint64_t(uint32_t(kvf[min(lr + 32 * k, R - 1)]) * HW + p) * ld + lp * 8;
    uint32_t ld_h = 0, ld_w = 0, ld_slot = 0;
    auto issue = [&]() {
        if (ld_h < heads) {
            const bool qk = ld_w < nch;
            const uint32_t ch = qk ? ld_w : ld_w - nch;
            const uint32_t col = ld_h * d + ch * kDC;
            const uint32_t bytes = lp * 8 < d - ch * kDC ? 16u : 0u;  // zero-fill past the head dim
            const uint32_t st = sbase + ld_slot * LL::stage;
            if (qk && q_ok) {
                cp_async16(st + swz(lr, lp), q_src + col, bytes);
                if (SPLIT) cp_async16(st + LL::QT + swz(lr, lp), q_src + qkv_lo + col, bytes);
            } else if (!qk && q_ok && fo.y) {
                // fused output: the chunk's residual rows into the idle Q slot of the PV stage
                // (bf16: one piece per thread; fp32: 16 pieces of 4 floats a row, columns 0-31
                // in the hi plane's slot, 32-63 in the lo plane's)
                const uint64_t ro = (uint64_t(a0 + lr) * HW + p) * C + col;
                if (fo.res_bf16) {
                    cp_async16(st + swz(lr, lp), static_cast<const __nv_bfloat16*>(fo.res) + ro + (bytes ? lp * 8 : 0),
                               bytes);
                } else {
#pragma unroll
                    for (uint32_t k = 0; k < 2; ++k) {
                        const uint32_t pc = lp + 8 * k;
                        const uint32_t rb = pc * 4 < d - ch * kDC ? 16u : 0u;
                        cp_async16(st + k * LL::QT + swz(lr, lp),
                                   static_cast<const float*>(fo.res) + ro + (rb ? pc * 4 : 0), rb);
                    }
                }
            }
            const uint32_t kc = (qk ? C : 2 * C) + col;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                if (lr + 32 * k < R) {
                    const uint32_t dst = st + LL::PL * LL::QT + swz(lr + 32 * k, lp);
                    cp_async16(dst, k_src[k] + kc, bytes);
                    if (SPLIT) cp_async16(dst + LL::KT, k_src[k] + qkv_lo + kc, bytes);
                }
            }
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
    const uint32_t r7 = lane & 7, hb = lane >> 4, b1 = (lane >> 3) & 1;
    uint32_t a_off[4], b_off[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        a_off[kk] = (mt * 16 + r7 + b1 * 8) * 128 + (((kk * 2 + hb) ^ r7) << 4);
        b_off[kk] = LL::PL * LL::QT + r7 * 128 + (((kk * 2 + b1) ^ r7) << 4);
    }
    const uint32_t v_off = LL::PL * LL::QT + (r7 + b1 * 8) * 128 + (((2 * wq + hb) ^ r7) << 4);
    const int g = lane >> 2, t4 = lane & 3;
    auto p_addr = [&](int kq) {  // P fragment (A operand) of k16 step kq, plane 0
        return sbase + LL::pb + uint32_t(kq >> 2) * (kQBlock * 128) + (mt * 16 + r7 + b1 * 8) * 128 +
               ((((kq & 3) * 2 + hb) ^ r7) << 4);
    };
    // staged chunk -> ctx rows; rslot: the ring slot of the chunk's PV stage (fused output: its
    // residual rows sit in the slot's Q area)
    auto store_ctx = [&](uint32_t buf, uint32_t c0, uint32_t vw, uint32_t rslot) {
        if (tid < int(nqh) * 8) {
            const uint32_t r = tid >> 3, c = tid & 7;
            if (c * 8 < vw) {
                const uint8_t* ost = sm + LL::ost + buf * (LL::PL * LL::QT);
                const uint64_t o = (uint64_t(a0 + r) * HW + p) * C + c0 + c * 8;
                const uint4 hv = *reinterpret_cast<const uint4*>(ost + swz(r, c));
                if (fo.y) {  // y = ctx' + residual (one head)
                    float v[8];
                    unpack8(hv, v);
                    if (SPLIT) unpack8_add(*reinterpret_cast<const uint4*>(ost + LL::QT + swz(r, c)), v);
                    const uint8_t* rs = sm + rslot * LL::stage;
                    if (fo.res_bf16) {
                        fuse_o_add_bf16(fo, *reinterpret_cast<const uint4*>(rs + swz(r, c)), c0 + c * 8, v);
                    } else {
                        const uint32_t p0 = 2 * c, p1 = 2 * c + 1;
                        const float4 r0 = *reinterpret_cast<const float4*>(rs + (p0 >> 3) * LL::QT + swz(r, p0 & 7));
                        const float4 r1 = *reinterpret_cast<const float4*>(rs + (p1 >> 3) * LL::QT + swz(r, p1 & 7));
                        v[0] += r0.x; v[1] += r0.y; v[2] += r0.z; v[3] += r0.w;
                        v[4] += r1.x; v[5] += r1.y; v[6] += r1.z; v[7] += r1.w;
                    }
                    fuse_o_write(fo, o, v);
                } else {
                    *reinterpret_cast<uint4*>(ctx + o) = hv;
                    if (SPLIT)
                        *reinterpret_cast<uint4*>(ctx + ctx_lo + o) =
                            *reinterpret_cast<const uint4*>(ost + LL::QT + swz(r, c));
                }
            }
        }
    };

    uint32_t cslot = 0, och = 0;
    for (uint32_t h = 0; h < heads; ++h) {
        // ---------------- S = Q K^T ----------------
        // warp: m tile mt (16 queries) x n8 tiles wq, wq + 4, ... of the RP key columns
        float acc[NJ][4];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (uint32_t ch = 0; ch < nch; ++ch) {
            cp_wait<NS - 2>();
            __syncthreads();
            issue();
            const uint32_t st = sbase + cslot * LL::stage;
            cslot = cslot + 1 == NS ? 0 : cslot + 1;
            const uint32_t vw = min(uint32_t(kDC), d - ch * kDC);
#pragma unroll
            for (int kk = 0; kk < kDC / 16; ++kk) {
                if (kk * 16 >= int(vw)) break;  // zero-filled past the head dim
                uint32_t a[4], al[4];
                ldsm_x4(st + a_off[kk], a);
                if (SPLIT) ldsm_x4(st + LL::QT + a_off[kk], al);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    if (wq + 4 * j < NTL) {
                        uint32_t k0, k1;
                        ldsm_x2(st + b_off[kk] + (wq + 4 * j) * 1024, k0, k1);
                        mma_bf16(acc[j], a, k0, k1);
                        if (SPLIT) {
                            uint32_t l0, l1;
                            ldsm_x2(st + LL::KT + b_off[kk] + (wq + 4 * j) * 1024, l0, l1);
                            mma_bf16(acc[j], a, l0, l1);
                            mma_bf16(acc[j], al, k0, k1);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int nt = wq + 4 * j;
            if (nt < NTL) {
                const int col = nt * 8 + t4 * 2;
                *reinterpret_cast<float2*>(&sp[(mt * 16 + g) * SP + col]) = make_float2(acc[j][0], acc[j][1]);
                *reinterpret_cast<float2*>(&sp[(mt * 16 + g + 8) * SP + col]) = make_float2(acc[j][2], acc[j][3]);
            }
        }
        __syncthreads();
        if constexpr (RP == 64) {
            // 64-column tiles (long clips): eight threads per row, eight columns each (three
            // shuffle steps per reduction), P written straight to its bf16 planes
            const uint32_t r = uint32_t(tid) >> 3, oct = uint32_t(tid) & 7u;
            uint32_t w[4], wl[4];
            if (r < nqh) {
                const uint32_t qa = a0 + r;
                const int lo = tt.wlo[qa], hi = tt.whi[qa];
                const uint8_t* gm = tt.gmult + size_t(qb) * kKvMax;
                const float bw = tt.wflag ? bias : 0.f, bg = tt.gflag ? bias : 0.f;
                const float4 s0 = *reinterpret_cast<const float4*>(sp + r * SP + oct * 8);
                const float4 s1 = *reinterpret_cast<const float4*>(sp + r * SP + oct * 8 + 4);
                const float sr[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
                float sv[8], m = -INFINITY;
                bool inw[8];
                int ng[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int c = int(oct) * 8 + k;
                    const bool ok = c < int(R);
                    sv[k] = ok ? scale * sr[k] : 0.f;
                    inw[k] = ok && c >= lo && c <= hi;
                    ng[k] = ok ? gm[c] : 0;
                    if (inw[k]) m = fmaxf(m, sv[k] + bw);
                    if (ng[k]) m = fmaxf(m, sv[k] + bg);
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                float e[8], z = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    e[k] = inw[k] ? (SPLIT ? expf(sv[k] + bw - m) : __expf(sv[k] + bw - m)) : 0.f;
                    if (ng[k]) e[k] += float(ng[k]) * (SPLIT ? expf(sv[k] + bg - m) : __expf(sv[k] + bg - m));
                    z += e[k];
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
                const float zi = 1.0f / z;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (SPLIT)
                        split2(e[2 * k] * zi, e[2 * k + 1] * zi, w[k], wl[k]);
                    else
                        w[k] = pack_bf16(e[2 * k] * zi, e[2 * k + 1] * zi);
                }
            } else {
                // rows past the block: P = 0, the octet's shuffles kept converged
                float m = 0.f;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = wl[k] = 0u;
            }
            const uint32_t off = LL::pb + swz(r, oct);
            *reinterpret_cast<uint4*>(sm + off) = make_uint4(w[0], w[1], w[2], w[3]);
            if (SPLIT) *reinterpret_cast<uint4*>(sm + off + LL::PB) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            __syncthreads();
        } else {
        // ---------------- softmax over the token lists, per column -> P (in place) ----------
            // The reference's token list (window, then globals, duplicates kept; ops.cpp:209-241)
            // in column form: column c carries the window token iff wlo <= c <= whi and gmult[c]
            // global tokens; p_c = [window] e^(l_w - m) + gmult[c] e^(l_g - m), summed one token
            // at a time. Lane l owns columns l + 32k: no token-list walk, no smem atomics.
            for (uint32_t a = warp; a < uint32_t(kQBlock); a += kWarps) {
                float* row = sp + a * SP;
                float pv[KC];
                float zi = 0.f;
    #pragma unroll
                for (int k = 0; k < KC; ++k) pv[k] = 0.f;
                if (a < nqh) {
                    const uint32_t qa = a0 + a;
                    const int lo = tt.wlo[qa], hi = tt.whi[qa];
                    const uint8_t* gm = tt.gmult + size_t(qb) * kKvMax;
                    const float bw = tt.wflag ? bias : 0.f, bg = tt.gflag ? bias : 0.f;
                    float sv[KC];
                    bool inw[KC];
                    int ng[KC];
                    float m = -INFINITY;
    #pragma unroll
                    for (int k = 0; k < KC; ++k) {
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
                    for (int k = 0; k < KC; ++k) {
                        // (the column's ng[k] global tokens as one product: bf16 mode in the fast exp)
                        float e = inw[k] ? (SPLIT ? expf(sv[k] + bw - m) : __expf(sv[k] + bw - m)) : 0.f;
                        if (ng[k]) e += float(ng[k]) * (SPLIT ? expf(sv[k] + bg - m) : __expf(sv[k] + bg - m));
                        pv[k] = e;
                        z += e;
                    }
    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
                    zi = 1.0f / z;
                }
                __syncwarp();
    #pragma unroll
                for (int k = 0; k < KC; ++k) {
                    const int c = lane + 32 * k;
                    if (c < SP) row[c] = pv[k];
                }
                if (lane < SP - 32 * KC) row[32 * KC + lane] = 0.f;
                if (lane == 0) zinv[a] = zi;
            }
            __syncthreads();
            // P = S_normalised -> bf16 planes (64-column blocks in the swizzled row layout)
            for (int i = tid; i < int(kQBlock * RP / 8); i += kThreads) {
                const uint32_t r = i / (RP / 8), c8 = i % (RP / 8);
                const float zi = zinv[r];
                const float4 s0 = *reinterpret_cast<const float4*>(sp + r * SP + c8 * 8);
                const float4 s1 = *reinterpret_cast<const float4*>(sp + r * SP + c8 * 8 + 4);
                const float v[8] = {s0.x * zi, s0.y * zi, s0.z * zi, s0.w * zi,
                                    s1.x * zi, s1.y * zi, s1.z * zi, s1.w * zi};
                const uint32_t off = LL::pb + (c8 >> 3) * (kQBlock * 128) + swz(r, c8 & 7);
                uint32_t w[4], wl[4];
    #pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (SPLIT)
                        split2(v[2 * k], v[2 * k + 1], w[k], wl[k]);
                    else
                        w[k] = pack_bf16(v[2 * k], v[2 * k + 1]);
                }
                *reinterpret_cast<uint4*>(sm + off) = make_uint4(w[0], w[1], w[2], w[3]);
                if (SPLIT) *reinterpret_cast<uint4*>(sm + off + LL::PB) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            }
            __syncthreads();
        }
        // ---------------- ctx = P V ----------------
        // warp: m tile mt, n8 tiles 2wq, 2wq + 1 of each 64-wide output chunk
        uint32_t pa[LL::PREG ? NTL / 2 : 1][4], pal[LL::PREG && SPLIT ? NTL / 2 : 1][4];
        if (LL::PREG) {
#pragma unroll
            for (int kq = 0; kq < NTL / 2; ++kq) {
                ldsm_x4(p_addr(kq), pa[LL::PREG ? kq : 0]);
                if (SPLIT) ldsm_x4(p_addr(kq) + LL::PB, pal[LL::PREG && SPLIT ? kq : 0]);
            }
        }
        for (uint32_t ch = 0; ch < nch; ++ch, ++och) {
            cp_wait<NS - 2>();
            __syncthreads();
            if (ch > 0)
                store_ctx((och - 1) & 1, h * d + (ch - 1) * kDC, min(uint32_t(kDC), d - (ch - 1) * kDC),
                          cslot == 0 ? NS - 1 : cslot - 1);
            issue();
            const uint32_t st = sbase + cslot * LL::stage;
            cslot = cslot + 1 == NS ? 0 : cslot + 1;
            const uint32_t vw = min(uint32_t(kDC), d - ch * kDC);
            float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            if (uint32_t(wq) * 16 < vw) {  // this warp's 16 output columns hold data
#pragma unroll
                for (int kq = 0; kq < NTL / 2; ++kq) {
                    uint32_t b[4], bl[4], a[4], al[4];
                    ldsm_x4_t(st + v_off + kq * 2048, b);
                    if (LL::PREG) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) a[k] = pa[LL::PREG ? kq : 0][k];
                        if (SPLIT)
#pragma unroll
                            for (int k = 0; k < 4; ++k) al[k] = pal[LL::PREG && SPLIT ? kq : 0][k];
                    } else {
                        ldsm_x4(p_addr(kq), a);
                        if (SPLIT) ldsm_x4(p_addr(kq) + LL::PB, al);
                    }
                    mma_bf16(o[0], a, b[0], b[1]);
                    mma_bf16(o[1], a, b[2], b[3]);
                    if (SPLIT) {
                        ldsm_x4_t(st + LL::KT + v_off + kq * 2048, bl);
                        mma_bf16(o[0], a, bl[0], bl[1]);
                        mma_bf16(o[1], a, bl[2], bl[3]);
                        mma_bf16(o[0], al, b[0], b[1]);
                        mma_bf16(o[1], al, b[2], b[3]);
                    }
                }
            }
            uint8_t* ost = sm + LL::ost + (och & 1) * (LL::PL * LL::QT);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t col = (2 * wq + j) * 8 + t4 * 2;
                const uint32_t r0 = mt * 16 + g;
                const uint32_t o0 = swz(r0, col >> 3) + (col & 7) * 2, o1 = swz(r0 + 8, col >> 3) + (col & 7) * 2;
                if (SPLIT) {
                    uint32_t h0, l0, h1, l1;
                    split2(o[j][0], o[j][1], h0, l0);
                    split2(o[j][2], o[j][3], h1, l1);
                    *reinterpret_cast<uint32_t*>(ost + o0) = h0;
                    *reinterpret_cast<uint32_t*>(ost + o1) = h1;
                    *reinterpret_cast<uint32_t*>(ost + LL::QT + o0) = l0;
                    *reinterpret_cast<uint32_t*>(ost + LL::QT + o1) = l1;
                } else {
                    *reinterpret_cast<uint32_t*>(ost + o0) = pack_bf16(o[j][0], o[j][1]);
                    *reinterpret_cast<uint32_t*>(ost + o1) = pack_bf16(o[j][2], o[j][3]);
                }
            }
        }
        __syncthreads();
        store_ctx((och - 1) & 1, h * d + (nch - 1) * kDC, min(uint32_t(kDC), d - (nch - 1) * kDC),
                  cslot == 0 ? NS - 1 : cslot - 1);
        // the staging buffer and S / P scratch are rewritten only after the next head's
        // first S-phase barrier
    }
    cp_wait<0>();
}

template <int NTL, int NS, bool SPLIT, int D = 0>
int launch_core(const void* qkv, int64_t qkv_lo, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
                uint32_t q_frame0, const TokenTable& tt, float scale, float bias, void* ctx, int64_t ctx_lo,
                cudaStream_t s, const FuseO& fo) {
    using LL = CoreLay<NTL, NS, SPLIT>;
    static_assert(LL::total <= 227 * 1024, "attention core shared memory");
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(attention_core_kernel<NTL, NS, SPLIT, D>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(LL::total));
        if (e != cudaSuccess) return int(e);
        attr = true;
    }
    dim3 grid(HW * ((nq + kQBlock - 1) / kQBlock));
    return int(launch_pdl(attention_core_kernel<NTL, NS, SPLIT, D>, grid, dim3(kThreads), LL::total, s,
                          static_cast<const __nv_bfloat16*>(qkv), qkv_lo, HW, C, heads, nq, q_frame0, tt,
                          scale, bias, static_cast<__nv_bfloat16*>(ctx), ctx_lo, fo));
}

// ring depth per (K/V width, mode): deep rings for the narrow tiles (4 CTAs/SM at cfg2),
// shallower where one CTA's tiles are wide
template <int NTL, bool SPLIT>
int launch_ntl(const void* qkv, int64_t qkv_lo, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
               uint32_t q_frame0, const TokenTable& tt, float scale, float bias, void* ctx, int64_t ctx_lo,
               cudaStream_t s, const FuseO& fo) {
    constexpr int NS = NTL <= 4 ? 5 : (NTL <= 8 ? 4 : (SPLIT ? 2 : 3));
    // the long clips' 48/64-row tiles (bf16), and the fp32 mode's tiles up to 64 rows
    if constexpr ((!SPLIT && (NTL == 6 || NTL == 8)) || (SPLIT && NTL <= 8)) {
        if (heads == 1) switch (C) {
                case 320: return launch_core<NTL, NS, SPLIT, 320>(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s, fo);
                case 640: return launch_core<NTL, NS, SPLIT, 640>(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s, fo);
                case 1280: return launch_core<NTL, NS, SPLIT, 1280>(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s, fo);
                default: break;
            }
    }
    return launch_core<NTL, NS, SPLIT>(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s, fo);
}

template <bool SPLIT>
int launch_mode(uint32_t RP, const void* qkv, int64_t qkv_lo, uint32_t HW, uint32_t C, uint32_t heads,
                uint32_t nq, uint32_t q_frame0, const TokenTable& tt, float scale, float bias, void* ctx,
                int64_t ctx_lo, cudaStream_t s, const FuseO& fo) {
#define CORE(NTL) \
    case NTL * 8: \
        return launch_ntl<NTL, SPLIT>(qkv, qkv_lo, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, ctx_lo, s, fo)
    switch (RP) {
        CORE(2); CORE(4); CORE(6); CORE(8); CORE(10); CORE(12);
        CORE(14); CORE(16); CORE(18); CORE(20); CORE(22); CORE(24);
        default: return int(cudaErrorInvalidValue);
    }
#undef CORE
}

}  // namespace

int launch_attention_core_cpasync(const void* qkv, const void* qkv_lo, uint32_t HW, uint32_t C, uint32_t heads,
                          uint32_t nq, uint32_t q_frame0, const TokenTable& tt, float scale, float bias,
                          void* ctx, void* ctx_lo, cudaStream_t s, const FuseO* fo) {
    if (HW == 0 || !qkv || !ctx || (qkv_lo == nullptr) != (ctx_lo == nullptr))
        return int(cudaErrorInvalidValue);
    if (fo && fo->y && (heads != 1 || !fo->res || (fo->s == nullptr) != (fo->t == nullptr)))
        return int(cudaErrorInvalidValue);
    const FuseO f = fo ? *fo : FuseO{};
    if (nq == 0) return 0;
    if (!(heads > 0 && C % heads == 0 && (C / heads) % 8 == 0 && tt.kv_ok && tt.max_kv > 0 && tt.max_kv <= kKvMax))
        return int(cudaErrorInvalidValue);
    const uint32_t RP = (uint32_t(tt.max_kv) + 15) & ~15u;
    using bf = __nv_bfloat16;
    if (qkv_lo) {
        const int64_t ql = static_cast<const bf*>(qkv_lo) - static_cast<const bf*>(qkv);
        const int64_t cl = static_cast<bf*>(ctx_lo) - static_cast<bf*>(ctx);
        return launch_mode<true>(RP, qkv, ql, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, cl, s, f);
    }
    return launch_mode<false>(RP, qkv, 0, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, 0, s, f);
}

}  // namespace vinf
