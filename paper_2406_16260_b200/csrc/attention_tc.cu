// Tensor-core dual-scope attention core for the bf16 mode (mma.sync m16n8k16 bf16 ->
// fp32). Per spatial position p and block of 32 query frames:
//
//   S  = Q K^T            [32 x R]   over the head dim in 64-wide chunks (cp.async double
//                                    buffer, ldmatrix from XOR-swizzled smem)
//   P  = token softmax    [32 x R]   the reference's explicit token list per query
//                                    (window then globals, duplicates kept, +bias on the
//                                    flagged side): p_r = sum_{i: col_i = r} e^{l_i - m} / Z
//   ctx = P V             [32 x d]   in 64-wide output chunks, staged through smem for
//                                    128-byte row stores
//
// R = the distinct K/V frames the block's queries touch (<= 64; window band + globals).
// tcgen05 needs M >= 64 and this tile has M = 32 queries (24 at the VideoCrafter2 clip), so
// the dense S/PV tiles run on the warp-level tensor path; the kernel is bound by reading
// Q/K/V once and writing ctx once (SURVEY §7 "attention-core tile shape").
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kDC = 64;  // head-dim chunk (one 128-byte swizzle row)
constexpr int kTcThreads = 128;

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    // byte offset of 16B chunk `chunk` of a 128-byte row
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

struct TcSmem {
    alignas(128) uint8_t q[2][kQBlock * 128];   // Q chunk (also output staging in phase 3)
    alignas(128) uint8_t kv[2][kKvMax * 128];   // K chunk (phase 1) / V chunk (phase 3)
    alignas(128) uint8_t pb[kQBlock * 128];     // P as bf16 (A operand of P V)
    float s[kQBlock][kKvMax + 4];               // logits
    float pf[kQBlock][kKvMax];                  // un-normalised weights (duplicates summed)
    float zinv[kQBlock];
    uint32_t qrow[kQBlock];                     // QKV row index of each query (this position)
    uint32_t kvrow[kKvMax];                     // QKV row index of each K/V column
};

__global__ void __launch_bounds__(kTcThreads)
    attention_core_tc_kernel(const __nv_bfloat16* __restrict__ qkv, uint32_t HW, uint32_t C,
                             uint32_t heads, uint32_t nq, uint32_t q_frame0, TokenTable tt,
                             float scale, float bias, __nv_bfloat16* __restrict__ ctx) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t p = blockIdx.x, qb = blockIdx.y;
    const uint32_t a0 = qb * kQBlock;
    const uint32_t nqh = min(uint32_t(kQBlock), nq - a0);
    const uint32_t R = tt.kv_count[qb];
    const uint32_t RP = (R + 15) & ~15u;  // padded K/V columns (multiple of 16)
    const uint32_t NT = RP / 8;           // n8 tiles of S
    const uint32_t d = C / heads;
    const uint64_t ld = 3ull * C;

    if (tid < kQBlock) sm.qrow[tid] = (q_frame0 + a0 + min(uint32_t(tid), nqh - 1)) * HW + p;
    if (tid < kKvMax)
        sm.kvrow[tid] = uint32_t(tt.kv_frames[qb * kKvMax + min(uint32_t(tid), R - 1)]) * HW + p;
    __syncthreads();

    const uint32_t q_s = dev::smem_u32(sm.q[0]);
    const uint32_t kv_s = dev::smem_u32(sm.kv[0]);
    const uint32_t pb_s = dev::smem_u32(sm.pb);
    const int mt = warp & 1;         // 16-row m tile of this warp
    const int half = warp >> 1;      // which half of the n tiles

    // loads of one 64-wide chunk: Q rows (phase 1 only) and K or V rows
    auto load_chunk = [&](int buf, uint32_t col0, bool with_q, uint32_t kv_col0) {
        if (with_q) {
            for (int i = tid; i < kQBlock * 8; i += kTcThreads) {
                const uint32_t r = i >> 3, c = i & 7;
                cp_async16(q_s + buf * (kQBlock * 128) + swz(r, c),
                           qkv + uint64_t(sm.qrow[r]) * ld + col0 + c * 8);
            }
        }
        for (int i = tid; i < int(RP) * 8; i += kTcThreads) {
            const uint32_t r = i >> 3, c = i & 7;
            cp_async16(kv_s + buf * (kKvMax * 128) + swz(r, c),
                       qkv + uint64_t(sm.kvrow[r]) * ld + kv_col0 + c * 8);
        }
        cp_commit();
    };

    for (uint32_t h = 0; h < heads; ++h) {
        const uint32_t hc0 = h * d;
        const uint32_t nch = d / kDC;
        // ---------------- phase 1: S = Q K^T ----------------
        float acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[j][k] = 0.f;
        const int nt_per = int(NT) / 2;          // n tiles per warp (1..4)
        const int nt0 = half * nt_per;
        load_chunk(0, hc0, true, C + hc0);
        for (uint32_t ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) {
                load_chunk((ch + 1) & 1, hc0 + (ch + 1) * kDC, true, C + hc0 + (ch + 1) * kDC);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const int buf = ch & 1;
            const uint32_t qa = q_s + buf * (kQBlock * 128);
            const uint32_t ka = kv_s + buf * (kKvMax * 128);
#pragma unroll
            for (int kk = 0; kk < kDC / 16; ++kk) {
                uint32_t a[4];
                {
                    const uint32_t row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    const uint32_t chunk = kk * 2 + (lane >> 4);
                    ldsm_x4(qa + swz(row, chunk), a[0], a[1], a[2], a[3]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j < nt_per) {
                        uint32_t b0, b1;
                        const uint32_t row = (nt0 + j) * 8 + (lane & 7);
                        const uint32_t chunk = kk * 2 + ((lane >> 3) & 1);
                        ldsm_x2(ka + swz(row, chunk), b0, b1);
                        mma_bf16(acc[j], a[0], a[1], a[2], a[3], b0, b1);
                    }
                }
            }
            __syncthreads();
        }
        // ---------------- phase 2: token softmax -> P ----------------
        {
            const int g = lane >> 2, tq = lane & 3;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j < nt_per) {
                    const int col = (nt0 + j) * 8 + tq * 2;
                    sm.s[mt * 16 + g][col] = acc[j][0];
                    sm.s[mt * 16 + g][col + 1] = acc[j][1];
                    sm.s[mt * 16 + g + 8][col] = acc[j][2];
                    sm.s[mt * 16 + g + 8][col + 1] = acc[j][3];
                }
            }
        }
        for (int i = tid; i < kQBlock * kKvMax; i += kTcThreads) (&sm.pf[0][0])[i] = 0.f;
        __syncthreads();
        for (uint32_t a = warp; a < nqh; a += kTcThreads / 32) {
            const uint32_t qa = a0 + a;
            const int n = tt.count[qa];
            const uint8_t* cols = tt.col + size_t(qa) * kMaxTokens;
            const uint8_t* flg = tt.biased + size_t(qa) * kMaxTokens;
            float m = -INFINITY;
            for (int i = lane; i < n; i += 32)
                m = fmaxf(m, scale * sm.s[a][cols[i]] + (flg[i] ? bias : 0.f));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float z = 0.f;
            for (int i = lane; i < n; i += 32) {
                const float e = expf(scale * sm.s[a][cols[i]] + (flg[i] ? bias : 0.f) - m);
                z += e;
                atomicAdd(&sm.pf[a][cols[i]], e);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            if (lane == 0) sm.zinv[a] = 1.0f / z;
        }
        __syncthreads();
        for (int i = tid; i < kQBlock * int(RP) / 8; i += kTcThreads) {
            const uint32_t r = i / (RP / 8), c = i % (RP / 8);  // 8 bf16 per 16B chunk
            const float zi = r < nqh ? sm.zinv[r] : 0.f;
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(sm.pf[r][c * 8 + 2 * k] * zi,
                                                                sm.pf[r][c * 8 + 2 * k + 1] * zi);
                w[k] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            *reinterpret_cast<uint4*>(sm.pb + swz(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        __syncthreads();
        // ---------------- phase 3: ctx = P V ----------------
        load_chunk(0, 0, false, 2 * C + hc0);
        for (uint32_t ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) {
                load_chunk((ch + 1) & 1, 0, false, 2 * C + hc0 + (ch + 1) * kDC);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const uint32_t va = kv_s + (ch & 1) * (kKvMax * 128);
            float o[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) o[j][k] = 0.f;
            for (uint32_t kk = 0; kk < RP / 16; ++kk) {
                uint32_t a[4];
                {
                    const uint32_t row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    const uint32_t chunk = kk * 2 + (lane >> 4);
                    ldsm_x4(pb_s + swz(row, chunk), a[0], a[1], a[2], a[3]);
                }
#pragma unroll
                for (int jp = 0; jp < 2; ++jp) {
                    // two n8 tiles (16 output columns) per x4.trans load
                    uint32_t b[4];
                    const uint32_t row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    const uint32_t chunk = half * 4 + jp * 2 + (lane >> 4);
                    ldsm_x4_t(va + swz(row, chunk), b[0], b[1], b[2], b[3]);
                    mma_bf16(o[jp * 2], a[0], a[1], a[2], a[3], b[0], b[1]);
                    mma_bf16(o[jp * 2 + 1], a[0], a[1], a[2], a[3], b[2], b[3]);
                }
            }
            // stage the 32 x 64 bf16 chunk in the (free) Q buffer, then 16B row stores
            uint8_t* ost = sm.q[0];
            {
                const int g = lane >> 2, tq = lane & 3;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t col = half * 32 + j * 8 + tq * 2;
                    const __nv_bfloat162 lo2 = __floats2bfloat162_rn(o[j][0], o[j][1]);
                    const __nv_bfloat162 hi2 = __floats2bfloat162_rn(o[j][2], o[j][3]);
                    const uint32_t r0 = mt * 16 + g, r1 = r0 + 8;
                    *reinterpret_cast<__nv_bfloat162*>(ost + swz(r0, col >> 3) + (col & 7) * 2) = lo2;
                    *reinterpret_cast<__nv_bfloat162*>(ost + swz(r1, col >> 3) + (col & 7) * 2) = hi2;
                }
            }
            __syncthreads();
            for (int i = tid; i < int(nqh) * 8; i += kTcThreads) {
                const uint32_t r = i >> 3, c = i & 7;
                const uint4 v = *reinterpret_cast<const uint4*>(ost + swz(r, c));
                *reinterpret_cast<uint4*>(ctx + (uint64_t(a0 + r) * HW + p) * C + hc0 + ch * kDC +
                                          c * 8) = v;
            }
            __syncthreads();
        }
    }
}

}  // namespace

bool attention_tc_supported(uint32_t C, uint32_t heads, const TokenTable& tt) {
    return heads > 0 && C % heads == 0 && (C / heads) % kDC == 0 && tt.kv_ok;
}

int launch_attention_core_tc(const void* qkv, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
                             uint32_t q_frame0, TokenTable tt, float scale, float bias, void* ctx,
                             cudaStream_t s) {
    const uint32_t nqb = (nq + kQBlock - 1) / kQBlock;
    const size_t shm = sizeof(TcSmem);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attention_core_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(shm));
        attr = true;
    }
    dim3 grid(HW, nqb);
    attention_core_tc_kernel<<<grid, kTcThreads, shm, s>>>(
        static_cast<const __nv_bfloat16*>(qkv), HW, C, heads, nq, q_frame0, tt, scale, bias,
        static_cast<__nv_bfloat16*>(ctx));
    return int(cudaGetLastError());
}

}  // namespace vinf
