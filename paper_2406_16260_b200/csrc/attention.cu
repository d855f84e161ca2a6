// Dual-scope attention core (ops.cpp:209-241 attend_tokens, applied per spatial position
// as in ops.cpp:318-336 / clip_parallel.cpp:311-334). The Q/K/V projections run as
// tcgen05 GEMMs beforehand; this kernel does only the banded+global token mixing,
// which is ~1.5% of block FLOPs and bound by reading Q/K/V once.
//
// One CTA per spatial position; warp w handles query frames a = w, w + nwarps, ...
// For each head: logits over the query's explicit token list (window first, then the
// sampled global frames; duplicates kept, exactly as the reference), +bias on the
// flagged side, max-subtracted softmax in fp32, and ctx = sum p_i v_i with lanes
// striding the head dimension (coalesced K/V row reads; rows of one position are
// re-read by up to 33 queries of the same CTA and hit L1).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kCoreWarps = 4;

template <bool BF16>
__device__ __forceinline__ float ld_elem(const void* base, uint64_t idx) {
    if (BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
    return static_cast<const float*>(base)[idx];
}

// OUT: 0 = fp32 ctx, 1 = bf16 ctx, 2 = split only (bf16 hi/lo planes, fp32 mode operand)
template <bool BF16, int OUT>
__global__ void __launch_bounds__(kCoreWarps * 32)
    attention_core_kernel(const void* __restrict__ qkv, uint32_t HW, uint32_t C, uint32_t heads,
                          uint32_t nq, uint32_t q_frame0, TokenTable tt, float scale, float bias,
                          void* __restrict__ ctx, __nv_bfloat16* __restrict__ hi,
                          __nv_bfloat16* __restrict__ lo) {
    extern __shared__ float sh[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    float* sq = sh + warp * (C + kMaxTokens);  // q row (fp32)
    float* sl = sq + C;                        // logits / weights
    const uint32_t p = blockIdx.x;
    const uint64_t ld = 3ull * C;
    const uint32_t d = C / heads;

    for (uint32_t a = warp; a < nq; a += kCoreWarps) {
        const int n = tt.count[a];
        const uint16_t* rows = tt.rows + size_t(a) * kMaxTokens;
        const uint8_t* flg = tt.biased + size_t(a) * kMaxTokens;
        const uint64_t qrow = uint64_t(q_frame0 + a) * HW + p;
        for (uint32_t c = lane; c < C; c += 32) sq[c] = ld_elem<BF16>(qkv, qrow * ld + c);
        __syncwarp();
        const uint64_t orow = uint64_t(a) * HW + p;
        for (uint32_t h = 0; h < heads; ++h) {
            const uint32_t c0 = h * d;
            for (int i = 0; i < n; ++i) {
                const uint64_t krow = uint64_t(rows[i]) * HW + p;
                const uint64_t kb = krow * ld + C + c0;
                float part = 0.0f;
                for (uint32_t c = lane; c < d; c += 32)
                    part = fmaf(sq[c0 + c], ld_elem<BF16>(qkv, kb + c), part);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                if (lane == 0) sl[i] = scale * part + (flg[i] ? bias : 0.0f);
            }
            __syncwarp();
            float m = -INFINITY;
            for (int i = lane; i < n; i += 32) m = fmaxf(m, sl[i]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float s = 0.0f;
            for (int i = lane; i < n; i += 32) {
                const float e = expf(sl[i] - m);
                sl[i] = e;
                s += e;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            __syncwarp();
            const float inv = 1.0f / s;
            for (uint32_t c = lane; c < d; c += 32) {
                float acc = 0.0f;
                for (int i = 0; i < n; ++i) {
                    const uint64_t vrow = uint64_t(rows[i]) * HW + p;
                    acc = fmaf(sl[i], ld_elem<BF16>(qkv, vrow * ld + 2ull * C + c0 + c), acc);
                }
                const float y = acc * inv;
                const uint64_t oi = orow * C + c0 + c;
                if (OUT == 1)
                    static_cast<__nv_bfloat16*>(ctx)[oi] = __float2bfloat16_rn(y);
                else if (OUT == 0)
                    static_cast<float*>(ctx)[oi] = y;
                if (OUT == 2) {
                    __nv_bfloat16 hh, ll;
                    dev::split_bf16(y, hh, ll);
                    hi[oi] = hh;
                    lo[oi] = ll;
                }
            }
            __syncwarp();
        }
    }
}

}  // namespace

int launch_attention_core(const void* qkv, uint64_t qkv_rows, bool bf16, uint32_t HW, uint32_t C, uint32_t heads,
                          uint32_t nq, uint32_t q_frame0, TokenTable tt, float scale, float bias,
                          void* ctx, bool ctx_bf16, __nv_bfloat16* hi, __nv_bfloat16* lo,
                          cudaStream_t s) {
    if (heads == 0 || C % heads != 0 || HW == 0) return int(cudaErrorInvalidValue);
    if (nq == 0) return 0;
    if (bf16 && ctx_bf16 && hi == nullptr && attention_tc_supported(C, heads, tt))
        return launch_attention_core_tc(qkv, qkv_rows, HW, C, heads, nq, q_frame0, tt, scale, bias, ctx, s);
    const size_t shm = sizeof(float) * kCoreWarps * (C + kMaxTokens);
    if (shm > 200 * 1024) return int(cudaErrorInvalidValue);
    const int out = hi != nullptr ? 2 : (ctx_bf16 ? 1 : 0);
#define AC(B, O)                                                                               \
    if (bf16 == B && out == O) {                                                               \
        if (shm > 48 * 1024)                                                                   \
            cudaFuncSetAttribute(attention_core_kernel<B, O>,                                  \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));       \
        attention_core_kernel<B, O><<<HW, kCoreWarps * 32, shm, s>>>(qkv, HW, C, heads, nq,    \
                                                                     q_frame0, tt, scale,     \
                                                                     bias, ctx, hi, lo);      \
        return int(cudaGetLastError());                                                        \
    }
    AC(false, 0) AC(false, 1) AC(false, 2) AC(true, 0) AC(true, 1) AC(true, 2)
#undef AC
    return int(cudaErrorInvalidValue);
}

}  // namespace vinf
