// Bandwidth-bound elementwise kernels: seeded synthetic fill (bit-exact SplitMix64,
// rng.hpp:14-26 / tensor.cpp:98-106), the per-frame spatial stub (ops.cpp:42-55),
// and the fp32 -> (bf16 hi, bf16 lo) operand split used by the fp32 ("bf16x3") mode.
// All vectorised 16 B per lane, grid-stride, grid sized to a multiple of the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

bool pdl_enabled() {
    static const bool on = getenv("VINF_NO_PDL") == nullptr;
    return on;
}

namespace {

__device__ __forceinline__ float unit_from_state(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const uint32_t top24 = uint32_t(z >> 40);
    // exact in binary32: k * 2^-23 - 1 with k < 2^24
    return __fsub_rn(__fmul_rn(float(top24), 2.0f / 16777216.0f), 1.0f);
}

template <bool BF16>
__global__ void fill_seeded_kernel(void* out, uint64_t n, uint64_t seed, uint64_t first,
                                   float scale, int apply_scale) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        // state after (first + i + 1) draws
        const uint64_t z = seed + (first + i + 1) * 0x9E3779B97F4A7C15ull;
        float u = unit_from_state(z);
        if (apply_scale) u = __fmul_rn(u, scale);
        if (BF16)
            static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(u);
        else
            static_cast<float*>(out)[i] = u;
    }
}

// o = tanh(a[c] * x + c[c]); separate rounding of mul and add (no FMA contraction),
// as the reference evaluates it in binary32.
__device__ __forceinline__ float stub_fn(float x, float a, float c) {
    return tanhf(__fadd_rn(__fmul_rn(a, x), c));
}

// bf16 -> bf16 fast path (bf16 mode): 16 B in / 16 B out per lane, hardware tanh.approx
// (max rel. error ~2^-11, below the bf16 output rounding of 2^-9).
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Thread mapping as in the GroupNorm kernels: a block is CC x R threads (CC = C / 8), the
// grid strides over rows, so each lane keeps the same 8 channels (coefficients loaded
// once) and keeps UNR rows of 16 B loads in flight.
__global__ void __launch_bounds__(256)
    stub_bf16_kernel(const uint4* __restrict__ in, uint64_t rows, uint32_t C,
                     const float* __restrict__ a, const float* __restrict__ c,
                     uint4* __restrict__ out) {
    dev::pdl_wait();
    dev::pdl_trigger();
    constexpr int UNR = 4;
    const uint32_t CC = C / 8, R = blockDim.x / CC;
    const uint32_t cc = threadIdx.x % CC, rl = threadIdx.x / CC;
    if (rl >= R) return;
    float ka[8], kc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        ka[k] = __ldg(a + cc * 8 + k);
        kc[k] = __ldg(c + cc * 8 + k);
    }
    const uint64_t rstride = uint64_t(gridDim.x) * R;
    for (uint64_t r = uint64_t(blockIdx.x) * R + rl; r < rows; r += UNR * rstride) {
        uint4 w[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (r + u * rstride < rows) w[u] = __ldg(in + (r + u * rstride) * CC + cc);
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (r + u * rstride >= rows) break;
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
            uint32_t o[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float x0 = __uint_as_float(ws[h] << 16), x1 = __uint_as_float(ws[h] & 0xFFFF0000u);
                const float y0 = tanh_fast(fmaf(ka[2 * h], x0, kc[2 * h]));
                const float y1 = tanh_fast(fmaf(ka[2 * h + 1], x1, kc[2 * h + 1]));
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(y0, y1);
                o[h] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            out[(r + u * rstride) * CC + cc] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

template <bool IN_BF16, bool OUT_BF16, bool SPLIT>
__global__ void stub_kernel(const void* __restrict__ in, uint64_t n, uint32_t C,
                            const float* __restrict__ a, const float* __restrict__ c,
                            void* __restrict__ out, __nv_bfloat16* __restrict__ hi,
                            __nv_bfloat16* __restrict__ lo) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t nv = n / 4;
    for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv; v += stride) {
        const uint64_t i = v * 4;
        float x[4];
        if (IN_BF16) {
            const uint2 w = reinterpret_cast<const uint2*>(in)[v];
            x[0] = __uint_as_float(w.x << 16);
            x[1] = __uint_as_float(w.x & 0xFFFF0000u);
            x[2] = __uint_as_float(w.y << 16);
            x[3] = __uint_as_float(w.y & 0xFFFF0000u);
        } else {
            const float4 w = reinterpret_cast<const float4*>(in)[v];
            x[0] = w.x; x[1] = w.y; x[2] = w.z; x[3] = w.w;
        }
        const uint32_t ch = uint32_t(i % C);
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) y[k] = stub_fn(x[k], __ldg(a + ch + k), __ldg(c + ch + k));
        if (OUT_BF16) {
            __nv_bfloat162 p0 = __floats2bfloat162_rn(y[0], y[1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(y[2], y[3]);
            reinterpret_cast<uint2*>(out)[v] =
                make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
        } else {
            reinterpret_cast<float4*>(out)[v] = make_float4(y[0], y[1], y[2], y[3]);
        }
        if (SPLIT) {
            __nv_bfloat16 h[4], l[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) dev::split_bf16(y[k], h[k], l[k]);
            reinterpret_cast<uint2*>(hi)[v] = *reinterpret_cast<uint2*>(h);
            reinterpret_cast<uint2*>(lo)[v] = *reinterpret_cast<uint2*>(l);
        }
    }
}

template <bool IN_BF16>
__global__ void split_kernel(const void* __restrict__ in, uint64_t n,
                             __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float x = IN_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(in)[i])
                                : static_cast<const float*>(in)[i];
        __nv_bfloat16 h, l;
        dev::split_bf16(x, h, l);
        hi[i] = h;
        if (lo) lo[i] = l;
    }
}

__global__ void cast_kernel(const void* __restrict__ in, int in_bf16, void* __restrict__ out,
                            int out_bf16, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float x = in_bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(in)[i])
                                : static_cast<const float*>(in)[i];
        if (out_bf16)
            static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(x);
        else
            static_cast<float*>(out)[i] = x;
    }
}

// x = x - lambda * eps in f64 arithmetic, rounded to the storage type
// (euler_update_inplace, pipeline.cpp:93-100).
template <bool BF16>
__global__ void euler_kernel(void* __restrict__ x, const void* __restrict__ eps, uint64_t n,
                             double lambda) {
    dev::pdl_wait();
    dev::pdl_trigger();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (BF16) {
            auto* px = static_cast<__nv_bfloat16*>(x);
            const double v = double(__bfloat162float(px[i])) -
                             lambda * double(__bfloat162float(static_cast<const __nv_bfloat16*>(eps)[i]));
            px[i] = __float2bfloat16_rn(float(v));
        } else {
            auto* px = static_cast<float*>(x);
            px[i] = float(double(px[i]) - lambda * double(static_cast<const float*>(eps)[i]));
        }
    }
}

// out[c][r] = in[r][c] through a 32 x 33 tile (weight layout change, once per set_block)
__global__ void transpose_kernel(const float* __restrict__ in, float* __restrict__ out, uint32_t rows,
                                 uint32_t cols) {
    __shared__ float t[32][33];
    const uint32_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (uint32_t i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint32_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[i][threadIdx.x] = in[uint64_t(r) * cols + c];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint32_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[uint64_t(c) * rows + r] = t[threadIdx.x][i];
    }
}

}  // namespace

int launch_transpose_f32(const float* in, float* out, uint32_t rows, uint32_t cols, cudaStream_t s) {
    if (!rows || !cols) return 0;
    transpose_kernel<<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(in, out, rows, cols);
    return int(cudaGetLastError());
}

int launch_euler(void* x, const void* eps, bool bf16, uint64_t n, double lambda, cudaStream_t s) {
    if (n == 0) return 0;
    if (bf16)
        return int(launch_pdl(euler_kernel<true>, dim3(grid_for(n, 256)), dim3(256), 0, s, x, eps, n, lambda));
    return int(launch_pdl(euler_kernel<false>, dim3(grid_for(n, 256)), dim3(256), 0, s, x, eps, n, lambda));
}

int grid_for(uint64_t work_items, int block) {
    const uint64_t want = (work_items + block - 1) / block;
    const uint64_t cap = uint64_t(num_sms()) * 8;
    return int(want < 1 ? 1 : (want > cap ? cap : want));
}

int launch_fill_seeded(void* out, bool bf16, uint64_t n, uint64_t seed, uint64_t first,
                       float scale, cudaStream_t s) {
    if (n == 0) return 0;
    const int apply = scale != 1.0f;
    if (bf16)
        fill_seeded_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(out, n, seed, first, scale, apply);
    else
        fill_seeded_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(out, n, seed, first, scale, apply);
    return int(cudaGetLastError());
}

int launch_stub(const void* in, bool in_bf16, uint64_t n, uint32_t C, const float* a,
                const float* c, void* out, bool out_bf16, __nv_bfloat16* hi, __nv_bfloat16* lo,
                cudaStream_t s) {
    if (n == 0) return 0;
    if (C % 4 != 0 || n % 4 != 0) return int(cudaErrorInvalidValue);
    if (in_bf16 && out_bf16 && hi == nullptr && C % 8 == 0 && C / 8 <= 256) {
        const uint32_t CC = C / 8, R = 256 / CC;
        const uint64_t rows = n / C;
        uint64_t grid = (rows + R - 1) / R;
        const uint64_t cap = uint64_t(num_sms()) * 4;
        if (grid > cap) grid = cap;
        return int(launch_pdl(stub_bf16_kernel, dim3(unsigned(grid)), dim3(CC * R), 0, s,
                              static_cast<const uint4*>(in), rows, C, a, c, static_cast<uint4*>(out)));
    }
    const uint64_t nv = n / 4;
    const int g = grid_for(nv, 256);
    const bool split = hi != nullptr;
#define STUB_CASE(IB, OB, SP)                                                              \
    if (in_bf16 == IB && out_bf16 == OB && split == SP) {                                  \
        stub_kernel<IB, OB, SP><<<g, 256, 0, s>>>(in, n, C, a, c, out, hi, lo);            \
        return int(cudaGetLastError());                                                    \
    }
    STUB_CASE(false, false, false)
    STUB_CASE(false, false, true)
    STUB_CASE(true, true, false)
    STUB_CASE(true, true, true)
    STUB_CASE(false, true, false)
    STUB_CASE(true, false, false)
    STUB_CASE(true, false, true)
    STUB_CASE(false, true, true)
#undef STUB_CASE
    return int(cudaErrorInvalidValue);
}

int launch_split(const void* in, bool in_bf16, uint64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo,
                 cudaStream_t s) {
    if (n == 0) return 0;
    if (in_bf16)
        split_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(in, n, hi, lo);
    else
        split_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(in, n, hi, lo);
    return int(cudaGetLastError());
}

int launch_cast(const void* in, bool in_bf16, void* out, bool out_bf16, uint64_t n,
                cudaStream_t s) {
    if (n == 0) return 0;
    cast_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, in_bf16, out, out_bf16, n);
    return int(cudaGetLastError());
}

}  // namespace vinf
