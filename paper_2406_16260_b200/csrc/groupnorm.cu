// GroupNorm over [rows, C] clips with contiguous channel groups (ops.cpp:112-173,
// clip_parallel.cpp:211-254). HBM-bound: one streaming read per statistics pass and
// one read + write for the normalise/affine pass, 16 B per lane per access.
//
// Thread mapping: a block is CC x R threads (CC = C / VEC column chunks, R rows) and the
// grid strides over rows by gridDim.x * R, so every thread keeps the SAME VEC channels
// for the whole pass: per-channel affine constants are loaded once, and statistics are
// accumulated per channel in registers (fp32 over a few dozen rows), reduced per block
// into per-group f64 partials, then combined in a fixed order (deterministic, no atomics).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.cuh"

namespace vinf {

namespace {

constexpr int kMaxBlocksPerSm = 2;
constexpr uint32_t kScratchRows = 1024;  // matches the engine layout's kScratchBlocks

template <int VEC, bool BF16>
__device__ __forceinline__ void load_vec(const void* base, uint64_t idx, float (&v)[VEC]) {
    if (VEC == 8) {
        if (BF16) {
            const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + idx);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                v[2 * h] = __uint_as_float(ws[h] << 16);
                v[2 * h + 1] = __uint_as_float(ws[h] & 0xFFFF0000u);
            }
        } else {
            const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx);
            const float4 b = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
            v[k] = BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx + k])
                        : static_cast<const float*>(base)[idx + k];
    }
}

template <int VEC, bool BF16>
__global__ void group_sums_kernel(const void* __restrict__ x, uint64_t rows, uint32_t C,
                                  uint32_t groups, const double* __restrict__ center,
                                  double* __restrict__ partial /* [gridDim.x][groups] */) {
    extern __shared__ double sh[];  // [groups]
    const uint32_t CC = C / VEC;
    const uint32_t R = blockDim.x / CC;
    const uint32_t cc = threadIdx.x % CC;
    const uint32_t rl = threadIdx.x / CC;
    const uint32_t gs = C / groups;
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) sh[g] = 0.0;
    __syncthreads();
    if (rl < R) {
        float ctr[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) ctr[k] = center ? float(center[(cc * VEC + k) / gs]) : 0.0f;
        float acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[k] = 0.0f;
        const uint64_t rstride = uint64_t(gridDim.x) * R;
        for (uint64_t r = uint64_t(blockIdx.x) * R + rl; r < rows; r += rstride) {
            float v[VEC];
            load_vec<VEC, BF16>(x, r * C + cc * VEC, v);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                if (center) {
                    const float d = v[k] - ctr[k];
                    acc[k] = fmaf(d, d, acc[k]);
                } else {
                    acc[k] += v[k];
                }
            }
        }
        // per-channel partials -> per-group f64 in shared memory
#pragma unroll
        for (int k = 0; k < VEC; ++k) atomicAdd(&sh[(cc * VEC + k) / gs], double(acc[k]));
    }
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x)
        partial[uint64_t(blockIdx.x) * groups + g] = sh[g];
}

// sums[g] (+)= sum_b partial[b][g]: one block per output, strided per-thread sums then a
// fixed-shape tree (deterministic for a given nblocks).
__global__ void __launch_bounds__(256)
    group_combine_kernel(const double* __restrict__ partial, uint32_t nblocks, uint32_t groups,
                         double* __restrict__ sums, int accumulate) {
    __shared__ double red[256];
    const uint32_t g = blockIdx.x;
    double s = 0.0;
    for (uint32_t b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[uint64_t(b) * groups + g];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[g] = (accumulate ? sums[g] : 0.0) + red[0];
}

__global__ void group_finalize_kernel(const double* __restrict__ sums, double count,
                                      uint32_t groups, double* __restrict__ stats) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < groups) stats[g] = sums[g] / count;
}

// One streaming pass computing both per-group sum and sum of squares. Thread keeps VEC
// channels; 4 rows in flight per iteration (16 B loads) for memory-level parallelism;
// per-channel fp32 partials -> smem -> per-group f64 partial per block (no atomics;
// combined in block order by group_combine_kernel -> deterministic).
template <bool BF16>
__global__ void __launch_bounds__(256)
    group_moments_partial_kernel(const void* __restrict__ x, uint64_t rows, uint32_t C,
                                 uint32_t groups, double* __restrict__ partial /* [grid][2G] */) {
    constexpr int VEC = 8, UNR = 4;
    extern __shared__ float shm[];  // [R][2][C]
    const uint32_t CC = C / VEC;
    const uint32_t R = blockDim.x / CC;
    const uint32_t cc = threadIdx.x % CC;
    const uint32_t rl = threadIdx.x / CC;
    float s[VEC], q[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) s[k] = q[k] = 0.f;
    if (rl < R) {
        const uint64_t rstride = uint64_t(gridDim.x) * R;
        uint64_t r = uint64_t(blockIdx.x) * R + rl;
        for (; r + (UNR - 1) * rstride < rows; r += UNR * rstride) {
            float v[UNR][VEC];
#pragma unroll
            for (int u = 0; u < UNR; ++u) load_vec<VEC, BF16>(x, (r + u * rstride) * C + cc * VEC, v[u]);
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int k = 0; k < VEC; ++k) {
                    s[k] += v[u][k];
                    q[k] = fmaf(v[u][k], v[u][k], q[k]);
                }
        }
        for (; r < rows; r += rstride) {
            float v[VEC];
            load_vec<VEC, BF16>(x, r * C + cc * VEC, v);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                s[k] += v[k];
                q[k] = fmaf(v[k], v[k], q[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            shm[(rl * 2 + 0) * C + cc * VEC + k] = s[k];
            shm[(rl * 2 + 1) * C + cc * VEC + k] = q[k];
        }
    }
    __syncthreads();
    // per group: f64 sum over its channels and the R row lanes
    const uint32_t gs = C / groups;
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (uint32_t l = 0; l < R; ++l)
            for (uint32_t ch = g * gs; ch < (g + 1) * gs; ++ch) {
                a += double(shm[(l * 2 + 0) * C + ch]);
                b += double(shm[(l * 2 + 1) * C + ch]);
            }
        partial[uint64_t(blockIdx.x) * 2 * groups + g] = a;
        partial[uint64_t(blockIdx.x) * 2 * groups + groups + g] = b;
    }
}

// (sum, sum of squares) -> (mean, variance) in f64.
__global__ void group_moments_kernel(const double* __restrict__ sums, double count,
                                     uint32_t groups, double* __restrict__ stats) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < groups) {
        const double m = sums[g] / count;
        const double v = sums[groups + g] / count - m * m;
        stats[g] = m;
        stats[groups + g] = v > 0.0 ? v : 0.0;
    }
}

constexpr uint32_t kMaxGroupsApply = 1024;

template <int VEC, bool IN_BF16, bool OUT_BF16, bool SPLIT>
__global__ void group_apply_kernel(const void* __restrict__ x, uint64_t rows, uint32_t C,
                                   uint32_t groups, const double* __restrict__ means,
                                   const double* __restrict__ vars,
                                   const float* __restrict__ gamma, const float* __restrict__ beta,
                                   float eps, void* __restrict__ y, __nv_bfloat16* __restrict__ hi,
                                   __nv_bfloat16* __restrict__ lo, double count) {
    dev::pdl_wait();
    dev::pdl_trigger();
    // per-channel (mean, scale, shift) built once per CTA in shared memory: the f64
    // 1/sqrt per group and the f64 gamma product per channel (ops.cpp:152-160) are computed
    // by a few threads instead of every thread redoing them for its 8 channels
    extern __shared__ float tab[];  // [3][C]
    __shared__ double inv_s[kMaxGroupsApply], mu_s[kMaxGroupsApply];
    const uint32_t gs = C / groups;
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) {
        double m, v;
        if (count > 0.0) {  // `means` holds the whole video's (sum, sum of squares)
            m = means[g] / count;
            v = means[groups + g] / count - m * m;
            v = v > 0.0 ? v : 0.0;
        } else {
            m = means[g];
            v = vars[g];
        }
        mu_s[g] = m;
        inv_s[g] = 1.0 / sqrt(v + double(eps));  // ops.cpp:152
    }
    __syncthreads();
    for (uint32_t ch = threadIdx.x; ch < C; ch += blockDim.x) {
        const uint32_t g = ch / gs;
        tab[ch] = float(mu_s[g]);
        tab[C + ch] = float(double(gamma[ch]) * inv_s[g]);
        tab[2 * C + ch] = beta[ch];
    }
    __syncthreads();
    const uint32_t CC = C / VEC;
    const uint32_t R = blockDim.x / CC;
    const uint32_t cc = threadIdx.x % CC;
    const uint32_t rl = threadIdx.x / CC;
    if (rl >= R) return;
    float mu[VEC], sc[VEC], bt[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
        const uint32_t ch = cc * VEC + k;
        mu[k] = tab[ch];
        sc[k] = tab[C + ch];
        bt[k] = tab[2 * C + ch];
    }
    const uint64_t rstride = uint64_t(gridDim.x) * R;
    constexpr int UNR = 4;  // rows in flight per lane
    for (uint64_t r0 = uint64_t(blockIdx.x) * R + rl; r0 < rows; r0 += UNR * rstride) {
      float vin[UNR][VEC];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
          if (r0 + u * rstride < rows) load_vec<VEC, IN_BF16>(x, (r0 + u * rstride) * C + cc * VEC, vin[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint64_t r = r0 + u * rstride;
        if (r >= rows) break;
        const uint64_t idx = r * C + cc * VEC;
        float v[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = fmaf(vin[u][k] - mu[k], sc[k], bt[k]);
        if (OUT_BF16) {
            if (VEC == 8) {
                uint32_t w[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
                    w[h] = *reinterpret_cast<uint32_t*>(&b2);
                }
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(y) + idx) =
                    make_uint4(w[0], w[1], w[2], w[3]);
            } else {
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    static_cast<__nv_bfloat16*>(y)[idx + k] = __float2bfloat16_rn(v[k]);
            }
        } else {
            if (VEC == 8) {
                float* yo = static_cast<float*>(y) + idx;
                *reinterpret_cast<float4*>(yo) = make_float4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<float4*>(yo + 4) = make_float4(v[4], v[5], v[6], v[7]);
            } else {
#pragma unroll
                for (int k = 0; k < VEC; ++k) static_cast<float*>(y)[idx + k] = v[k];
            }
        }
        if (SPLIT) {
            __nv_bfloat16 h[VEC], l[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k) dev::split_bf16(v[k], h[k], l[k]);
            if (VEC == 8) {
                *reinterpret_cast<uint4*>(hi + idx) = *reinterpret_cast<uint4*>(h);
                *reinterpret_cast<uint4*>(lo + idx) = *reinterpret_cast<uint4*>(l);
            } else {
#pragma unroll
                for (int k = 0; k < VEC; ++k) { hi[idx + k] = h[k]; lo[idx + k] = l[k]; }
            }
        }
      }
    }
}

// Block = CC * R threads with R = max(1, 256 / CC); returns 0 if C is too wide.
// bf16 -> bf16 apply (the engine's bf16 mode), shaped like the stub kernel: 16-byte rows
// in flight as raw words (4 registers each) so four CTAs fit an SM; per-channel
// (mean, scale, shift) built once per CTA with the same f64 arithmetic as above, so the
// output bits equal group_apply_kernel<8, true, true, false>'s.
__global__ void __launch_bounds__(256, 4)
    group_apply_bf16_kernel(const uint4* __restrict__ x, uint64_t rows, uint32_t C, uint32_t groups,
                            const double* __restrict__ means, const double* __restrict__ vars,
                            const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                            uint4* __restrict__ y, double count) {
    dev::pdl_wait();
    dev::pdl_trigger();
    extern __shared__ float tab[];  // [3][C]
    __shared__ double inv_s[kMaxGroupsApply], mu_s[kMaxGroupsApply];
    const uint32_t gs = C / groups;
    for (uint32_t g = threadIdx.x; g < groups; g += blockDim.x) {
        double m, v;
        if (count > 0.0) {  // `means` holds the whole video's (sum, sum of squares)
            m = means[g] / count;
            v = means[groups + g] / count - m * m;
            v = v > 0.0 ? v : 0.0;
        } else {
            m = means[g];
            v = vars[g];
        }
        mu_s[g] = m;
        inv_s[g] = 1.0 / sqrt(v + double(eps));  // ops.cpp:152
    }
    __syncthreads();
    for (uint32_t ch = threadIdx.x; ch < C; ch += blockDim.x) {
        const uint32_t g = ch / gs;
        tab[ch] = float(mu_s[g]);
        tab[C + ch] = float(double(gamma[ch]) * inv_s[g]);
        tab[2 * C + ch] = beta[ch];
    }
    __syncthreads();
    constexpr int UNR = 4;
    const uint32_t CC = C / 8, R = blockDim.x / CC;
    const uint32_t cc = threadIdx.x % CC, rl = threadIdx.x / CC;
    if (rl >= R) return;
    float mu[8], sc[8], bt[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        mu[k] = tab[cc * 8 + k];
        sc[k] = tab[C + cc * 8 + k];
        bt[k] = tab[2 * C + cc * 8 + k];
    }
    const uint64_t rstride = uint64_t(gridDim.x) * R;
    for (uint64_t r = uint64_t(blockIdx.x) * R + rl; r < rows; r += UNR * rstride) {
        uint4 w[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (r + u * rstride < rows) w[u] = __ldg(x + (r + u * rstride) * CC + cc);
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (r + u * rstride >= rows) break;
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
            uint32_t o[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float x0 = __uint_as_float(ws[h] << 16), x1 = __uint_as_float(ws[h] & 0xFFFF0000u);
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(fmaf(x0 - mu[2 * h], sc[2 * h], bt[2 * h]),
                                                                fmaf(x1 - mu[2 * h + 1], sc[2 * h + 1], bt[2 * h + 1]));
                o[h] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            y[(r + u * rstride) * CC + cc] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

inline int block_for(uint32_t C, int vec, int* R) {
    const uint32_t CC = C / vec;
    if (CC == 0 || CC > 1024) return 0;
    *R = CC >= 256 ? 1 : int(256 / CC);
    return int(CC) * *R;
}

}  // namespace

uint64_t group_sums_scratch_elems(uint32_t C) {
    return uint64_t(num_sms()) * kMaxBlocksPerSm * (C ? C : 1);
}

int launch_group_sums(const void* x, bool bf16, uint64_t rows, uint32_t C, uint32_t groups,
                      const double* center, double* sums, double* scratch, bool accumulate,
                      cudaStream_t s) {
    if (groups == 0 || C % groups != 0) return int(cudaErrorInvalidValue);
    const int vec = (C % 8 == 0) ? 8 : 1;
    int R = 1;
    const int block = block_for(C, vec, &R);
    if (block == 0) return int(cudaErrorInvalidValue);
    int grid = int((rows + R - 1) / R);
    const int cap = num_sms() * kMaxBlocksPerSm;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    const size_t shm = sizeof(double) * groups;
    if (rows > 0) {
        if (vec == 8) {
            if (bf16) group_sums_kernel<8, true><<<grid, block, shm, s>>>(x, rows, C, groups, center, scratch);
            else group_sums_kernel<8, false><<<grid, block, shm, s>>>(x, rows, C, groups, center, scratch);
        } else {
            if (bf16) group_sums_kernel<1, true><<<grid, block, shm, s>>>(x, rows, C, groups, center, scratch);
            else group_sums_kernel<1, false><<<grid, block, shm, s>>>(x, rows, C, groups, center, scratch);
        }
    } else {
        grid = 0;
    }
    group_combine_kernel<<<groups, 256, 0, s>>>(scratch, uint32_t(grid), groups, sums,
                                                             accumulate ? 1 : 0);
    return int(cudaGetLastError());
}

int launch_group_finalize(const double* sums, double count, uint32_t groups, double* stats,
                          cudaStream_t s) {
    group_finalize_kernel<<<(groups + 127) / 128, 128, 0, s>>>(sums, count, groups, stats);
    return int(cudaGetLastError());
}

int launch_group_moment_sums(const void* x, bool bf16, uint64_t rows, uint32_t C,
                             uint32_t groups, double* sums, double* scratch, cudaStream_t s) {
    if (groups == 0 || C % groups != 0 || C % 8 != 0 || C / 8 > 256)
        return int(cudaErrorInvalidValue);
    const uint32_t CC = C / 8;
    const uint32_t R = 256 / CC;
    const int block = int(CC * R);
    int grid = int(std::min<uint64_t>((rows + R - 1) / R, uint64_t(num_sms()) * 4));
    grid = std::min<int>(grid, int(kScratchRows / 2));
    if (grid < 1) grid = 1;
    const size_t shm = sizeof(float) * 2 * C * R;
    if (shm > 48 * 1024) {
        cudaFuncSetAttribute(group_moments_partial_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
        cudaFuncSetAttribute(group_moments_partial_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm));
    }
    if (bf16)
        group_moments_partial_kernel<true><<<grid, block, shm, s>>>(x, rows, C, groups, scratch);
    else
        group_moments_partial_kernel<false><<<grid, block, shm, s>>>(x, rows, C, groups, scratch);
    // combine [grid][2G] in block order
    group_combine_kernel<<<2 * groups, 256, 0, s>>>(scratch, uint32_t(grid),
                                                                  2 * groups, sums, 0);
    return int(cudaGetLastError());
}

constexpr uint32_t kColSegs = 256;  // sizes the fold scratch (colpart_scratch_elems)

uint64_t colpart_scratch_elems(uint32_t C) { return uint64_t(kColSegs) * 2 * C; }

// Fold of the conv epilogue's 32-row column partials into per-group (sum, sum of squares)
// in one launch: CTA (statistic, group, segment) sums its segment of row blocks (fixed
// per-thread order + fixed tree) into scratch; the last CTA of each (statistic, group)
// — found with an atomic ticket — adds the segment partials in segment order. The
// result is therefore independent of CTA scheduling (bitwise reproducible).
constexpr uint32_t kFoldSegs = 32;

// The conv epilogue's partials are of v = u - b (the stored value minus the per-column
// shift b, the conv bias): summing u^2 in fp32 would cancel catastrophically for channels
// whose mean is far from zero, (u - b)^2 does not. Sums of u follow exactly in f64:
//   sum u   = sum v + M b
//   sum u^2 = sum (v^2 + 2 b v) + M b^2
// so an entry contributes v (which = 0) or v^2 + 2 b v (which = 1; k2 = 2b), and the
// group's constant M * sum_c b_c (or b_c^2) is added once.
__device__ __forceinline__ double colpart_entry(const float* base, uint32_t C, uint32_t row, uint32_t c,
                                                uint32_t which, double k2) {
    const float* r = base + uint64_t(row) * 2 * C + c;
    return which ? double(r[C]) + k2 * double(r[0]) : double(r[0]);
}

__global__ void __launch_bounds__(128)
    colpart_fold_kernel(const float* __restrict__ part, uint32_t blocks, uint32_t C, uint32_t groups,
                        const float* __restrict__ shift, double rows, double* __restrict__ seg,
                        uint32_t* __restrict__ tickets, double* __restrict__ sums) {
    dev::pdl_wait();
    dev::pdl_trigger();
    __shared__ double red[128];
    __shared__ bool last;
    const uint32_t sg = blockIdx.x / kFoldSegs, sid = blockIdx.x % kFoldSegs;  // sg = which*G + g
    const uint32_t which = sg / groups, g = sg % groups, gs = C / groups;
    const uint32_t per = (blocks + kFoldSegs - 1) / kFoldSegs;
    const uint32_t b0 = min(blocks, sid * per), b1 = min(blocks, b0 + per);
    const float* base = part + uint64_t(g) * gs;
    // thread = (row lane, group column): rows b0 + rl, b0 + rl + nrl, ... of one column;
    // a warp reads whole runs of the group's columns, loads independent (no divisions)
    double a = 0.0;
    const uint32_t nrl = gs <= 128 ? 128 / gs : 1;
    const uint32_t rl = threadIdx.x / gs, c = threadIdx.x % gs;
    if (rl < nrl && c < gs && gs <= 128) {
        const double k2 = (which && shift) ? 2.0 * double(shift[g * gs + c]) : 0.0;
        double a1 = 0.0;
        uint32_t b = b0 + rl;
        for (; b + nrl < b1; b += 2 * nrl) {
            a += colpart_entry(base, C, b, c, which, k2);
            a1 += colpart_entry(base, C, b + nrl, c, which, k2);
        }
        if (b < b1) a += colpart_entry(base, C, b, c, which, k2);
        a += a1;
    }
    if (gs > 128) {  // wide groups: every thread strides the columns as well
        a = 0.0;
        for (uint32_t cc = threadIdx.x; cc < gs; cc += 128) {
            const double k2 = (which && shift) ? 2.0 * double(shift[g * gs + cc]) : 0.0;
            for (uint32_t b = b0; b < b1; ++b) a += colpart_entry(base, C, b, cc, which, k2);
        }
    }
    red[threadIdx.x] = a;
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        seg[uint64_t(sg) * kFoldSegs + sid] = red[0];
        __threadfence();
        last = atomicAdd(&tickets[sg], 1u) == kFoldSegs - 1;
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {  // the segment partials, loaded in parallel, fixed tree
        static_assert(kFoldSegs == 32, "one partial per lane");
        __threadfence();
        double t = reinterpret_cast<const volatile double*>(seg)[uint64_t(sg) * kFoldSegs + threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        double st = 0.0;  // the shift constant, one column per lane (loads in parallel)
        if (shift)
            for (uint32_t cc = threadIdx.x; cc < gs; cc += 32) {
                const double bb = double(shift[g * gs + cc]);
                st += which ? bb * bb : bb;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) st += __shfl_xor_sync(0xffffffffu, st, o);
        if (threadIdx.x == 0) {
            sums[which * groups + g] = t + rows * st;
            tickets[sg] = 0;  // ready for the next fold
        }
    }
}

// Few partial rows (the conv GEMM's per-CTA statistics: 4 rows per CTA group): one CTA per
// (statistic, group) reads the group's whole column block, each thread a fixed strided set of
// (row, column) entries in f64, then a fixed tree. No tickets, one dependent step.
constexpr uint32_t kDirectThreads = 256;
constexpr uint32_t kDirectMaxEntries = 16384;  // rows x group width handled by one CTA

__global__ void __launch_bounds__(kDirectThreads)
    colpart_fold_direct_kernel(const float* __restrict__ part, uint32_t blocks, uint32_t C,
                               uint32_t groups, const float* __restrict__ shift, double rows,
                               double* __restrict__ sums) {
    __shared__ double red[kDirectThreads];
    const uint32_t which = blockIdx.x / groups, g = blockIdx.x % groups, gs = C / groups;
    // thread = (row lane rl, group column c): rows rl, rl + nrl, ... of one column, four
    // independent loads in flight; the column's shift (the conv bias, a weight) is read
    // before the dependency wait and its constant rows * b (or b^2) joins the same tree
    const uint32_t nrl = gs <= kDirectThreads ? kDirectThreads / gs : 1;
    const uint32_t rl = threadIdx.x / gs, c = threadIdx.x - rl * gs;
    const bool active = gs <= kDirectThreads && rl < nrl;
    const double b = (active && shift) ? double(__ldg(shift + g * gs + c)) : 0.0;
    const double k2 = which ? 2.0 * b : 0.0;
    dev::pdl_wait();
    dev::pdl_trigger();
    double a = 0.0;
    if (active) {
        const float* col = part + uint64_t(g) * gs + c;
        auto entry = [&](uint32_t r) {
            const float* e = col + uint64_t(r) * 2 * C;
            return which ? double(e[C]) + k2 * double(e[0]) : double(e[0]);
        };
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        uint32_t r = rl;
        for (; r + 3 * nrl < blocks; r += 4 * nrl) {
            a0 += entry(r);
            a1 += entry(r + nrl);
            a2 += entry(r + 2 * nrl);
            a3 += entry(r + 3 * nrl);
        }
        for (; r < blocks; r += nrl) a0 += entry(r);
        a = (a0 + a1) + (a2 + a3);
        if (rl == 0 && shift) a += rows * (which ? b * b : b);
    } else if (gs > kDirectThreads) {  // wide groups: every thread strides the columns too
        for (uint32_t cc = threadIdx.x; cc < gs; cc += kDirectThreads) {
            const double bb = shift ? double(shift[g * gs + cc]) : 0.0;
            const double kk = which ? 2.0 * bb : 0.0;
            for (uint32_t r = 0; r < blocks; ++r) a += colpart_entry(part + uint64_t(g) * gs, C, r, cc, which, kk);
            a += rows * (which ? bb * bb : bb);
        }
    }
    red[threadIdx.x] = a;
    __syncthreads();
    for (uint32_t w = kDirectThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[which * groups + g] = red[0];
}

int launch_colpart_to_groups(const float* part, uint32_t blocks, uint32_t C, uint32_t groups,
                             const float* shift, double rows, double* sums, double* scratch,
                             cudaStream_t s) {
    if (groups == 0 || C % groups != 0) return int(cudaErrorInvalidValue);
    if (uint64_t(blocks) * (C / groups) <= kDirectMaxEntries)
        return int(launch_pdl(colpart_fold_direct_kernel, dim3(2 * groups), dim3(kDirectThreads), 0, s,
                              part, blocks, C, groups, shift, rows, sums));
    // scratch: [2G][kFoldSegs] doubles of segment partials, then 2G uint32 tickets (zero
    // at rest: the workspace is zeroed at creation and every fold resets its tickets)
    double* seg = scratch;
    uint32_t* tickets = reinterpret_cast<uint32_t*>(scratch + uint64_t(2) * groups * kFoldSegs);
    return int(launch_pdl(colpart_fold_kernel, dim3(2 * groups * kFoldSegs), dim3(128), 0, s, part, blocks,
                          C, groups, shift, rows, seg, tickets, sums));
}

// GroupNorm folded into the following projection (bf16 mode): with per-channel
// s_c = gamma_c / sqrt(var_g + eps) and t_c = beta_c - mu_g s_c (the same f64 moments as
// group_apply_bf16_kernel), GN(y) W^T = y (W diag(s))^T + W t. One warp per output row n
// of W [N][C] (16-byte loads): W'[n][:] = bf16(W[n][:] * s) and bias[n] = sum_k W[n][k] t_k
// (fixed-order lane sums + butterfly: deterministic). CTA 0 also stores s and t for the
// O GEMM (residual scale s, bias t).
__global__ void __launch_bounds__(256)
    group_fold_kernel(const double* __restrict__ sums, double count, uint32_t C, uint32_t groups,
                      const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                      const __nv_bfloat16* __restrict__ w, uint32_t N, __nv_bfloat16* __restrict__ wf,
                      float* __restrict__ bias, float* __restrict__ st, const float* __restrict__ shift) {
    extern __shared__ __align__(16) float tab[];  // [2][C]: s, t
    constexpr int kMaxV = 5;   // 16-byte pieces of a row per lane: C <= 1280
    constexpr int kMaxCh = 8;  // channels per thread for (s, t): C <= 8 * blockDim
    const uint32_t lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    const uint32_t n = blockIdx.x * warps + (threadIdx.x >> 5);
    const bool vec = C % 8 == 0 && C <= 32 * 8 * kMaxV;
    // weights do not depend on the preceding kernels: fetch this warp's row and this
    // thread's (gamma, beta) before the dependency wait
    uint4 wr[kMaxV];
#pragma unroll
    for (int i = 0; i < kMaxV; ++i) {
        const uint32_t v = lane + 32 * i;
        wr[i] = (vec && n < N && v < C / 8) ? __ldg(reinterpret_cast<const uint4*>(w + uint64_t(n) * C) + v)
                                             : make_uint4(0u, 0u, 0u, 0u);
    }
    float gm[kMaxCh], bt[kMaxCh], sh[kMaxCh];
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
        const uint32_t ch = threadIdx.x + blockDim.x * i;
        gm[i] = ch < C ? __ldg(gamma + ch) : 0.f;
        bt[i] = ch < C ? __ldg(beta + ch) : 0.f;
        sh[i] = (ch < C && shift) ? __ldg(shift + ch) : 0.f;
    }
    dev::pdl_wait();
    dev::pdl_trigger();
    // mean and variance in f64 from the (all-reduced) sums; the scale in f32 (it is
    // rounded into bf16 weights)
    const uint32_t gs = C / groups;
    const double ic = 1.0 / count;
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
        const uint32_t ch = threadIdx.x + blockDim.x * i;
        if (ch >= C) break;
        const uint32_t g = ch / gs;
        const double m = sums[g] * ic;
        double var = fma(-m, m, sums[groups + g] * ic);
        var = var > 0.0 ? var : 0.0;
        const float sc = gm[i] * rsqrtf(float(var + double(eps)));
        // the normalised tensor holds u - shift (the conv stores its output without the bias):
        // GN(u) = s (u - shift) + beta - s (mu - shift)
        const float t = bt[i] - float(m - double(sh[i])) * sc;
        tab[ch] = sc;
        tab[C + ch] = t;
        if (blockIdx.x == 0 && st) {
            st[ch] = sc;
            st[C + ch] = t;
        }
    }
    __syncthreads();
    if (n >= N) return;
    float acc = 0.f;
    if (vec) {
        uint4* orow = reinterpret_cast<uint4*>(wf + uint64_t(n) * C);
#pragma unroll
        for (int i = 0; i < kMaxV; ++i) {
            const uint32_t v = lane + 32 * i;
            if (v >= C / 8) break;
            const uint32_t in[4] = {wr[i].x, wr[i].y, wr[i].z, wr[i].w};
            const float4 s0 = *reinterpret_cast<const float4*>(tab + v * 8);
            const float4 s1 = *reinterpret_cast<const float4*>(tab + v * 8 + 4);
            const float4 t0 = *reinterpret_cast<const float4*>(tab + C + v * 8);
            const float4 t1 = *reinterpret_cast<const float4*>(tab + C + v * 8 + 4);
            const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            const float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
            uint32_t out[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float w0 = __uint_as_float(in[h] << 16), w1 = __uint_as_float(in[h] & 0xFFFF0000u);
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(w0 * sv[2 * h], w1 * sv[2 * h + 1]);
                out[h] = *reinterpret_cast<const uint32_t*>(&b2);
                acc = fmaf(w0, tv[2 * h], acc);
                acc = fmaf(w1, tv[2 * h + 1], acc);
            }
            orow[v] = make_uint4(out[0], out[1], out[2], out[3]);
        }
    } else {
        for (uint32_t k = lane; k < C; k += 32) {
            const float wk = __bfloat162float(w[uint64_t(n) * C + k]);
            wf[uint64_t(n) * C + k] = __float2bfloat16_rn(wk * tab[k]);
            acc = fmaf(wk, tab[C + k], acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) bias[n] = acc;
}

int launch_group_fold(const double* sums, double count, uint32_t C, uint32_t groups, const float* gamma,
                      const float* beta, float eps, const __nv_bfloat16* w, uint32_t N,
                      __nv_bfloat16* wf, float* bias, float* st, const float* shift, cudaStream_t s) {
    if (groups == 0 || C % groups != 0 || groups > kMaxGroupsApply || count <= 0.0)
        return int(cudaErrorInvalidValue);
    const size_t shm = sizeof(float) * 2 * C;
    if (shm > 48 * 1024 || C > 8 * 256) return int(cudaErrorInvalidValue);
    const uint32_t grid = (N + 7) / 8;  // one warp per row, 8 per CTA (s, t built per CTA)
    return int(launch_pdl(group_fold_kernel, dim3(grid), dim3(256), shm, s, sums, count, C, groups,
                          gamma, beta, eps, w, N, wf, bias, st, shift));
}

int launch_group_moments(const double* sums, double count, uint32_t groups, double* stats,
                         cudaStream_t s) {
    group_moments_kernel<<<(groups + 127) / 128, 128, 0, s>>>(sums, count, groups, stats);
    return int(cudaGetLastError());
}

int launch_group_apply(const void* x, bool in_bf16, uint64_t rows, uint32_t C, uint32_t groups,
                       const double* means, const double* vars, const float* gamma,
                       const float* beta, float eps, void* y, bool out_bf16, __nv_bfloat16* hi,
                       __nv_bfloat16* lo, cudaStream_t s, double count) {
    if (groups == 0 || C % groups != 0) return int(cudaErrorInvalidValue);
    if (rows == 0) return 0;
    const int vec = (C % 8 == 0) ? 8 : 1;
    int R = 1;
    const int block = block_for(C, vec, &R);
    if (block == 0) return int(cudaErrorInvalidValue);
    int grid = int((rows + R - 1) / R);
    const int cap = num_sms() * 4;
    if (grid > cap) grid = cap;
    const bool split = hi != nullptr;
    if (groups > kMaxGroupsApply) return int(cudaErrorInvalidValue);
    const size_t shm = sizeof(float) * 3 * C;
    if (shm > 48 * 1024) return int(cudaErrorInvalidValue);
    if (vec == 8 && in_bf16 && out_bf16 && !split) {
        return int(launch_pdl(group_apply_bf16_kernel, dim3(grid), dim3(block), shm, s,
                              static_cast<const uint4*>(x), rows, C, groups, means, vars, gamma, beta,
                              eps, static_cast<uint4*>(y), count));
    }
#define GA(V, IB, OB, SP)                                                                     \
    if (vec == V && in_bf16 == IB && out_bf16 == OB && split == SP) {                         \
        return int(launch_pdl(group_apply_kernel<V, IB, OB, SP>, dim3(grid), dim3(block), shm, s, \
                              x, rows, C, groups, means, vars, gamma, beta, eps, y, hi, lo,   \
                              count));                                                        \
    }
    GA(8, false, false, false) GA(8, false, false, true) GA(8, true, true, false)
    GA(8, true, true, true) GA(8, false, true, false) GA(8, true, false, false)
    GA(1, false, false, false) GA(1, false, false, true) GA(1, true, true, false)
    GA(1, false, true, false) GA(1, true, false, false)
#undef GA
    return int(cudaErrorInvalidValue);
}

}  // namespace vinf
