// Persistent, warp-specialised tcgen05 GEMM (sm_100a). See gemm_tc.cuh for the contract.
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one thread issues
// tcgen05.mma), warp 2 = TMEM allocator, warps 4..7 = epilogue (TMEM -> registers ->
// bias/residual/convert -> global). Operand tiles are 128 x 64 (A) and BN x 64 (B) bf16,
// TMA-loaded with 128B swizzle into a STAGES-deep mbarrier ring. The fp32 accumulator
// lives in TMEM, double-buffered (2 x BN columns) so the epilogue of tile i overlaps
// the main loop of tile i+1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm_tc.cuh"

namespace vinf {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 256;
constexpr uint32_t kABytes = kBM * kBK * 2;

template <int BN>
struct TileCfg {
    static constexpr uint32_t kBBytes = BN * kBK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = std::min<int>(8, (200 * 1024) / kStageBytes);
    static constexpr uint32_t kAccStride = BN <= 128 ? 128 : 256;  // TMEM columns per buffer
    static constexpr uint32_t kTmemCols = 2 * kAccStride;
    static constexpr uint32_t kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*bars*/;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dev::smem_u32(bar)) : "memory");
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ GemmParams p) {
    using Cfg = TileCfg<BN>;
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
            dev::mbar_init(&tempty[i], 4);
        }
        dev::fence_barrier_init();
    }
    if (warp == 2) dev::tmem_alloc(tmem_holder, Cfg::kTmemCols);
    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

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
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int row_in_tile = q * 32 + lane;
        uint32_t local = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const uint32_t acc = local & 1;
            const int m0 = (tile / n_tiles) * kBM;
            const int n0 = (tile % n_tiles) * BN;
            dev::mbar_wait(&tfull[acc], (local >> 1) & 1);
            dev::tc_fence_after();
            const int64_t gm = int64_t(m0) + row_in_tile;
            const bool row_ok = gm < p.M;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                dev::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * Cfg::kAccStride + c,
                                        r);
                dev::tmem_wait_ld();
                const int n_base = n0 + c;
                const int n_lim = min(p.N, n0 + BN);
                if (!row_ok || n_base >= n_lim) continue;
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                const bool full_chunk = (n_base + 32 <= n_lim);
                if (full_chunk) {
                    if (p.bias) {
                        const float4* b4 = reinterpret_cast<const float4*>(p.bias + n_base);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 b = __ldg(b4 + j);
                            v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
                        }
                    }
                    if (p.res) {
                        if (p.res_bf16) {
                            const uint4* r4 = reinterpret_cast<const uint4*>(
                                static_cast<const __nv_bfloat16*>(p.res) + gm * p.res_ld + n_base);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint4 w = __ldg(r4 + j);
                                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                for (int h = 0; h < 4; ++h) {
                                    v[8 * j + 2 * h] += __uint_as_float(ws[h] << 16);
                                    v[8 * j + 2 * h + 1] += __uint_as_float(ws[h] & 0xFFFF0000u);
                                }
                            }
                        } else {
                            const float4* r4 = reinterpret_cast<const float4*>(
                                static_cast<const float*>(p.res) + gm * p.res_ld + n_base);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float4 w = __ldg(r4 + j);
                                v[4 * j] += w.x; v[4 * j + 1] += w.y; v[4 * j + 2] += w.z; v[4 * j + 3] += w.w;
                            }
                        }
                    }
                    if (p.out_bf16) {
                        uint4* o4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) +
                                                             gm * p.out_ld + n_base);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint32_t w[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const __nv_bfloat162 b2 =
                                    __floats2bfloat162_rn(v[8 * j + 2 * h], v[8 * j + 2 * h + 1]);
                                w[h] = *reinterpret_cast<const uint32_t*>(&b2);
                            }
                            o4[j] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    } else {
                        float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(p.out) +
                                                               gm * p.out_ld + n_base);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    }
                } else {
                    for (int j = 0; j < 32 && n_base + j < n_lim; ++j) {
                        const int64_t n = n_base + j;
                        float x = v[j];
                        if (p.bias) x += p.bias[n];
                        if (p.res) {
                            x += p.res_bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(
                                                  p.res)[gm * p.res_ld + n])
                                            : static_cast<const float*>(p.res)[gm * p.res_ld + n];
                        }
                        if (p.out_bf16)
                            static_cast<__nv_bfloat16*>(p.out)[gm * p.out_ld + n] =
                                __float2bfloat16_rn(x);
                        else
                            static_cast<float*>(p.out)[gm * p.out_ld + n] = x;
                    }
                }
            }
            dev::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }

    dev::tc_fence_before();
    __syncthreads();
    dev::tc_fence_after();
    if (warp == 2) dev::tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

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

int g_num_sms = 0;

template <int BN>
int launch(const GemmMaps& maps, const GemmParams& p, cudaStream_t stream) {
    using Cfg = TileCfg<BN>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN>,
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
    const int tiles = ((p.N + BN - 1) / BN) * ((p.M + kBM - 1) / kBM);
    const int grid = std::max(1, std::min(tiles, g_num_sms));
    gemm_tc_kernel<BN><<<grid, kThreads, Cfg::kSmemBytes, stream>>>(maps, p);
    return int(cudaGetLastError());
}

}  // namespace

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

int gemm_pick_block_n(int N) {
    static const int cands[] = {256, 240, 192, 160, 128, 64};
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
    if (p.M <= 0 || p.N <= 0 || p.K <= 0 || p.nseg <= 0 || p.nseg > kGemmMaxSeg)
        return int(cudaErrorInvalidValue);
    switch (block_n) {
        case 256: return launch<256>(maps, p, stream);
        case 240: return launch<240>(maps, p, stream);
        case 192: return launch<192>(maps, p, stream);
        case 160: return launch<160>(maps, p, stream);
        case 128: return launch<128>(maps, p, stream);
        case 64: return launch<64>(maps, p, stream);
        default: return int(cudaErrorInvalidValue);
    }
}

}  // namespace vinf
