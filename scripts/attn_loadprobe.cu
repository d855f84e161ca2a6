// Diagnostic: achievable HBM read bandwidth of the attention core's access patterns
// (loads only, no math). QKV rows of 3C = 1920 bf16; 24 frames x 2560 positions.
//   A: frame-major rows, per CTA (position) 20 chunks of {24 Q rows + 24 K rows (or V)} x 128 B
//   B: position-major rows (a position's 24 frame rows contiguous), same chunk pattern
//   C: position-major, whole 92 KB of a position streamed contiguously (16 B per thread)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/attn_loadprobe.cu -o /tmp/probe
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

constexpr int F = 24, HW = 2560, C3 = 1920, NS = 6;

__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool POSMAJOR>
__global__ void __launch_bounds__(256) chunks(const uint16_t* q, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, p = blockIdx.x;
    const int r = tid >> 3, pc = tid & 7;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    auto row = [&](int f) -> const uint16_t* {
        const uint64_t rr = POSMAJOR ? uint64_t(p) * F + f : uint64_t(f) * HW + p;
        return q + rr * C3 + pc * 8;
    };
    const uint16_t* src = row(r < F ? r : F - 1);
    int issued = 0;
    auto issue = [&]() {
        if (issued < 20) {
            const int qk = issued < 10;
            const int col = (qk ? issued : issued - 10) * 64;
            const uint32_t st = sb + (issued % NS) * 8192;
            if (r < F) {
                if (qk) cp16(st + r * 128 + pc * 16, src + col);
                cp16(st + 4096 + r * 128 + pc * 16, src + (qk ? 640 : 1280) + col);
            }
        }
        commit();
        ++issued;
    };
    for (int i = 0; i < NS - 1; ++i) issue();
    float acc = 0.f;
    for (int i = 0; i < 20; ++i) {
        waitg<NS - 2>();
        __syncthreads();
        issue();
        acc += reinterpret_cast<const float*>(sm + (i % NS) * 8192)[tid];
    }
    waitg<0>();
    if (acc == 123.f) sink[p] = acc;
}

__global__ void __launch_bounds__(256) whole(const uint16_t* q, float* sink) {
    // position-major: a position's 24 rows x 3840 B = 92160 B contiguous; 6 x 16 KB stages
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, p = blockIdx.x;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(q) + uint64_t(p) * F * C3 * 2;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    constexpr int kChunk = 4096 * 4, nchunk = F * C3 * 2 / kChunk;  // 16 KB pieces: 5.6 -> 6
    int issued = 0;
    auto issue = [&]() {
        if (issued < nchunk + 1) {
            for (int k = 0; k < kChunk / 16 / 256; ++k) {
                const uint64_t off = uint64_t(issued) * kChunk + (k * 256 + tid) * 16;
                if (off < uint64_t(F) * C3 * 2) cp16(sb + (issued % 4) * kChunk + (k * 256 + tid) * 16, base + off);
            }
        }
        commit();
        ++issued;
    };
    for (int i = 0; i < 3; ++i) issue();
    float acc = 0.f;
    for (int i = 0; i < nchunk + 1; ++i) {
        waitg<2>();
        __syncthreads();
        issue();
        acc += reinterpret_cast<const float*>(sm + (i % 4) * kChunk)[tid];
    }
    waitg<0>();
    if (acc == 123.f) sink[p] = acc;
}


// D: TMA 3D box loads ({64 ch, 1 position, 24 frames}, SW128) issued by one thread,
// completion on per-slot mbarriers; one __syncthreads per chunk for slot reuse.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256) tma_chunks(const __grid_constant__ CUtensorMap map, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NS * 8192);
    const int tid = threadIdx.x, p = blockIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int i) {
        if (tid != 0 || i >= 20) return;
        const int s = i % NS;
        const int qk = i < 10;
        const int col = (qk ? i : i - 10) * 64;
        const uint32_t st = su32(sm + s * 8192);
        const uint32_t bar = su32(&bars[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(qk ? 6144 : 3072) : "memory");
        if (qk)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(st), "l"(&map), "r"(col), "r"(p), "r"(0), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(st + 4096), "l"(&map), "r"((qk ? 640 : 1280) + col), "r"(p), "r"(0), "r"(bar) : "memory");
    };
    for (int i = 0; i < NS - 1; ++i) issue(i);
    float acc = 0.f;
    for (int i = 0; i < 20; ++i) {
        const uint32_t bar = su32(&bars[i % NS]);
        const uint32_t par = (i / NS) & 1;
        asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(par) : "memory");
        __syncthreads();
        issue(i + NS - 1);
        acc += reinterpret_cast<const float*>(sm + (i % NS) * 8192)[tid];
    }
    if (acc == 123.f) sink[p] = acc;
}

// E: frame-major whole rows (3840 B per (frame, position)) by cp.async.bulk, one thread
// issuing; persistent CTAs with two position buffers (the next position loads while the
// current one is consumed).
__global__ void __launch_bounds__(256) rows_bulk(const uint16_t* q, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr uint32_t kRow = C3 * 2, kPitch = kRow + 16, kBuf = F * kPitch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * kBuf);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int p, int b) {
        const uint32_t bar = su32(&bars[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(F * kRow) : "memory");
        for (int f = 0; f < F; ++f) {
            const uint16_t* src = q + (uint64_t(f) * HW + p) * C3;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm + b * kBuf + f * kPitch)), "l"(src), "r"(kRow), "r"(bar) : "memory");
        }
    };
    float acc = 0.f;
    int it = 0;
    if (tid == 0 && blockIdx.x < HW) issue(blockIdx.x, 0);
    for (int p = blockIdx.x; p < HW; p += gridDim.x, ++it) {
        const int b = it & 1;
        if (tid == 0 && p + int(gridDim.x) < HW) issue(p + gridDim.x, b ^ 1);
        const uint32_t bar = su32(&bars[b]);
        const uint32_t par = (it >> 1) & 1;
        asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(par) : "memory");
        acc += reinterpret_cast<const float*>(sm + b * kBuf)[tid];
        __syncthreads();
    }
    if (acc == 123.f) sink[0] = acc;
}

int main() {
    uint16_t* q;
    float* sink;
    const size_t n = size_t(F) * HW * C3;
    cudaMalloc(&q, n * 2);
    cudaMalloc(&sink, HW * 4);
    cudaMemset(q, 0, n * 2);
    uint8_t* flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(chunks<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 8192);
    cudaFuncSetAttribute(chunks<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 8192);
    cudaFuncSetAttribute(whole, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    const double bytes = double(F) * HW * C3 * 2;
    CUtensorMap map;
    {
        PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &qr);
        cuuint64_t gdim[3] = {C3, HW, F};
        cuuint64_t gstr[2] = {C3 * 2ull, uint64_t(HW) * C3 * 2};
        cuuint32_t box[3] = {64, 1, 24};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)q, gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) printf("tensor map encode failed %d\n", int(r));
    }
    cudaFuncSetAttribute(tma_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 8192 + 1024);
    const int rows_smem = 2 * F * (C3 * 2 + 16) + 64;
    cudaFuncSetAttribute(rows_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, rows_smem);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int v = 0; v < 5; ++v) {
        float best = 1e9;
        for (int it = 0; it < 10; ++it) {
            cudaMemset(flush, it, 512 << 20);
            cudaEventRecord(a);
            if (v == 0) chunks<false><<<HW, 256, NS * 8192>>>(q, sink);
            if (v == 1) chunks<true><<<HW, 256, NS * 8192>>>(q, sink);
            if (v == 2) whole<<<HW, 256, 4 * 16384>>>(q, sink);
            if (v == 3) tma_chunks<<<HW, 256, NS * 8192 + 1024>>>(map, sink);
            if (v == 4) rows_bulk<<<nsm, 256, rows_smem>>>(q, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%s: %.1f us  %.0f GB/s  (%s)\n", v == 0 ? "A frame-major chunks" : v == 1 ? "B position-major chunks" : v == 2 ? "C position-major whole" : v == 3 ? "D frame-major TMA boxes" : "E frame-major whole rows, bulk, 2 buffers/SM",
               best * 1000, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
