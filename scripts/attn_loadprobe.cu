// Diagnostic: achievable HBM read bandwidth of the attention core's access patterns
// (loads only, no math). QKV rows of 3C = 1920 bf16; 24 frames x 2560 positions.
//   A: frame-major rows, per CTA (position) 20 chunks of {24 Q rows + 24 K rows (or V)} x 128 B
//   B: position-major rows (a position's 24 frame rows contiguous), same chunk pattern
//   C: position-major, whole 92 KB of a position streamed contiguously (16 B per thread)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/attn_loadprobe.cu -o /tmp/probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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
    for (int v = 0; v < 3; ++v) {
        float best = 1e9;
        for (int it = 0; it < 10; ++it) {
            cudaMemset(flush, it, 512 << 20);
            cudaEventRecord(a);
            if (v == 0) chunks<false><<<HW, 256, NS * 8192>>>(q, sink);
            if (v == 1) chunks<true><<<HW, 256, NS * 8192>>>(q, sink);
            if (v == 2) whole<<<HW, 256, 4 * 16384>>>(q, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%s: %.1f us  %.0f GB/s  (%s)\n", v == 0 ? "A frame-major chunks" : v == 1 ? "B position-major chunks" : "C position-major whole",
               best * 1000, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
