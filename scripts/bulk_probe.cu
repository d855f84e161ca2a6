// Diagnostic: 1D bulk copies global->shared of strided rows, checked against the source.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2406_16260_b200/csrc scripts/bulk_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace vinf;

__global__ void probe(const uint8_t* src, uint64_t stride, uint32_t rowbytes, uint32_t nrows,
                      uint32_t pitch, uint8_t* out, int mode) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + nrows * pitch);
    if (threadIdx.x == 0) {
        dev::mbar_init(bar, 1);
        dev::fence_barrier_init();
    }
    __syncthreads();
    const uint32_t sbase = dev::smem_u32(sm);
    const uint8_t* base = src + uint64_t(blockIdx.x) * rowbytes;
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) dev::mbar_arrive_expect_tx(bar, nrows * rowbytes);
        __syncwarp();
        for (uint32_t i = threadIdx.x; i < nrows; i += 32)
            dev::bulk_g2s(sbase + i * pitch, base + i * stride, rowbytes, bar);
    }
    dev::mbar_wait(bar, 0);
    for (uint32_t i = threadIdx.x; i < nrows * rowbytes; i += blockDim.x) {
        const uint32_t r = i / rowbytes, c = i % rowbytes;
        out[(uint64_t(blockIdx.x) * nrows + r) * rowbytes + c] = sm[r * pitch + c];
    }
}

int main() {
    struct Cfg { uint32_t rowbytes, nrows, blocks; } cfgs[] = {
        {128, 48, 4}, {1280, 48, 4}, {640, 48, 4}, {1280, 48, 2560}, {128, 48, 2560}};
    for (auto c : cfgs) {
        const uint64_t stride = uint64_t(c.rowbytes) * 3 * c.blocks;  // frame stride like QKV
        const size_t n = stride * c.nrows;
        uint8_t *src, *out;
        cudaMalloc(&src, n);
        cudaMalloc(&out, size_t(c.blocks) * c.nrows * c.rowbytes);
        std::vector<uint8_t> h(n);
        for (size_t i = 0; i < n; ++i) h[i] = uint8_t(i * 131 + 7);
        cudaMemcpy(src, h.data(), n, cudaMemcpyHostToDevice);
        const uint32_t pitch = c.rowbytes + 16;
        const size_t shm = c.nrows * pitch + 16;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        probe<<<c.blocks, 256, shm>>>(src, stride, c.rowbytes, c.nrows, pitch, out, 0);
        cudaError_t e = cudaDeviceSynchronize();
        size_t bad = 0;
        if (e == cudaSuccess) {
            std::vector<uint8_t> o(size_t(c.blocks) * c.nrows * c.rowbytes);
            cudaMemcpy(o.data(), out, o.size(), cudaMemcpyDeviceToHost);
            for (uint32_t b = 0; b < c.blocks; ++b)
                for (uint32_t r = 0; r < c.nrows; ++r)
                    for (uint32_t k = 0; k < c.rowbytes; ++k)
                        bad += o[(size_t(b) * c.nrows + r) * c.rowbytes + k] !=
                               h[uint64_t(b) * c.rowbytes + r * stride + k];
        }
        printf("rowbytes=%u nrows=%u blocks=%u -> %s bad=%zu\n", c.rowbytes, c.nrows, c.blocks,
               cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        cudaFree(src);
        cudaFree(out);
    }
    return 0;
}
