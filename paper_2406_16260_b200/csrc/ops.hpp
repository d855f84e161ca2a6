// Operator forms (device tensors) behind the C ABI; see ops.cpp.
#pragma once

#include "host.hpp"

namespace vinf {

size_t elem_size(vinf_dtype t);
void check_tensor(const vinf_tensor* t, const char* what);
uint64_t numel(const vinf_tensor* t);

// Stream-ordered temporary (cudaMallocAsync / cudaFreeAsync).
struct TmpBuf {
    TmpBuf(size_t bytes, cudaStream_t s);
    ~TmpBuf();
    TmpBuf(const TmpBuf&) = delete;
    TmpBuf& operator=(const TmpBuf&) = delete;
    void* p = nullptr;
    cudaStream_t s_;
};

struct ActOperand {
    ActOperand(const void* data, vinf_dtype dt, uint64_t rows, uint32_t C, cudaStream_t s);
    TmpBuf planes;
    Operand op;
};

void conv_over_extended(const vinf_tensor* ext, uint32_t out_start, uint32_t out_len,
                        const vinf_conv_kernel* k, const vinf_tensor* out, cudaStream_t s);
void group_sums(const vinf_tensor* v, uint32_t groups, const double* center, double* sums,
                cudaStream_t s);
void group_stat(const vinf_tensor* v, uint32_t groups, const double* center, double* out,
                cudaStream_t s);
void normalize_with_stats(const vinf_tensor* v, const vinf_group_norm_params* p,
                          const double* means, const double* vars, const vinf_tensor* out,
                          cudaStream_t s);
void group_norm(const vinf_tensor* v, const vinf_group_norm_params* p, const vinf_tensor* out,
                cudaStream_t s);
void dual_scope(const vinf_tensor* v, double t, const vinf_attention_params* p,
                const vinf_dual_scope_config* cfg, const vinf_tensor* out, cudaStream_t s);
void attention_full(const vinf_tensor* v, const vinf_attention_params* p, const vinf_tensor* out,
                    cudaStream_t s);
void conv_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                   const vinf_tensor* pre, const vinf_tensor* post, const vinf_conv_kernel* k,
                   const vinf_tensor* out, cudaStream_t s);
void attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                        const vinf_tensor* pre, const vinf_tensor* post, const vinf_tensor* glob,
                        double t, const vinf_attention_params* p,
                        const vinf_dual_scope_config* cfg, const vinf_tensor* out,
                        cudaStream_t s);

}  // namespace vinf
