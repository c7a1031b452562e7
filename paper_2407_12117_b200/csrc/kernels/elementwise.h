// elementwise.h — HBM-bound kernels of the Llama block (elementwise.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace memo {

// Counter-hash init, bit-identical to oracle/llama_cpu.c oc_init.
cudaError_t init_uniform(__nv_bfloat16* w, float* master, long long n, uint64_t seed,
                         uint64_t tid, bool is_norm, cudaStream_t st);
cudaError_t embed_fwd(const int* tok, const __nv_bfloat16* E, float* x, int S, int h,
                      cudaStream_t st);
cudaError_t embed_bwd(const int* offsets, const int* pos, const float* dx, float* dE, int V,
                      int h, cudaStream_t st);
// y = bf16((x [+ a]) * rstd * g)
cudaError_t rmsnorm_fwd(const float* x, const __nv_bfloat16* a, const __nv_bfloat16* g,
                        __nv_bfloat16* y, int S, int h, float eps, cudaStream_t st);
int rmsnorm_bwd_partials(int S);
// dx = dres + dnorm(dy); optional bf16 copy; dg (=|+=) column sums via `partial`
// ([rmsnorm_bwd_partials(S), h] f32 workspace).
cudaError_t rmsnorm_bwd(const float* x, const __nv_bfloat16* a, const __nv_bfloat16* g,
                        const float* dy, const float* dres, float* dx, __nv_bfloat16* dx_bf16,
                        float* partial, float* dg, int S, int h, float eps, bool accumulate_dg,
                        cudaStream_t st);
cudaError_t swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* act, long long S, int F,
                       cudaStream_t st);
cudaError_t swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* dact, __nv_bfloat16* dgu,
                       long long S, int F, cudaStream_t st);
cudaError_t cross_entropy(const float* logits, const int* labels, __nv_bfloat16* dlogits,
                          float* loss_rows, int T, int V, const float* inv_n, cudaStream_t st);
cudaError_t sum_scaled(const float* v, long long n, const float* scale, float* out, cudaStream_t st);
// The step counter lives on the device (`step`, incremented by the launch
// itself) so a captured CUDA graph replays the optimizer correctly; `c12`
// (float2) receives the bias corrections 1/(1-b1^t), 1/(1-b2^t).
cudaError_t adamw(float* master, __nv_bfloat16* w, const float* grad, float* m, float* v,
                  long long n, float lr, float b1, float b2, float eps, float wd, int* step,
                  float2* c12, cudaStream_t st);

// Tensor-parallel helpers.
cudaError_t init_sliced(__nv_bfloat16* w, float* master, long long R, long long C,
                        const long long* local0, const long long* count, const long long* global0,
                        int nseg, long long C_glob, long long c_off, uint64_t seed, uint64_t tid,
                        bool is_norm, cudaStream_t st);
cudaError_t resid_round(const float* x, const float* a, __nv_bfloat16* a_bf16, float* out,
                        long long n, cudaStream_t st);
cudaError_t ce_vp_max(const float* logits, float* rmax, int T, int V, cudaStream_t st);
cudaError_t ce_vp_sum(const float* logits, const float* gmax, const int* labels, int v0,
                      float* stats, int T, int V, cudaStream_t st);
cudaError_t ce_vp_grad(const float* logits, const float* gmax, const float* gstats,
                       const int* labels, int v0, __nv_bfloat16* dlogits, float* loss_rows, int T,
                       int V, const float* inv_n, cudaStream_t st);

}  // namespace memo
