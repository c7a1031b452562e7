// capi_kernels.cu — C-ABI entry points for the individual sm_100a kernels.
#include <cuda_runtime.h>

#include <string>

#include "host/status.hpp"
#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/gemm_tc.h"
#include "memo.h"

using memo::set_error;

extern "C" int memo_gemm(const memo_gemm_args* a, void* stream) {
  if (!a) return set_error(MEMO_ERR_INPUT, "memo_gemm: null args");
  memo::GemmDesc d;
  d.M = a->M;
  d.N = a->N;
  d.K = a->K;
  d.a = a->a;
  d.lda = a->lda;
  d.a_mn_major = a->a_mn_major;
  d.b = a->b;
  d.ldb = a->ldb;
  d.b_mn_major = a->b_mn_major;
  d.epi = a->epilogue;
  d.c = a->c;
  d.ldc = a->ldc;
  d.out_f32 = a->out_f32;
  d.resid = a->resid;
  d.ld_f32 = a->ld_f32;
  d.q = static_cast<__nv_bfloat16*>(a->q);
  d.k = static_cast<__nv_bfloat16*>(a->k);
  d.v = static_cast<__nv_bfloat16*>(a->v);
  d.hidden = a->hidden;
  d.head_dim = a->head_dim;
  d.rope = a->rope;
  d.pos0 = a->pos0;
  d.variant = a->variant;
  d.raster = a->raster;
  cudaError_t e = memo::gemm_tc(d, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(MEMO_ERR_INTERNAL, std::string("memo_gemm: ") + cudaGetErrorString(e));
  return MEMO_OK;
}

extern "C" int memo_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                             int32_t S, int32_t H, int32_t D, float scale, void* stream) {
  memo::AttnFwdArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.S = S;
  a.H = H;
  a.D = D;
  a.softmax_scale = scale;
  cudaError_t e = memo::attn_fwd(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(MEMO_ERR_INTERNAL, std::string("memo_attn_fwd: ") + cudaGetErrorString(e));
  return MEMO_OK;
}

extern "C" uint64_t memo_attn_bwd_workspace_bytes(int32_t S, int32_t H, int32_t D) {
  return static_cast<uint64_t>(memo::attn_bwd_workspace_bytes(S, H, D));
}

extern "C" int memo_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                             const float* lse, const void* dout, float* delta, void* dq, void* dk,
                             void* dv, int64_t ld, const void* rope, int64_t pos0, int32_t S,
                             int32_t H, int32_t D, float scale, void* stream) {
  return memo_attn_bwd_timed(q, k, v, o, lse, dout, delta, dq, dk, dv, ld, rope, pos0, S, H, D,
                             scale, stream, nullptr);
}

extern "C" int memo_attn_bwd_timed(const void* q, const void* k, const void* v, const void* o,
                                   const float* lse, const void* dout, float* delta, void* dq,
                                   void* dk, void* dv, int64_t ld, const void* rope, int64_t pos0,
                                   int32_t S, int32_t H, int32_t D, float scale, void* stream,
                                   float* ms3) {
  memo::AttnBwdArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<const __nv_bfloat16*>(o);
  a.lse = lse;
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.delta = delta;
  a.dq = static_cast<__nv_bfloat16*>(dq);
  a.dk = static_cast<__nv_bfloat16*>(dk);
  a.dv = static_cast<__nv_bfloat16*>(dv);
  a.ld_dqkv = ld;
  a.rope = rope;
  a.pos0 = pos0;
  a.S = S;
  a.H = H;
  a.D = D;
  a.softmax_scale = scale;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (ms3) {
    for (auto& x : ev) cudaEventCreate(&x);
    for (int i = 0; i < 4; ++i) a.ev[i] = ev[i];
  }
  cudaError_t e = memo::attn_bwd(a, static_cast<cudaStream_t>(stream));
  if (ms3 && e == cudaSuccess) {
    cudaEventSynchronize(ev[3]);
    for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&ms3[i], ev[i], ev[i + 1]);
  }
  if (ms3)
    for (auto& x : ev) cudaEventDestroy(x);
  if (e != cudaSuccess)
    return set_error(MEMO_ERR_INTERNAL, std::string("memo_attn_bwd: ") + cudaGetErrorString(e));
  return MEMO_OK;
}

extern "C" int32_t memo_rmsnorm_bwd_partials(int32_t S) { return memo::rmsnorm_bwd_partials(S); }

extern "C" int memo_rmsnorm_bwd(const float* x, const void* a, const void* g, const float* dy,
                                const float* dres, float* dx, void* dx_bf16, float* partial, float* dg,
                                int32_t S, int32_t h, float eps, int32_t accumulate_dg, void* stream) {
  cudaError_t e = memo::rmsnorm_bwd(x, static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(g),
                                    dy, dres, dx, static_cast<__nv_bfloat16*>(dx_bf16), partial, dg, S, h, eps,
                                    accumulate_dg != 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(MEMO_ERR_INTERNAL, std::string("memo_rmsnorm_bwd: ") + cudaGetErrorString(e));
  return MEMO_OK;
}
