// attention.h — causal FlashAttention on tcgen05 (attention.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace memo {

struct AttnFwdArgs {
  const __nv_bfloat16* q;  // [S, H*D]
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;        // [S, H*D]
  float* lse;              // [H, S], natural log
  int S, H, D;
  float softmax_scale;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // optional: recorded around the kernel
};
cudaError_t attn_fwd(const AttnFwdArgs& a, cudaStream_t stream);

struct AttnBwdArgs {
  const __nv_bfloat16* q;   // [S, H*D] (RoPE-rotated)
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const __nv_bfloat16* o;
  const float* lse;         // [H, S]
  const __nv_bfloat16* dout;  // [S, H*D]
  float* delta;             // workspace of attn_bwd_workspace_bytes(S, H, D)
  __nv_bfloat16* dq;        // rows of pitch ld_dqkv
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  long long ld_dqkv;
  const void* rope;         // float2 [pos][D/2]; NULL = no inverse rotation
  long long pos0;
  int S, H, D;
  float softmax_scale;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // optional: before prep, after prep, after dkdv, after dq
};
// delta/lse2 [2][H][S] f32, then (D == 128 with MEMO_ATTN_BWD=fused) the f32
// dQ accumulator [H][S][D] and the per-64-query-chunk ordering counters.
size_t attn_bwd_workspace_bytes(int S, int H, int D);
cudaError_t attn_bwd(const AttnBwdArgs& a, cudaStream_t stream);

}  // namespace memo
