// gemm_tc.h — host interface of the tcgen05 GEMM (gemm_tc.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace memo {

enum GemmEpilogue {
  GEMM_EPI_BF16 = 0,      // c(bf16)[m, n] = acc
  GEMM_EPI_F32 = 1,       // c(f32)[m, n] = acc
  GEMM_EPI_F32_ACC = 2,   // c(f32)[m, n] += acc
  GEMM_EPI_RESID = 3,     // c(bf16) = acc (optional); out_f32 = resid + bf16(acc)
  GEMM_EPI_QKV_ROPE = 4,  // columns [0,h)->q (RoPE), [h,2h)->k (RoPE), [2h,3h)->v
};

// Kernel choice.  GEMM_VARIANT_AUTO is the product rule (gemm_tc.cu:launch);
// the others force one kernel for the bitwise-equivalence tests and A/B tools.
enum GemmVariant {
  GEMM_VARIANT_AUTO = 0,
  GEMM_VARIANT_SINGLE = 1,  // single-CTA 128x256 tiles, unclustered
  GEMM_VARIANT_MC2 = 2,     // single-CTA tiles in 2-CTA clusters, B multicast
  GEMM_VARIANT_MC4 = 3,     // 2x2 clusters, A and B multicast
  GEMM_VARIANT_PAIR = 4,    // CTA-pair 256x256 tiles (cta_group::2)
  GEMM_VARIANT_PAIR2 = 5,   // two CTA pairs per cluster sharing B by multicast (K-major B)
};

// Tile order: GEMM_RASTER_AUTO (serpentine bands) or the round-1 order (A/B tools).
enum GemmRaster { GEMM_RASTER_AUTO = 0, GEMM_RASTER_LEGACY = 1 };

// C = A . B^T with A logical [M, K], B logical [N, K].
//   a_mn_major = 0: A stored [M][lda], K contiguous;  1: stored [K][lda], M contiguous.
//   b_mn_major = 0: B stored [N][ldb], K contiguous;  1: stored [K][ldb], N contiguous.
struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const void* a = nullptr;
  long long lda = 0;
  int a_mn_major = 0;
  const void* b = nullptr;
  long long ldb = 0;
  int b_mn_major = 0;
  int epi = GEMM_EPI_BF16;
  void* c = nullptr;
  long long ldc = 0;
  float* out_f32 = nullptr;
  const float* resid = nullptr;
  long long ld_f32 = 0;
  __nv_bfloat16* q = nullptr;
  __nv_bfloat16* k = nullptr;
  __nv_bfloat16* v = nullptr;
  int hidden = 0;
  int head_dim = 0;
  const void* rope = nullptr;  // float2 [positions][head_dim/2] (cos, sin)
  long long pos0 = 0;          // absolute position of row 0
  int variant = GEMM_VARIANT_AUTO;
  int raster = GEMM_RASTER_AUTO;
};

cudaError_t gemm_tc(const GemmDesc& d, cudaStream_t stream);

}  // namespace memo
