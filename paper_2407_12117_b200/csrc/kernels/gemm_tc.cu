// gemm_tc.cu — persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[m, n] = sum_k A[m, k] * B[n, k]          (bf16 x bf16 -> f32 in TMEM)
//
// A and B may each be K-major (row-major with K contiguous) or MN-major
// (K rows, M/N contiguous), which covers the three GEMMs of a linear layer:
//   fwd    Y  = X  . W^T   A=X  K-major,  B=W  K-major
//   dgrad  dX = dY . W     A=dY K-major,  B=W  MN-major
//   wgrad  dW = dY^T . X   A=dY MN-major, B=X  MN-major
// Operands are staged by TMA (128-byte swizzle) into a 4-deep shared-memory
// ring; one thread issues tcgen05.mma (M=128, N=256, K=16) into a
// double-buffered TMEM accumulator so the epilogue of tile i overlaps the
// main loop of tile i+1.  Epilogues are fused: bf16/f32 store, f32
// accumulate, residual add, and the RoPE-rotating Q/K/V split.  The plain
// bf16/f32 epilogues turn their row-per-lane TMEM values around in a
// shared-memory slab so global stores leave as full 128-byte row segments.
// By default the tiles run in 2-CTA clusters (vertically adjacent M-tiles)
// that load each B tile once, half per CTA, by TMA multicast.
//
// The K loop order is the same for every output row, so recomputing a token
// suffix reproduces the full-pass rows bit for bit (MEMO's recompute must be
// indistinguishable from the swapped tensors; see swap.hpp:172-188).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "gemm_tc.h"
#include "sm100.cuh"
#include "tma_util.h"

namespace {
constexpr int MAX_DEVICES = 64;
}

namespace memo {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_TILE_BYTES = BM * BK * 2;  // 16 KiB
constexpr int B_TILE_BYTES = BN * BK * 2;  // 32 KiB
constexpr int STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
constexpr int NUM_THREADS = 192;  // warp0 TMA, warp1 MMA, warps2-5 epilogue
constexpr int TMEM_COLS = 2 * BN;
constexpr int GROUP_M = 16;  // rasterisation: 16 M-tiles share a B panel in L2
constexpr int SLAB_BYTES = 4 * 32 * 128;  // epilogue: one 32-row x 128 B slab per epilogue warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + SLAB_BYTES;

struct EpiParams {
  int kind;
  void* c;
  long long ldc;
  float* out_f32;
  const float* resid;
  long long ld_f32;
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* v;
  int hidden;
  int head_dim;
  const float2* rope;
  long long pos0;
  int staged;  // BF16/F32 stores through the shared-memory slab
  int serpentine;  // odd raster bands walk N backwards (the last band's B tiles are still in L2)
};

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* x) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u;
    u.x = dev::pack_bf16(x[8 * i + 0], x[8 * i + 1]);
    u.y = dev::pack_bf16(x[8 * i + 2], x[8 * i + 3]);
    u.z = dev::pack_bf16(x[8 * i + 4], x[8 * i + 5]);
    u.w = dev::pack_bf16(x[8 * i + 6], x[8 * i + 7]);
    d[i] = u;
  }
}

// One thread owns one row; `x` holds 32 consecutive accumulator columns.
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, int m, int n0, int N,
                                               float (&x)[32]) {
  if (n0 >= N) return;
  switch (ep.kind) {
    case GEMM_EPI_BF16: {
      store_bf16x32(reinterpret_cast<__nv_bfloat16*>(ep.c) + m * ep.ldc + n0, x);
      break;
    }
    case GEMM_EPI_F32: {
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.c) + m * ep.ldc + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
      break;
    }
    case GEMM_EPI_F32_ACC: {
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.c) + m * ep.ldc + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 o = d[i];
        o.x += x[4 * i];
        o.y += x[4 * i + 1];
        o.z += x[4 * i + 2];
        o.w += x[4 * i + 3];
        d[i] = o;
      }
      break;
    }
    case GEMM_EPI_RESID: {
      // The projection output is a bf16 tensor; the residual stream is f32.
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = dev::bf16_round(x[i]);
      if (ep.c) store_bf16x32(reinterpret_cast<__nv_bfloat16*>(ep.c) + m * ep.ldc + n0, x);
      const float4* r = reinterpret_cast<const float4*>(ep.resid + m * ep.ld_f32 + n0);
      float4* o = reinterpret_cast<float4*>(ep.out_f32 + m * ep.ld_f32 + n0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 a = r[i];
        a.x += x[4 * i];
        a.y += x[4 * i + 1];
        a.z += x[4 * i + 2];
        a.w += x[4 * i + 3];
        o[i] = a;
      }
      break;
    }
    case GEMM_EPI_QKV_ROPE: {
      const int which = n0 / ep.hidden;
      const int col = n0 - which * ep.hidden;
      __nv_bfloat16* base = which == 0 ? ep.q : (which == 1 ? ep.k : ep.v);
      if (which < 2) {
        // Interleaved-pair rotary embedding on absolute token position.
        const int j0 = col % ep.head_dim;  // multiple of 32
        const float2* cs = ep.rope + (ep.pos0 + m) * (ep.head_dim / 2) + j0 / 2;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const float2 t = cs[p];
          // Round to bf16 first: the rotation applies to the bf16 projection.
          const float a = dev::bf16_round(x[2 * p]);
          const float b = dev::bf16_round(x[2 * p + 1]);
          x[2 * p] = a * t.x - b * t.y;
          x[2 * p + 1] = a * t.y + b * t.x;
        }
      }
      store_bf16x32(base + static_cast<long long>(m) * ep.hidden + col, x);
      break;
    }
    default:
      break;
  }
}

// Staged row stores for the plain BF16 / F32 epilogues.  tcgen05.ld gives each
// lane one accumulator row, so a direct store puts 32 rows x 16 B into every
// warp store instruction, each half-filling a 32-byte L2 sector.  Here the
// warp's 32 rows x 128 B go through an XOR-swizzled 4 KiB shared-memory slab
// (conflict-free on both sides) and leave as 4 full 128-byte row segments per
// store instruction.  Same values, same bytes, same addresses.
__device__ __forceinline__ void slab_store(uint4* slab, const uint4 (&v)[8], uint32_t lane, uint8_t* row0,
                                           long long ld_bytes, int rows_valid, int bytes_valid) {
#pragma unroll
  for (int i = 0; i < 8; ++i) slab[lane * 8 + (i ^ (lane & 7))] = v[i];
  __syncwarp();
  const int u = lane & 7;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = it * 4 + static_cast<int>(lane >> 3);
    const uint4 w = slab[r * 8 + (u ^ (r & 7))];
    if (r < rows_valid && u * 16 < bytes_valid)
      *reinterpret_cast<uint4*>(row0 + r * ld_bytes + u * 16) = w;
  }
  __syncwarp();
}

// One epilogue warp's 32 rows x NCOLS columns of an accumulator buffer.
// t_row: TMEM address of the warp's lane quarter at the tile's column 0;
// m0: output row of lane 0; n_base: output column of the tile's column 0.
template <int NCOLS>
__device__ __forceinline__ void epilogue_rows(const EpiParams& ep, uint4* slab, uint32_t t_row, int m0,
                                              int M, int n_base, int N, uint32_t lane) {
  if (ep.staged && ep.kind == GEMM_EPI_BF16) {
#pragma unroll 1
    for (int c = 0; c < NCOLS / 64; ++c) {
      const int n0 = n_base + c * 64;
      if (n0 >= N) break;
      uint32_t r0[32], r1[32];
      dev::tmem_ld32(t_row + c * 64, r0);
      dev::tmem_ld32(t_row + c * 64 + 32, r1);
      dev::tmem_ld_wait_regs(r0, r1);
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = make_uint4(dev::pack_bf16(__uint_as_float(r0[8 * i + 0]), __uint_as_float(r0[8 * i + 1])),
                          dev::pack_bf16(__uint_as_float(r0[8 * i + 2]), __uint_as_float(r0[8 * i + 3])),
                          dev::pack_bf16(__uint_as_float(r0[8 * i + 4]), __uint_as_float(r0[8 * i + 5])),
                          dev::pack_bf16(__uint_as_float(r0[8 * i + 6]), __uint_as_float(r0[8 * i + 7])));
        v[4 + i] = make_uint4(dev::pack_bf16(__uint_as_float(r1[8 * i + 0]), __uint_as_float(r1[8 * i + 1])),
                              dev::pack_bf16(__uint_as_float(r1[8 * i + 2]), __uint_as_float(r1[8 * i + 3])),
                              dev::pack_bf16(__uint_as_float(r1[8 * i + 4]), __uint_as_float(r1[8 * i + 5])),
                              dev::pack_bf16(__uint_as_float(r1[8 * i + 6]), __uint_as_float(r1[8 * i + 7])));
      }
      slab_store(slab, v, lane,
                 reinterpret_cast<uint8_t*>(reinterpret_cast<__nv_bfloat16*>(ep.c) + m0 * ep.ldc + n0),
                 ep.ldc * 2, M - m0, (N - n0) * 2);
    }
    return;
  }
  if (ep.staged && ep.kind == GEMM_EPI_F32) {
#pragma unroll 1
    for (int c = 0; c < NCOLS / 32; ++c) {
      const int n0 = n_base + c * 32;
      if (n0 >= N) break;
      uint32_t r[32];
      dev::tmem_ld32(t_row + c * 32, r);
      dev::tmem_ld_wait_regs(r);
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
      slab_store(slab, v, lane, reinterpret_cast<uint8_t*>(reinterpret_cast<float*>(ep.c) + m0 * ep.ldc + n0),
                 ep.ldc * 4, M - m0, (N - n0) * 4);
    }
    return;
  }
  const int m = m0 + static_cast<int>(lane);
#pragma unroll 1
  for (int c = 0; c < NCOLS / 32; ++c) {
    uint32_t r[32];
    dev::tmem_ld32(t_row + c * 32, r);
    dev::tmem_ld_wait_regs(r);
    float x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(r[i]);
    if (m < M) epilogue_chunk(ep, m, n_base + c * 32, N, x);
  }
}

template <bool A_MN, bool B_MN, int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, int M, int N, int K,
                   EpiParams ep, int group_m) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint4* slab = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES + 256);

  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + BN - 1) / BN;
  // CL = 2: a 2-CTA cluster takes M-tiles 2u and 2u+1 of one N column; each
  // CTA loads its own A and half of the shared B tile, multicast to both.
  // CL = 4: a 2x2 cluster takes M-tiles 2u+rm and N-tiles 2v+rn; A is shared
  // by the two CTAs of one rm and B by the two of one rn, each loaded half by
  // each sharer.  The per-row K order is unchanged, so results equal the
  // unclustered kernel's bitwise.
  constexpr bool MC = CL > 1;
  const uint32_t rank = MC ? blockIdx.x % CL : 0;  // = %cluster_ctarank for 1-D clusters; uniform for ptxas
  const uint32_t rm = CL == 4 ? (rank & 1) : rank;  // M position in the cluster; also B's half
  const uint32_t rn = CL == 4 ? (rank >> 1) : 0;    // N position in the cluster; also A's half
  const int first = static_cast<int>(blockIdx.x) / CL;
  const int stride = static_cast<int>(gridDim.x) / CL;
  const int m_units = MC ? (m_tiles + 1) / 2 : m_tiles;
  const int n_units = CL == 4 ? (n_tiles + 1) / 2 : n_tiles;
  const int num_tiles = m_units * n_units;
  const int group_u = MC ? max(1, group_m / 2) : group_m;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_a);
    dev::tma_prefetch_desc(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&full_bar[s], 1);
      dev::mbar_init(&empty_bar[s], CL);
    }
    for (int b = 0; b < 2; ++b) {
      dev::mbar_init(&tfull_bar[b], 1);
      dev::mbar_init(&tempty_bar[b], 128);
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, TMEM_COLS);
  dev::tc_fence_before();
  __syncthreads();
  if constexpr (MC) dev::cluster_sync();  // the partner's barriers exist before any multicast
  dev::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) {
    const int group_size = group_u * n_units;
    const int g = t / group_size;
    const int first_m = g * group_u;
    const int gm = min(group_u, m_units - first_m);
    const int local = t - g * group_size;
    mb = first_m + local % gm;
    nb = local / gm;
    if (ep.serpentine && (g & 1)) nb = n_units - 1 - nb;
    if (MC) mb = 2 * mb + static_cast<int>(rm);
    if (CL == 4) nb = 2 * nb + static_cast<int>(rn);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = first; t < num_tiles; t += stride) {
        int mb, nb;
        tile_coords(t, mb, nb);
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_TILE_BYTES;
          dev::mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          if (CL == 4) {
            const uint16_t mask_a = static_cast<uint16_t>((1u << rm) | (1u << (rm + 2)));
            if (!A_MN)
              dev::tma_load_2d_mc(sa + rn * (A_TILE_BYTES / 2), &map_a, &full_bar[stage], kb * BK,
                                  mb * BM + static_cast<int>(rn) * (BM / 2), mask_a);
            else
              dev::tma_load_2d_mc(sa + rn * 8192, &map_a, &full_bar[stage], mb * BM + static_cast<int>(rn) * 64,
                                  kb * BK, mask_a);
          } else if (!A_MN) {
            dev::tma_load_2d(sa, &map_a, &full_bar[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              dev::tma_load_2d(sa + j * 8192, &map_a, &full_bar[stage], mb * BM + j * 64,
                               kb * BK);
          }
          if (MC) {
            const uint16_t mask_b = static_cast<uint16_t>(CL == 4 ? (3u << (2 * rn)) : 3u);
            if (!B_MN) {
              dev::tma_load_2d_mc(sb + rm * (B_TILE_BYTES / 2), &map_b, &full_bar[stage], kb * BK,
                                  nb * BN + static_cast<int>(rm) * (BN / 2), mask_b);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j) {
                const int jj = static_cast<int>(rm) * (BN / 128) + j;
                dev::tma_load_2d_mc(sb + jj * 8192, &map_b, &full_bar[stage], nb * BN + jj * 64, kb * BK, mask_b);
              }
            }
          } else if (!B_MN) {
            dev::tma_load_2d(sb, &map_b, &full_bar[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              dev::tma_load_2d(sb + j * 8192, &map_b, &full_bar[stage], nb * BN + j * 64,
                               kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // Producer tail: wait for every stage's last release.  With multicast the
      // releases are tcgen05.commit arrivals from the peer CTAs' MMA warps, and
      // the closing cluster_sync does not order those async arrivals: without
      // this wait a CTA could exit while one is still landing in its smem.
      for (int s = 0; s < STAGES; ++s) {
        dev::mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer: whole warp converged, elect.sync picks the issuing lane
      constexpr uint32_t idesc = dev::idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = first; t < num_tiles; t += stride, ++it) {
        const int buf = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        dev::mbar_wait_w(&tempty_bar[buf], acc_phase ^ 1);
        dev::tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait_w(&full_bar[stage], phase);
          dev::tc_fence_after();
          const uint32_t sa = dev::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_TILE_BYTES;
          const uint64_t ad0 = A_MN ? dev::umma_desc_sw128(sa, 8192, 1024) : dev::umma_desc_sw128(sa, 16, 1024);
          const uint64_t bd0 = B_MN ? dev::umma_desc_sw128(sb, 8192, 1024) : dev::umma_desc_sw128(sb, 16, 1024);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // only the start-address field moves with k (16-byte units)
            const uint64_t ad = ad0 + static_cast<uint64_t>((A_MN ? k * 2048 : k * 32) >> 4);
            const uint64_t bd = bd0 + static_cast<uint64_t>((B_MN ? k * 2048 : k * 32) >> 4);
            dev::mma_bf16_ss_w(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          if (MC)
            dev::mma_commit_mc_w(&empty_bar[stage], CL == 4 ? 0xF : 0x3);  // the sharers wrote this stage
          else
            dev::mma_commit_w(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        dev::mma_commit_w(&tfull_bar[buf]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 ; TMEM lane quarter = warp % 4
    const uint32_t q = warp & 3;
    int it = 0;
    for (int t = first; t < num_tiles; t += stride, ++it) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int buf = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      dev::mbar_wait(&tfull_bar[buf], acc_phase);
      dev::tc_fence_after();
      epilogue_rows<BN>(ep, slab + q * 256, tmem_base + ((q * 32) << 16) + buf * BN, mb * BM + q * 32, M,
                        nb * BN, N, lane);
      dev::tc_fence_before();
      dev::mbar_arrive(&tempty_bar[buf]);
    }
  }
  __syncthreads();
  if constexpr (MC) dev::cluster_sync();  // no multicast or remote arrive still targets this CTA
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA-pair GEMM
// Same contract and epilogues, on 256x256 output tiles computed by a CTA pair
// (cluster of 2, tcgen05.mma.cta_group::2, M=256 N=256 K=16).  Each CTA
// stages its own 128 rows of A and 128 of the 256 B rows, so per-CTA operand
// traffic (TMA writes + MMA reads of shared memory) per FLOP drops by a
// quarter, and the 32 KiB stage allows a 6-deep ring.  The leader CTA issues
// every MMA; its commits multicast to both CTAs' "stage empty" / "accumulator
// full" barriers.  Both CTAs' TMA loads complete on the leader's "stage full"
// barrier, and both epilogues release the leader's "accumulator empty".
constexpr int P_BM = 128;               // rows of A per CTA (pair tile M = 256)
constexpr int P_BN = 256;               // pair tile N; each CTA stages 128 B rows
constexpr int P_STAGES = 6;
constexpr int P_A_BYTES = P_BM * BK * 2;         // 16 KiB
constexpr int P_B_BYTES = (P_BN / 2) * BK * 2;   // 16 KiB
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + 1024 + 256 + SLAB_BYTES;
constexpr int P_GROUP_M = 16;  // raster band of pair tiles (8 measured slower)

// PC = 2: clusters of two CTA pairs on vertically adjacent pair tiles (same
// N columns).  Each stage's B half is shared across the pairs by multicast:
// CTA (pair p, half h) loads 64 of its 128 B rows and multicasts them to the
// same half of the other pair, so each SM reads 8 instead of 16 KiB of B per
// k-block from L2 (cuBLAS's 2x1-cluster 2-CTA layout).  A stage is then
// released by both pair leaders (empty barrier count 2).
template <bool A_MN, bool B_MN, int PC = 1>
__global__ void __cluster_dims__(2 * PC, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    int M, int N, int K, EpiParams ep) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + P_STAGES;
  uint64_t* tfull_bar = empty_bar + P_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint4* slab = reinterpret_cast<uint4*>(smem + P_STAGES * P_STAGE_BYTES + 256);

  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();
  const uint32_t crank = blockIdx.x % (2 * PC);  // = %cluster_ctarank for 1-D clusters; uniform for ptxas
  const uint32_t rank = crank & 1;             // rank inside the CTA pair
  const uint32_t pair = crank >> 1;            // pair inside the cluster (PC = 2)
  const uint32_t leader = crank & ~1u;         // the pair's MMA-issuing CTA
  const int cluster = blockIdx.x / (2 * PC), n_clusters = gridDim.x / (2 * PC);

  const int m_tiles = PC * ((M + 2 * PC * P_BM - 1) / (2 * PC * P_BM));  // pair tiles, whole clusters
  const int n_tiles = (N + P_BN - 1) / P_BN;
  const int num_tiles = (m_tiles / PC) * n_tiles;  // cluster units
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_a);
    dev::tma_prefetch_desc(&map_b);
    for (int s = 0; s < P_STAGES; ++s) {
      dev::mbar_init(&full_bar[s], 1);
      dev::mbar_init(&empty_bar[s], PC);  // one release per pair leader
    }
    for (int b = 0; b < 2; ++b) {
      dev::mbar_init(&tfull_bar[b], 1);
      dev::mbar_init(&tempty_bar[b], 2 * 128);  // epilogue threads of both CTAs
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc_cg2(tmem_slot, TMEM_COLS);
  dev::tc_fence_before();
  dev::cluster_sync();  // peer barriers initialised before any remote signal
  dev::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) {  // cluster unit t -> this pair's tile
    const int mu_tiles = m_tiles / PC;
    const int group_m = P_GROUP_M / PC;
    const int group_size = group_m * n_tiles;
    const int g = t / group_size;
    const int first_m = g * group_m;
    const int gm = min(group_m, mu_tiles - first_m);
    const int local = t - g * group_size;
    mb = (first_m + local % gm) * PC + static_cast<int>(pair);
    nb = local / gm;
    if (ep.serpentine && (g & 1)) nb = n_tiles - 1 - nb;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs): own A rows and own half of B
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < num_tiles; t += n_clusters) {
        int mb, nb;
        tile_coords(t, mb, nb);
        const int m0 = mb * 2 * P_BM + rank * P_BM;
        const int n0 = nb * P_BN + rank * (P_BN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * P_STAGE_BYTES;
          uint8_t* sb = sa + P_A_BYTES;
          const uint32_t fb = dev::mapa(dev::smem_u32(&full_bar[stage]), leader);  // pair leader's barrier
          if (rank == 0) dev::mbar_expect_tx(&full_bar[stage], 2 * P_STAGE_BYTES);
          if (!A_MN) {
            dev::tma_load_2d_cg2(sa, &map_a, fb, kb * BK, m0);
          } else {
#pragma unroll
            for (int j = 0; j < P_BM / 64; ++j) dev::tma_load_2d_cg2(sa + j * 8192, &map_a, fb, m0 + j * 64, kb * BK);
          }
          if (PC == 2 && !B_MN) {
            // 64 of this half's 128 B rows, multicast to the same half of both pairs
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
            dev::tma_load_2d_cg2_mc(sb + pair * (P_B_BYTES / 2), &map_b, fb, kb * BK,
                                    n0 + static_cast<int>(pair) * (P_BN / 4), mask);
          } else if (PC == 2) {
            // MN-major B: the half's two 64-column boxes, one per pair, multicast
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
            dev::tma_load_2d_cg2_mc(sb + pair * 8192, &map_b, fb, n0 + static_cast<int>(pair) * 64, kb * BK, mask);
          } else if (!B_MN) {
            dev::tma_load_2d_cg2(sb, &map_b, fb, kb * BK, n0);
          } else {
#pragma unroll
            for (int j = 0; j < P_BN / 2 / 64; ++j)
              dev::tma_load_2d_cg2(sb + j * 8192, &map_b, fb, n0 + j * 64, kb * BK);
          }
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // Producer tail: the leader's multicast commits release both CTAs'
      // stages; wait for the last of them before teardown (see gemm_tc_kernel).
      for (int s = 0; s < P_STAGES; ++s) {
        dev::mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == P_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA; whole warp converged, elect.sync issues)
      constexpr uint32_t idesc = dev::idesc_bf16_f32(2 * P_BM, P_BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cluster; t < num_tiles; t += n_clusters, ++it) {
        const int buf = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        dev::mbar_wait_w(&tempty_bar[buf], acc_phase ^ 1);
        dev::tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * P_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait_w(&full_bar[stage], phase);
          dev::tc_fence_after();
          const uint32_t sa = dev::smem_u32(smem + stage * P_STAGE_BYTES);
          const uint32_t sb = sa + P_A_BYTES;
          const uint64_t ad0 = A_MN ? dev::umma_desc_sw128(sa, 8192, 1024) : dev::umma_desc_sw128(sa, 16, 1024);
          const uint64_t bd0 = B_MN ? dev::umma_desc_sw128(sb, 8192, 1024) : dev::umma_desc_sw128(sb, 16, 1024);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ad0 + static_cast<uint64_t>((A_MN ? k * 2048 : k * 32) >> 4);
            const uint64_t bd = bd0 + static_cast<uint64_t>((B_MN ? k * 2048 : k * 32) >> 4);
            dev::mma2_bf16_ss_w(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          dev::mma2_commit_mc_w(&empty_bar[stage], PC == 2 ? 0xF : 0x3);  // every CTA the stage's B reached
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        dev::mma2_commit_mc_w(&tfull_bar[buf], static_cast<uint16_t>(0x3u << leader));
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 of both CTAs; TMEM lane quarter = warp % 4
    const uint32_t q = warp & 3;
    int it = 0;
    for (int t = cluster; t < num_tiles; t += n_clusters, ++it) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int buf = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      dev::mbar_wait(&tfull_bar[buf], acc_phase);
      dev::tc_fence_after();
      epilogue_rows<P_BN>(ep, slab + q * 256, tmem_base + ((q * 32) << 16) + buf * P_BN,
                          mb * 2 * P_BM + rank * P_BM + q * 32, M, nb * P_BN, N, lane);
      dev::tc_fence_before();
      dev::mbar_arrive_cluster(dev::mapa(dev::smem_u32(&tempty_bar[buf]), leader));
    }
  }
  dev::tc_fence_before();
  dev::cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc_cg2(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
template <bool A_MN, bool B_MN>
cudaError_t launch(const GemmDesc& d, cudaStream_t stream) {
  CUtensorMap ma, mb;
  bool ok;
  // CTA-pair 256x256 tiles (cta_group::2) where they measured faster: forward-
  // layout GEMMs (both operands K-major) with a short K and a wide N -- the QKV,
  // gate/up and classifier-logit projections (7 % / 6 % at 128K, interleaved
  // A/B, profiles/README.md); the single-CTA kernel everywhere else.  The choice
  // depends on (layout, N, K) only, never on M, so a recomputed row block runs
  // the same kernel as the forward and stays bitwise equal to it.
  // Single-CTA tiles run in 2-CTA clusters that share each B tile by TMA
  // multicast (half the B bytes per CTA; bitwise equal to unclustered tiles):
  // 3 % less GEMM time per cfg2 step.  d.variant (tests and A/B tools only)
  // forces one kernel: GEMM_VARIANT_SINGLE / _MC2 / _MC4 (2x2 clusters that
  // also share A) / _PAIR / _PAIR2 (two pairs per cluster, the pair default).
  bool pair;
  int cl;
  int pc = 1;  // CTA pairs per cluster (2: B shared across the pairs, K-major B only)
  switch (d.variant) {
    case GEMM_VARIANT_SINGLE: pair = false; cl = 1; break;
    case GEMM_VARIANT_MC2: pair = false; cl = 2; break;
    case GEMM_VARIANT_MC4: pair = false; cl = 4; break;
    case GEMM_VARIANT_PAIR: pair = true; cl = 1; break;
    case GEMM_VARIANT_PAIR2: pair = true; cl = 1; pc = 2; break;
    default:
      pair = !A_MN && !B_MN && d.K <= 4096 && d.N >= 8192;
      cl = pair ? 1 : 2;
      // the pair tiles run as two pairs per cluster sharing B (K-major B here):
      // +0.6 % per cfg2 step in three alternating whole-step runs, QKV +10 %
      // in the per-shape A/B (profiles/README.md)
      if (pair) pc = 2;
#ifdef MEMO_GEMM_ABLATIONS
      {  // whole-step A/B only (_lib_gemmexp): MEMO_GEMM_MN_VARIANT forces the MN-major layouts' kernel
        const char* ev = std::getenv("MEMO_GEMM_MN_VARIANT");
        const int v = ev ? std::atoi(ev) : 0;
        if ((A_MN || B_MN) && v > 0) {
          pair = v >= GEMM_VARIANT_PAIR;
          cl = v == GEMM_VARIANT_MC2 ? 2 : v == GEMM_VARIANT_MC4 ? 4 : 1;
          pc = v == GEMM_VARIANT_PAIR2 ? 2 : 1;
        }
        // MEMO_GEMM_KF_VARIANT: the same for the K-major shapes that take CTA pairs
        const char* ek = std::getenv("MEMO_GEMM_KF_VARIANT");
        const int vk = ek ? std::atoi(ek) : 0;
        if (pair && !A_MN && !B_MN && vk > 0) {
          pair = vk >= GEMM_VARIANT_PAIR;
          cl = vk == GEMM_VARIANT_MC2 ? 2 : vk == GEMM_VARIANT_MC4 ? 4 : 1;
          pc = vk == GEMM_VARIANT_PAIR2 ? 2 : 1;
        }
      }
#endif
  }
  const bool mc = cl > 1;
  if (!A_MN)
    ok = make_tma_2d_bf16(&ma, d.a, d.K, d.M, d.lda, BK, cl == 4 ? BM / 2 : BM);
  else
    ok = make_tma_2d_bf16(&ma, d.a, d.M, d.K, d.lda, 64, BK);
  if (!B_MN)
    ok = ok && make_tma_2d_bf16(&mb, d.b, d.K, d.N, d.ldb, BK, pc == 2 ? BN / 4 : (pair || mc) ? BN / 2 : BN);
  else
    ok = ok && make_tma_2d_bf16(&mb, d.b, d.N, d.K, d.ldb, 64, BK);
  if (!ok) return cudaErrorInvalidValue;
  EpiParams ep;
  ep.kind = d.epi;
  ep.c = d.c;
  ep.ldc = d.ldc;
  ep.out_f32 = d.out_f32;
  ep.resid = d.resid;
  ep.ld_f32 = d.ld_f32;
  ep.q = d.q;
  ep.k = d.k;
  ep.v = d.v;
  ep.hidden = d.hidden;
  ep.head_dim = d.head_dim;
  ep.rope = reinterpret_cast<const float2*>(d.rope);
  ep.pos0 = d.pos0;
  ep.staged = 1;  // swizzled shared-memory slab stores (the direct stores remain for the fused epilogues)
  // Serpentine raster: every other band of GROUP_M row tiles walks the N tiles
  // backwards, so a band starts on the B tiles the previous band read last
  // (still L2-resident).  Tile order only: results are bitwise unchanged.
  ep.serpentine = d.raster == GEMM_RASTER_LEGACY ? 0 : 1;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    cudaFuncSetAttribute(gemm_tc_kernel<A_MN, B_MN, 1>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(gemm_tc_kernel<A_MN, B_MN, 2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(gemm_tc_kernel<A_MN, B_MN, 4>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(gemm_tc2_kernel<A_MN, B_MN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
    cudaFuncSetAttribute(gemm_tc2_kernel<A_MN, B_MN, 2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
  });
  const int g_num_sms = num_sms();
  if (pair && pc == 2) {  // clusters of two CTA pairs sharing B
    const int units = ((d.M + 4 * P_BM - 1) / (4 * P_BM)) * ((d.N + P_BN - 1) / P_BN);
    // persistent clusters: no more than can be co-resident (4-CTA clusters need
    // not tile every GPC), else the surplus would run as a second wave
    static std::atomic<int> resident4[MAX_DEVICES];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>& slot = resident4[dev < MAX_DEVICES ? dev : 0];
    int res = slot.load(std::memory_order_relaxed);
    if (res == 0) {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(4 * (g_num_sms / 4));
      qc.blockDim = dim3(NUM_THREADS);
      qc.dynamicSmemBytes = P_SMEM_BYTES;
      if (cudaOccupancyMaxActiveClusters(&res, gemm_tc2_kernel<A_MN, B_MN, 2>, &qc) != cudaSuccess || res <= 0) {
        cudaGetLastError();
        res = g_num_sms / 4;
      }
      slot.store(res, std::memory_order_relaxed);
    }
    const int clusters = units < res ? units : res;
    gemm_tc2_kernel<A_MN, B_MN, 2><<<4 * clusters, NUM_THREADS, P_SMEM_BYTES, stream>>>(ma, mb, d.M, d.N, d.K, ep);
    return cudaGetLastError();
  }
  if (pair) {  // CTA pairs on 256x256 tiles
    const int tiles = ((d.M + 2 * P_BM - 1) / (2 * P_BM)) * ((d.N + P_BN - 1) / P_BN);
    const int clusters = tiles < g_num_sms / 2 ? tiles : g_num_sms / 2;
    gemm_tc2_kernel<A_MN, B_MN><<<2 * clusters, NUM_THREADS, P_SMEM_BYTES, stream>>>(ma, mb, d.M, d.N, d.K, ep);
    return cudaGetLastError();
  }
  const int tiles = ((d.M + BM - 1) / BM) * ((d.N + BN - 1) / BN);
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  const int group_m = GROUP_M;
  if (mc) {
    const int units = ((d.M + 2 * BM - 1) / (2 * BM)) * ((d.N + (cl == 4 ? 2 : 1) * BN - 1) / ((cl == 4 ? 2 : 1) * BN));
    auto kern = cl == 4 ? gemm_tc_kernel<A_MN, B_MN, 4> : gemm_tc_kernel<A_MN, B_MN, 2>;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // Persistent clusters: no more than can be co-resident (GPCs need not hold
    // a whole number of clusters), else the surplus would run as a second wave.
    // Cached per (device, cluster size); atomic because peer-local groups launch
    // GEMMs from several host threads (all of them compute the same value).
    static std::atomic<int> resident[MAX_DEVICES][5];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>& slot = resident[dev < MAX_DEVICES ? dev : 0][cl];
    int res = slot.load(std::memory_order_relaxed);
    if (res == 0) {
      cfg.gridDim = dim3(cl * (g_num_sms / cl));
      if (cudaOccupancyMaxActiveClusters(&res, kern, &cfg) != cudaSuccess || res <= 0) {
        cudaGetLastError();
        res = g_num_sms / cl;
      }
      slot.store(res, std::memory_order_relaxed);
    }
    const int clusters = units < res ? units : res;
    cfg.gridDim = dim3(cl * clusters);
    return cudaLaunchKernelEx(&cfg, kern, ma, mb, d.M, d.N, d.K, ep, group_m);
  }
  gemm_tc_kernel<A_MN, B_MN, 1><<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ma, mb, d.M, d.N,
                                                                              d.K, ep, group_m);
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_tc(const GemmDesc& d, cudaStream_t stream) {
  if (d.M <= 0 || d.N <= 0 || d.K <= 0) return cudaSuccess;
  if (d.N % 32 != 0 || d.K % 8 != 0) return cudaErrorInvalidValue;
  if (d.a_mn_major) {
    if (d.b_mn_major) return launch<true, true>(d, stream);
    return launch<true, false>(d, stream);
  }
  if (d.b_mn_major) return launch<false, true>(d, stream);
  return launch<false, false>(d, stream);
}

}  // namespace memo
