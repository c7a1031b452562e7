// attention.cu — causal FlashAttention forward/backward on tcgen05 (sm_100a).
//
// Layout: Q, K, V, O are token-major [S, H*D] bf16 (head hh occupies columns
// [hh*D, hh*D+D)); LSE is [H, S] f32 (natural log).  Tiles are 128 tokens.
// Every kernel is warp-specialised: warp 0 issues TMA, one thread of warp 1
// issues tcgen05.mma, warps 4-7 (one thread per TMEM lane / tile row) do the
// elementwise math between MMAs.  Operands that stay fixed for a CTA's whole
// loop (Q in the forward and in dQ, dO in dQ) are written once into TMEM and
// used as the A operand of .kind::f16 MMAs, which halves shared-memory operand
// traffic (the SS form of M128xN128 sits right at 128 B/clk).
//
// Forward (CTA per (query tile, head)):  S_j = Q K_j^T into a double-buffered
//   TMEM S; the softmax warps overwrite S_j with P_j (bf16) which feeds
//   O += P_j V_j as the TMEM A operand.  S_{j+1} is issued before P_j V_j so QK^T
//   of the next tile overlaps the softmax of this one (tcgen05 ops of a thread
//   execute in order, which makes reusing S's columns for P safe).  O is only
//   rescaled when a row max grows by > 2^8, and a quarter of the exponentials
//   run as a cubic on the FMA pipe to take load off MUFU.
// Backward is deterministic (no atomics), so swap+recompute and no-swap
// gradients are bit-identical.  Both kernels walk their partner tiles in
// 64-row halves with double-buffered TMEM so the P/dS math of half g overlaps
// the MMAs of half g+1:
//   attn_bwd_dkdv  CTA per (key tile, head):   S^T = K Q^T, dP^T = V dO^T,
//                  dV += P^T dO, dK += dS^T Q   (P^T, dS^T from TMEM)
//   attn_bwd_dq    CTA per (query tile, head): S = Q K^T, dP = dO V^T,
//                  dQ += dS K                    (Q, dO, dS from TMEM)
// RoPE's inverse rotation and the softmax scale are fused into the dQ/dK
// epilogues.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>

#include "attention.h"
#include "sm100.cuh"
#include "tma_util.h"

namespace memo {
namespace {

constexpr int TILE = 128;
constexpr int CHUNK_BYTES = TILE * 64 * 2;  // one [128 rows][64 cols] bf16 TMA box = 16 KiB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units


// Descriptors are built once per tile base; the k-steps only move the start
// address (bits [0,14) in 16-byte units), so each MMA issue is one 64-bit add
// of a compile-time constant.  (The single issuing thread is otherwise the
// bottleneck for the N=64 halves, whose MMAs take only 32 cycles.)
__device__ __forceinline__ uint64_t kmajor_base(uint32_t base) {
  return dev::umma_desc_sw128(base, 16, 1024);
}
__device__ __forceinline__ uint64_t mnmajor_base(uint32_t base) {
  return dev::umma_desc_sw128(base, CHUNK_BYTES, 1024);
}
// K-major tile split in 64-col chunks of 16 KiB; k-step of 16 elements.
__device__ __forceinline__ uint64_t kmajor_step(uint64_t d, int kk) {
  return d + static_cast<uint64_t>(((kk >> 2) * CHUNK_BYTES + (kk & 3) * 32) >> 4);
}
// Descriptor helpers for operand tiles whose 64-col chunks are CH bytes apart.
template <int CH>
__device__ __forceinline__ uint64_t kmajor_step_c(uint64_t d, int kk) {
  return d + static_cast<uint64_t>(((kk >> 2) * CH + (kk & 3) * 32) >> 4);
}
template <int CH>
__device__ __forceinline__ uint64_t mnmajor_base_c(uint32_t base) {
  return dev::umma_desc_sw128(base, CH, 1024);
}
// MN-major tile: 128 K-rows of 128 B per 64-wide MN chunk; k-step of 16 rows.
__device__ __forceinline__ uint64_t mnmajor_step(uint64_t d, int kk) {
  return d + static_cast<uint64_t>((kk * 2048) >> 4);
}


// 2^x for x <= 0 without the MUFU: round-to-nearest via the 1.5*2^23 magic
// add (no FRND/F2I, which would occupy the same XU pipe as MUFU.EX2), a
// degree-3 minimax polynomial for 2^f on [-0.5, 0.5] (max rel. error 7.6e-5;
// bf16 P needs 3.9e-3), and the exponent added in the integer domain.
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -126.f);  // round(x) >= -126 keeps the exponent field of the result >= 0
  const float j = x + 12582912.f;  // low mantissa bits = round(x)
  const float f = x - (j - 12582912.f);
  float p = fmaf(f, 0.05517027f, 0.24260795f);
  p = fmaf(p, f, 0.6932609f);
  p = fmaf(p, f, 0.9999283f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

// Each softmax/compute thread writes its own row (D bf16 from global) into
// TMEM columns [t_col, t_col + D/2) of its lane: the A-operand layout.
template <int D>
__device__ __forceinline__ void row_to_tmem(const __nv_bfloat16* src, uint32_t taddr) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int c = 0; c < D / 64; ++c) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = s4[c * 8 + i];
      r[4 * i + 0] = v.x;
      r[4 * i + 1] = v.y;
      r[4 * i + 2] = v.z;
      r[4 * i + 3] = v.w;
    }
    dev::tmem_st32(taddr + c * 32, r);
  }
}

constexpr int FWD_STAGES = 3;

template <int D, bool QT>
struct FwdSmem {
  static constexpr int NC = D / 64;  // 64-col chunks per tile
  static constexpr int TILE_BYTES = NC * CHUNK_BYTES;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = QT ? 0 : TILE_BYTES;
  static constexpr int V_OFF = K_OFF + FWD_STAGES * TILE_BYTES;
  static constexpr int BAR_OFF = V_OFF + FWD_STAGES * TILE_BYTES;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

// QT: Q lives in TMEM (A operand of S = QK^T) instead of shared memory.
// EMU: a quarter of the softmax exponentials run as a cubic on the FMA pipe.
template <int D, bool QT, bool EMU>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ q, const __grid_constant__ CUtensorMap map_q,
                    const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ out,
                    float* __restrict__ lse, int S, int H, float scale_log2) {
  using L = FwdSmem<D, QT>;
  constexpr int NC = L::NC;
  constexpr int NS = FWD_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_ready = bars + 0;
  uint64_t* k_full = bars + 1;        // [NS]
  uint64_t* k_empty = k_full + NS;    // [NS]
  uint64_t* v_full = k_empty + NS;    // [NS]
  uint64_t* v_empty = v_full + NS;    // [NS]
  uint64_t* s_full = v_empty + NS;    // [2]
  uint64_t* p_full = s_full + 2;      // [2]
  uint64_t* o_done = p_full + 2;
  uint64_t* o_final = o_done + 1;  // committed once, after the last PV (unambiguous epilogue wait)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 1);

  const int n_tiles = S / TILE;
  const int qt = n_tiles - 1 - static_cast<int>(blockIdx.x);  // heavy tiles first
  const int hh = blockIdx.y;
  const int n_kv = qt + 1;
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::tma_prefetch_desc(&map_q);
    dev::mbar_init(q_ready, QT ? 128 : 1);
    for (int s = 0; s < NS; ++s) {
      dev::mbar_init(&k_full[s], 1);
      dev::mbar_init(&k_empty[s], 1);
      dev::mbar_init(&v_full[s], 1);
      dev::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      dev::mbar_init(&s_full[s], 1);
      dev::mbar_init(&p_full[s], 128);
    }
    dev::mbar_init(o_done, 1);
    dev::mbar_init(o_final, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;
  const uint32_t t_q = tmem + 256 + D;

  if (warp == 0) {
    if (lane == 0) {
      if (!QT) {
        dev::mbar_expect_tx(q_ready, L::TILE_BYTES);
        for (int c = 0; c < NC; ++c)
          dev::tma_load_2d(smem + L::Q_OFF + c * CHUNK_BYTES, &map_q, q_ready, hh * D + c * 64, qt * TILE);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NS;
        const uint32_t ph = (j / NS) & 1;
        uint8_t* sk = smem + L::K_OFF + st * L::TILE_BYTES;
        uint8_t* sv = smem + L::V_OFF + st * L::TILE_BYTES;
        dev::mbar_wait(&k_empty[st], ph ^ 1);
        dev::mbar_expect_tx(&k_full[st], L::TILE_BYTES);
        for (int c = 0; c < NC; ++c)
          dev::tma_load_2d(sk + c * CHUNK_BYTES, &map_k, &k_full[st], hh * D + c * 64, j * TILE);
        dev::mbar_wait(&v_empty[st], ph ^ 1);
        dev::mbar_expect_tx(&v_full[st], L::TILE_BYTES);
        for (int c = 0; c < NC; ++c)
          dev::tma_load_2d(sv + c * CHUNK_BYTES, &map_v, &v_full[st], hh * D + c * 64, j * TILE);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_o = dev::idesc_bf16_f32(128, D, false, true);
      dev::mbar_wait_w(q_ready, 0);
      auto issue_s = [&](int j) {
        const int st = j % NS;
        dev::mbar_wait_w(&k_full[st], (j / NS) & 1);
        dev::tc_fence_after();
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + L::K_OFF + st * L::TILE_BYTES));
        const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::Q_OFF));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          if (QT)
            dev::mma_bf16_ts_w(t_s[j & 1], t_q + kk * 8, kmajor_step(kd, kk), idesc_s, kk > 0);
          else
            dev::mma_bf16_ss_w(t_s[j & 1], kmajor_step(qd, kk), kmajor_step(kd, kk), idesc_s, kk > 0);
        }
        dev::mma_commit_w(&s_full[j & 1]);
        dev::mma_commit_w(&k_empty[st]);
      };
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int st = j % NS;
        dev::mbar_wait_w(&p_full[j & 1], (j >> 1) & 1);
        dev::mbar_wait_w(&v_full[st], (j / NS) & 1);
        dev::tc_fence_after();
        const uint64_t vd = mnmajor_base(dev::smem_u32(smem + L::V_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          dev::mma_bf16_ts_w(t_o, t_s[j & 1] + kk * 8, mnmajor_step(vd, kk), idesc_o, (j | kk) != 0);
        // o_done phase j = PV(j) complete, consumed in order by the softmax
        // warps at tile j+1; the last PV commits o_final for the epilogue.
        dev::mma_commit_w(j + 1 < n_kv ? o_done : o_final);
        dev::mma_commit_w(&v_empty[st]);
      }
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int row = q4 * 32 + lane;  // TMEM lane == query row in tile
    const int qidx = qt * TILE + row;
    const uint32_t lane_off = (q4 * 32) << 16;
    if (QT) {
      row_to_tmem<D>(q + static_cast<long long>(qidx) * H * D + hh * D, t_q + lane_off);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(q_ready);
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      dev::mbar_wait(&s_full[st], (j >> 1) & 1);
      dev::tc_fence_after();
      float s[128];
      {
        uint32_t r[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) dev::tmem_ld32(t_s[st] + lane_off + c * 32, r[c]);
        dev::tmem_ld_wait_regs(r[0], r[1], r[2], r[3]);  // one wait for all four loads
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[c][i]);  // raw logits
      }
      if (j == qt) {  // diagonal tile: causal mask
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i > row) s[i] = -INFINITY;
      }
      // One warp per SMSP: reduce with 8 independent chains, not one
      // 127-deep dependent FMNMX chain.
      float mx8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx8[k] = s[k];
#pragma unroll
      for (int i = 8; i < 128; i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(mx8[k], s[i + k]);
#pragma unroll
      for (int k = 4; k > 0; k >>= 1)
#pragma unroll
        for (int q2 = 0; q2 < k; ++q2) mx8[q2] = fmaxf(mx8[q2], mx8[q2 + k]);
      const float mx = mx8[0] * scale_log2;  // scale > 0 commutes with max
      const float cand = fmaxf(m, mx);
      const bool need = j == 0 || cand > m + kRescaleThreshold;
      const bool any = __any_sync(0xffffffffu, need);
      float factor = 1.f;
      float m_new = m;
      if (any) {
        m_new = cand;
        factor = j == 0 ? 0.f : dev::ex2(m - m_new);
      }
      float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t p[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        float a, b;
        if (EMU && (i & 3) == 3) {  // a quarter of the exponentials on the FMA pipe
          a = exp2_fma(fmaf(s[2 * i], scale_log2, -m_new));
          b = exp2_fma(fmaf(s[2 * i + 1], scale_log2, -m_new));
        } else {
          a = dev::ex2(fmaf(s[2 * i], scale_log2, -m_new));
          b = dev::ex2(fmaf(s[2 * i + 1], scale_log2, -m_new));
        }
        sum8[i & 7] += a + b;
        p[i] = dev::pack_bf16(a, b);
      }
#pragma unroll
      for (int k = 4; k > 0; k >>= 1)
#pragma unroll
        for (int q2 = 0; q2 < k; ++q2) sum8[q2] += sum8[q2 + k];
      l = l * factor + sum8[0];
      m = m_new;
      {
        uint32_t (&p0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&p[0]);
        uint32_t (&p1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&p[32]);
        dev::tmem_st32(t_s[st] + lane_off, p0);
        dev::tmem_st32(t_s[st] + lane_off + 32, p1);
      }
      // Every phase of o_done (PV(j-1) complete) is consumed, in order, so the
      // parity wait is never ambiguous and no commit goes unwaited.
      if (j > 0) dev::mbar_wait(o_done, (j - 1) & 1);
      if (any && j > 0) {
        // O must hold P(j-1)V(j-1) before it is rescaled.
        dev::tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          dev::tmem_ld32(t_o + lane_off + c * 32, r);
          dev::tmem_ld_wait_regs(r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * factor);
          dev::tmem_st32(t_o + lane_off + c * 32, r);
        }
      }
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_full[st]);
    }
    // epilogue
    dev::mbar_wait(o_final, 0);
    dev::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + static_cast<long long>(qidx) * H * D + hh * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      dev::tmem_ld32(t_o + lane_off + c * 32, r);
      dev::tmem_ld_wait_regs(r);
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        u.x = dev::pack_bf16(__uint_as_float(r[8 * i + 0]) * inv, __uint_as_float(r[8 * i + 1]) * inv);
        u.y = dev::pack_bf16(__uint_as_float(r[8 * i + 2]) * inv, __uint_as_float(r[8 * i + 3]) * inv);
        u.z = dev::pack_bf16(__uint_as_float(r[8 * i + 4]) * inv, __uint_as_float(r[8 * i + 5]) * inv);
        u.w = dev::pack_bf16(__uint_as_float(r[8 * i + 6]) * inv, __uint_as_float(r[8 * i + 7]) * inv);
        dst[i] = u;
      }
    }
    lse[static_cast<long long>(hh) * S + qidx] = (m + log2f(l)) * kLn2;
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}


// ------------------------------------------------------------------ forward, split rows
// Same pipeline as attn_fwd_kernel (Q in TMEM, double-buffered S, P over S),
// but every query row is shared by two softmax warps on the same SMSP (warps
// w and w+4 own columns [0,64) and [64,128) of the key tile).  The single
// softmax warp per SMSP was the critical path (~1.8k clk per tile against
// 1024 clk of MMA); two warps interleave their dependency chains.  The row
// max is exchanged through shared memory behind a 64-thread named barrier,
// each warp keeps its own partial row sum (combined once in the epilogue),
// FFMA2/FADD2 process column pairs, and a quarter of the exponentials run on
// the FMA pipe (exp2_fma) to keep MUFU below the MMA time.
#ifdef MEMO_ATTN_ABLATIONS  // split-row forward layout (ablation build only)
struct Fwd2wSmem {
  static constexpr int TILE_BYTES = 2 * CHUNK_BYTES;  // D = 128
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + FWD_STAGES * TILE_BYTES;
  static constexpr int X_OFF = V_OFF + FWD_STAGES * TILE_BYTES;  // [2 parity][2 half][128] f32
  static constexpr int BAR_OFF = X_OFF + 2 * 2 * 128 * 4;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};
#endif  // MEMO_ATTN_ABLATIONS


__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, float b, float c) {  // a * b + c (b, c broadcast)
  uint64_t r;
  const uint64_t bb = f2_pack(b, b), cc = f2_pack(c, c);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(bb), "l"(cc));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ffma2_v(uint64_t a, float b, uint64_t c) {  // a * b + c (b broadcast)
  uint64_t r;
  const uint64_t bb = f2_pack(b, b);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(bb), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {  // a * b + c
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// max(a, b, c) in one FMNMX3 (sm_100)
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// exp2_fma on a column pair with the paired FP32 instructions: bitwise the
// scalar exp2_fma of each half (same operations, same rounding), in ~10
// instructions per pair instead of ~18.
__device__ __forceinline__ uint64_t exp2_fma2(uint64_t x2) {
  const uint64_t x = f2_pack(fmaxf(f2_lo(x2), -126.f), fmaxf(f2_hi(x2), -126.f));
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);
  const uint64_t j = fadd2(x, magic);                                        // low bits = round(x)
  const uint64_t t = fadd2(j, f2_pack(-12582912.f, -12582912.f));            // round(x) as float
  const uint64_t f = fma2(t, f2_pack(-1.f, -1.f), x);                         // x - round(x), exact sub
  uint64_t p = fma2(f, f2_pack(0.05517027f, 0.05517027f), f2_pack(0.24260795f, 0.24260795f));
  p = fma2(p, f, f2_pack(0.6932609f, 0.6932609f));
  p = fma2(p, f, f2_pack(0.9999283f, 0.9999283f));
  const uint32_t lo = static_cast<uint32_t>(p) + (static_cast<uint32_t>(j) << 23);
  const uint32_t hi = static_cast<uint32_t>(p >> 32) + (static_cast<uint32_t>(j >> 32) << 23);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}
[[maybe_unused]] __device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifdef MEMO_ATTN_ABLATIONS  // split-row forward (ablation build only)
template <int EMU_EVERY>  // 0: all exps on MUFU; n: every n-th column pair on the FMA pipe
__global__ void __launch_bounds__(384, 1)
    attn_fwd_2w_kernel(const __nv_bfloat16* __restrict__ q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, int S, int H, float scale_log2) {
  constexpr int D = 128;
  using L = Fwd2wSmem;
  constexpr int NC = 2;
  constexpr int NS = FWD_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_ready = bars + 0;
  uint64_t* k_full = bars + 1;        // [NS]
  uint64_t* k_empty = k_full + NS;    // [NS]
  uint64_t* v_full = k_empty + NS;    // [NS]
  uint64_t* v_empty = v_full + NS;    // [NS]
  uint64_t* s_full = v_empty + NS;    // [2]
  uint64_t* p_full = s_full + 2;      // [2]
  uint64_t* o_done = p_full + 2;
  uint64_t* o_final = o_done + 1;  // committed once, after the last PV (unambiguous epilogue wait)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + 1);
  const uint32_t xchg_s = dev::smem_u32(smem + L::X_OFF);

  const int n_tiles = S / TILE;
  const int qt = n_tiles - 1 - static_cast<int>(blockIdx.x);  // heavy tiles first
  const int hh = blockIdx.y;
  const int n_kv = qt + 1;
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::mbar_init(q_ready, 256);
    for (int s = 0; s < NS; ++s) {
      dev::mbar_init(&k_full[s], 1);
      dev::mbar_init(&k_empty[s], 1);
      dev::mbar_init(&v_full[s], 1);
      dev::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      dev::mbar_init(&s_full[s], 1);
      dev::mbar_init(&p_full[s], 256);
    }
    dev::mbar_init(o_done, 1);
    dev::mbar_init(o_final, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto t_s = [&](int b) { return tmem + 128 * b; };  // S buffers (no indexed array: it lands in local memory)
  const uint32_t t_o = tmem + 256;
  const uint32_t t_q = tmem + 256 + D;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NS;
        const uint32_t ph = (j / NS) & 1;
        uint8_t* sk = smem + L::K_OFF + st * L::TILE_BYTES;
        uint8_t* sv = smem + L::V_OFF + st * L::TILE_BYTES;
        dev::mbar_wait(&k_empty[st], ph ^ 1);
        dev::mbar_expect_tx(&k_full[st], L::TILE_BYTES);
        for (int c = 0; c < NC; ++c)
          dev::tma_load_2d(sk + c * CHUNK_BYTES, &map_k, &k_full[st], hh * D + c * 64, j * TILE);
        dev::mbar_wait(&v_empty[st], ph ^ 1);
        dev::mbar_expect_tx(&v_full[st], L::TILE_BYTES);
        for (int c = 0; c < NC; ++c)
          dev::tma_load_2d(sv + c * CHUNK_BYTES, &map_v, &v_full[st], hh * D + c * 64, j * TILE);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_o = dev::idesc_bf16_f32(128, D, false, true);
      dev::mbar_wait_w(q_ready, 0);
      dev::tc_fence_after();
      auto issue_s = [&](int j) {
        const int st = j % NS;
        dev::mbar_wait_w(&k_full[st], (j / NS) & 1);
        dev::tc_fence_after();
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + L::K_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ts_w(t_s(j & 1), t_q + kk * 8, kmajor_step(kd, kk), idesc_s, kk > 0);
        dev::mma_commit_w(&s_full[j & 1]);
        dev::mma_commit_w(&k_empty[st]);
      };
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int st = j % NS;
        dev::mbar_wait_w(&p_full[j & 1], (j >> 1) & 1);
        dev::mbar_wait_w(&v_full[st], (j / NS) & 1);
        dev::tc_fence_after();
        const uint64_t vd = mnmajor_base(dev::smem_u32(smem + L::V_OFF + st * L::TILE_BYTES));
        // P of keys [0,64) sits in S cols [0,32), keys [64,128) in cols [64,96)
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          dev::mma_bf16_ts_w(t_o, t_s(j & 1) + 8 * kk + 32 * (kk >> 2), mnmajor_step(vd, kk), idesc_o,
                             (j | kk) != 0);
        // o_done phase j = PV(j) complete, consumed in order by the softmax
        // warps at tile j+1; the last PV commits o_final for the epilogue.
        dev::mma_commit_w(j + 1 < n_kv ? o_done : o_final);
        dev::mma_commit_w(&v_empty[st]);
      }
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int hf = (warp - 4) >> 2;  // column half of the key tile (and of D for O)
    const int row = q4 * 32 + lane;
    const int qidx = qt * TILE + row;
    const uint32_t lane_off = (q4 * 32) << 16;
    const int bar_id = 1 + q4;       // warps w and w+4 (same rows)
    {  // Q row elements [64hf, 64hf+64) -> TMEM cols [32hf, 32hf+32)
      const uint4* s4 = reinterpret_cast<const uint4*>(q + static_cast<long long>(qidx) * H * D + hh * D + 64 * hf);
      uint32_t r[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = s4[i];
        r[4 * i + 0] = v.x;
        r[4 * i + 1] = v.y;
        r[4 * i + 2] = v.z;
        r[4 * i + 3] = v.w;
      }
      dev::tmem_st32(t_q + lane_off + 32 * hf, r);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(q_ready);
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      dev::mbar_wait(&s_full[st], (j >> 1) & 1);
      dev::tc_fence_after();
      uint32_t r[2][32];
      dev::tmem_ld32(t_s(st) + lane_off + 64 * hf, r[0]);
      dev::tmem_ld32(t_s(st) + lane_off + 64 * hf + 32, r[1]);
      dev::tmem_ld_wait_regs(r[0], r[1]);
      bool any = false;
      float factor = 1.f;
      uint32_t p[32];
      // The causal mask only exists on the diagonal tile; a separate
      // instantiation keeps the compiler from if-converting it into a
      // compare+select per element on every tile.
      auto tile = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        if (DIAG) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (64 * hf + i > row) r[i >> 5][i & 31] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = __uint_as_float(r[0][k2]);
#pragma unroll
        for (int i = 8; i < 64; i += 8)
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmaxf(mx8[k2], __uint_as_float(r[i >> 5][(i & 31) + k2]));
#pragma unroll
        for (int k2 = 4; k2 > 0; k2 >>= 1)
#pragma unroll
          for (int q2 = 0; q2 < k2; ++q2) mx8[q2] = fmaxf(mx8[q2], mx8[q2 + k2]);
        // row max across the two halves (explicit ld/st.shared: a generic
        // pointer here compiles to LD.E/ST.E on the global path)
        const uint32_t xp = xchg_s + (j & 1) * 1024;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(xp + (hf * 128 + row) * 4), "f"(mx8[0]) : "memory");
        named_bar(bar_id, 64);
        float other;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xp + ((hf ^ 1) * 128 + row) * 4) : "memory");
        const float mx = fmaxf(mx8[0], other) * scale_log2;
        const float cand = fmaxf(m, mx);
        const bool need = j == 0 || cand > m + kRescaleThreshold;
        any = __any_sync(0xffffffffu, need);  // same rows, same vote in both warps
        float m_new = m;
        if (any) {
          m_new = cand;
          factor = j == 0 ? 0.f : dev::ex2(m - m_new);
        }
        uint64_t sum4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint64_t x2 = ffma2(f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                            __uint_as_float(r[i >> 4][(2 * i + 1) & 31])),
                                    scale_log2, -m_new);
          float a, b;
          if (EMU_EVERY > 0 && (i % (EMU_EVERY > 0 ? EMU_EVERY : 1)) == EMU_EVERY - 1) {
            a = exp2_fma(f2_lo(x2));
            b = exp2_fma(f2_hi(x2));
          } else {
            a = dev::ex2(f2_lo(x2));
            b = dev::ex2(f2_hi(x2));
          }
          sum4[i & 3] = fadd2(sum4[i & 3], f2_pack(a, b));
          p[i] = dev::pack_bf16(a, b);
        }
        const uint64_t s01 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l = l * factor + (f2_lo(s01) + f2_hi(s01));
        m = m_new;
      };
      if (j == qt)
        tile(std::true_type{});
      else
        tile(std::false_type{});
      dev::tmem_st32(t_s(st) + lane_off + 64 * hf, p);  // inside this warp's own columns
      if (j > 0) dev::mbar_wait(o_done, (j - 1) & 1);  // every phase consumed in order
      if (any && j > 0) {
        // O must hold P(j-1)V(j-1) before it is rescaled; this warp owns D cols [64hf, 64hf+64)
        dev::tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t o[32];
          dev::tmem_ld32(t_o + lane_off + 64 * hf + 32 * c, o);
          dev::tmem_ld_wait_regs(o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
          dev::tmem_st32(t_o + lane_off + 64 * hf + 32 * c, o);
        }
      }
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_full[st]);
    }
    // epilogue: combine the two partial row sums, write O columns [64hf, 64hf+64) and the LSE
    const uint32_t xp = xchg_s + (n_kv & 1) * 1024;
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(xp + (hf * 128 + row) * 4), "f"(l) : "memory");
    named_bar(bar_id, 64);
    float l_other;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(l_other) : "r"(xp + ((hf ^ 1) * 128 + row) * 4) : "memory");
    const float lt = l + l_other;
    dev::mbar_wait(o_final, 0);
    dev::tc_fence_after();
    const float inv = 1.f / lt;
    __nv_bfloat16* orow = out + static_cast<long long>(qidx) * H * D + hh * D + 64 * hf;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      dev::tmem_ld32(t_o + lane_off + 64 * hf + 32 * c, o);
      dev::tmem_ld_wait_regs(o);
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        u.x = dev::pack_bf16(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv);
        u.y = dev::pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv);
        u.z = dev::pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv);
        u.w = dev::pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv);
        dst[i] = u;
      }
    }
    if (hf == 0) lse[static_cast<long long>(hh) * S + qidx] = (m + log2f(lt)) * kLn2;
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}
#endif  // MEMO_ATTN_ABLATIONS

// ------------------------------------------------------------------ forward, ping-pong
// Two adjacent query tiles (A = 2p, B = 2p+1) of one head per CTA, each with
// its own softmax warpgroup (one thread per row, all 128 columns in
// registers).  The tensor pipe alternates between the groups:
//   PV_A(j-1) S_A(j) PV_B(j-1) S_B(j) ...
// so while group A turns S_A(j) into P_A(j) the pipe runs PV_B(j-1) and S_B(j)
// (1024 cycles of work), and vice versa.  K and V tiles are shared by both
// groups (half the L2->SMEM traffic per FLOP of the one-tile kernels).
// TMEM: S_A | S_B | O_A | O_B (P overwrites its S), so Q stays in shared
// memory (SS-mode S).  setmaxnreg moves registers from the TMA/MMA warpgroup
// (56) to the softmax warpgroups (224) so a row's 128 logits stay resident.
struct FwdPpSmem {
  static constexpr int TILE_BYTES = 2 * CHUNK_BYTES;  // D = 128
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = TILE_BYTES;
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;  // 2-stage K and V rings
  static constexpr int BAR_OFF = V_OFF + 2 * TILE_BYTES;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

// Optional cycle accounting of the ping-pong forward (build with -DMEMO_FWD_PROF,
// tools/fwd_prof.py), one softmax thread per group (g = 0, 1), summed over
// tiles: [8g+0] waiting for S, [8g+1] S ready -> keys [0,64) released, [8g+2]
// S ready -> all of P released, [8g+3] release -> end of tile (row sum), [8g+4]
// tiles; [16] MMA warp waiting for P, [17] MMA warp waiting for K/V, [18] MMA
// warp total.
#ifdef MEMO_FWD_PROF
__device__ unsigned long long g_fwd_prof[24];
#define FWD_PROF(...) __VA_ARGS__
#else
#define FWD_PROF(...)
#endif

// SPLIT_P: release P in two key halves.  NULL_SM (ablation build only): no row
// max and no exponentials (P = bf16(S)); every load, store, barrier and MMA is
// kept, so its time is the kernel's ceiling with free softmax math.
// SEQ (ablation): the two groups' softmax warps of one SMSP take turns on the
// exponential phase (named barriers: A(j) -> B(j) -> A(j+1) ...), so each runs
// alone on its SMSP instead of both slowing each other down.
// QSTORE (ablation): P in four quarters stored as packed, keys [0,64) released
// after the third quarter, row sum after the release (measured 1-2 % slower).
// LDSB: no tcgen05.wait::ld after the S loads.  ptxas scoreboards the
// tcgen05.ld destination registers like any load's (CUTLASS's sm_100 kernels
// issue no wait::ld at all), so the row max starts on the first 32 columns
// while the other three loads are in flight.  Safe here because nothing
// reuses S's columns before this thread's P stores, which depend on every
// loaded value.  0.5-1 % at 128K, bitwise equal (LDSB = false: ablation 33).
// CL2 (the default when the pair count is even): CTA pairs (clusters of 2) on query-tile pairs pp and
// pp-1 of one head share every K/V tile by multicast (each CTA loads one
// 64-column chunk of K_j and of V_j for both); the lower CTA releases the upper
// one's two extra key tiles without computing on them.
template <int EMU_EVERY, bool SPLIT_P = true, bool NULL_SM = false, bool NULL_MMA = false, bool SEQ = false,
          bool QSTORE = false, bool LDSB = true, bool CL2 = false>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, int S, int H, float scale_log2) {
  constexpr int D = 128;
  using L = FwdPpSmem;
  constexpr int NC = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2] per group
  uint64_t* p_full = bars + 11;  // [2 groups][2 key halves]: P of keys [0,64) / [64,128) written
  uint64_t* o_done = bars + 15;  // [2] per group
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int n_pairs = S / (2 * TILE);
  const int pp = n_pairs - 1 - static_cast<int>(blockIdx.x);  // heavy pairs first
  const int hh = blockIdx.y;
  const int qt0 = 2 * pp;
  const int n_kv = qt0 + 2;  // key tiles of group B; group A uses n_kv - 1
  // rank in the 1-D cluster of 2 = blockIdx.x & 1 (rank 1 holds the lower query-tile pair); derived from
  // blockIdx (not %cluster_ctarank) so ptxas keeps the loop state uniform
  const uint32_t crank = CL2 ? (blockIdx.x & 1u) : 0u;
  const int n_load = n_kv + 2 * static_cast<int>(crank);    // key tiles the pair walks together
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::mbar_init(q_full, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&k_full[s2], 1);
      dev::mbar_init(&k_empty[s2], CL2 ? 2 : 1);  // CL2: both CTAs release a stage
      dev::mbar_init(&v_full[s2], 1);
      dev::mbar_init(&v_empty[s2], CL2 ? 2 : 1);
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&p_full[2 * s2], 128);
      dev::mbar_init(&p_full[2 * s2 + 1], 128);
      dev::mbar_init(&o_done[s2], 1);
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  if (CL2)
    dev::cluster_sync();  // the peer's barriers exist before its first multicast lands here
  else
    __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      if (lane == 0) {
        dev::mbar_expect_tx(q_full, 2 * L::TILE_BYTES);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::QA_OFF + c * CHUNK_BYTES, &map_q, q_full, hh * D + c * 64, qt0 * TILE);
          dev::tma_load_2d(smem + L::QB_OFF + c * CHUNK_BYTES, &map_q, q_full, hh * D + c * 64, (qt0 + 1) * TILE);
        }
        for (int j = 0; j < n_load; ++j) {
          const int st = j & 1;
          const uint32_t ph = (j >> 1) & 1;
          const int c0 = CL2 ? static_cast<int>(crank) : 0, c1 = CL2 ? c0 + 1 : NC;  // CL2: this CTA's chunk
          dev::mbar_wait(&k_empty[st], ph ^ 1);
          dev::mbar_expect_tx(&k_full[st], L::TILE_BYTES);
          for (int c = c0; c < c1; ++c) {
            if (CL2)
              dev::tma_load_2d_mc(smem + L::K_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_k, &k_full[st],
                                  hh * D + c * 64, j * TILE, 0x3);
            else
              dev::tma_load_2d(smem + L::K_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_k, &k_full[st],
                               hh * D + c * 64, j * TILE);
          }
          dev::mbar_wait(&v_empty[st], ph ^ 1);
          dev::mbar_expect_tx(&v_full[st], L::TILE_BYTES);
          for (int c = c0; c < c1; ++c) {
            if (CL2)
              dev::tma_load_2d_mc(smem + L::V_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_v, &v_full[st],
                                  hh * D + c * 64, j * TILE, 0x3);
            else
              dev::tma_load_2d(smem + L::V_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_v, &v_full[st],
                               hh * D + c * 64, j * TILE);
          }
        }
        if (CL2) {  // producer tail: the peer's releases of the last stages land here asynchronously
          for (int j = n_load; j < n_load + 2; ++j) {
            dev::mbar_wait(&k_empty[j & 1], ((j >> 1) & 1) ^ 1);
            dev::mbar_wait(&v_empty[j & 1], ((j >> 1) & 1) ^ 1);
          }
        }
      }
    } else if (warp == 1) {
      // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_o = dev::idesc_bf16_f32(128, D, false, true);
      const uint64_t qd[2] = {kmajor_base(dev::smem_u32(smem + L::QA_OFF)),
                              kmajor_base(dev::smem_u32(smem + L::QB_OFF))};
      const int nA = n_kv - 1;
      dev::mbar_wait_w(q_full, 0);
      FWD_PROF(long long pf_total = clock64(); long long pf_kv = 0, pf_p = 0;)
      auto issue_s = [&](int g, int j) {  // S_g(j) = Q_g K_j^T ; group A always issues first for tile j
        const int st = j & 1;
        if (g == 0 || j == nA) {
          FWD_PROF(long long t = clock64();)
          dev::mbar_wait_w(&k_full[st], (j >> 1) & 1);
          FWD_PROF(pf_kv += clock64() - t;)
          dev::tc_fence_after();
        }
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + L::K_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          if (!NULL_MMA)
            dev::mma_bf16_ss_w(tmem + g * 128, kmajor_step(g ? qd[1] : qd[0], kk), kmajor_step(kd, kk), idesc_s,
                               kk > 0);
        dev::mma_commit_w(&s_full[g]);
        if (g == 1) {  // B is the last reader of K_j
          if (CL2)
            dev::mma_commit_mc_w(&k_empty[st], 0x3);
          else
            dev::mma_commit_w(&k_empty[st]);
        }
      };
      auto issue_pv = [&](int g, int j) {  // O_g += P_g(j) V_j, one key half at a time
        const int st = j & 1;
        FWD_PROF(long long t = clock64();)
        dev::mbar_wait_w(&p_full[2 * g], j & 1);
        FWD_PROF(long long t2 = clock64(); pf_p += t2 - t;)
        if (g == 0 || j == nA) {
          dev::mbar_wait_w(&v_full[st], (j >> 1) & 1);
        }
        FWD_PROF(pf_kv += clock64() - t2;)
        dev::tc_fence_after();
        const uint64_t vd = mnmajor_base(dev::smem_u32(smem + L::V_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < TILE / 32; ++kk)
          if (!NULL_MMA)
            dev::mma_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + kk * 8, mnmajor_step(vd, kk), idesc_o,
                               (j | kk) != 0);
        // keys [64,128): their P lands while the first half's MMAs run
        if (SPLIT_P) {
          FWD_PROF(long long t3 = clock64();)
          dev::mbar_wait_w(&p_full[2 * g + 1], j & 1);
          FWD_PROF(pf_p += clock64() - t3;)
          dev::tc_fence_after();
        }
#pragma unroll
        for (int kk = TILE / 32; kk < TILE / 16; ++kk)
          if (!NULL_MMA)
            dev::mma_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + kk * 8, mnmajor_step(vd, kk), idesc_o, true);
        // S_g(j+1) is issued after PV_g(j), so s_full already orders the
        // softmax's O rescale after PV_g(j); o_done only serves the epilogue.
        if (j == (g ? n_kv - 1 : nA - 1)) dev::mma_commit_w(&o_done[g]);
        if (g == 1) {
          if (CL2)
            dev::mma_commit_mc_w(&v_empty[st], 0x3);
          else
            dev::mma_commit_w(&v_empty[st]);
        }
      };
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j < nA) {
          issue_pv(0, j);
          if (j + 1 < nA) issue_s(0, j + 1);
        }
        issue_pv(1, j);
        if (j + 1 < n_kv) issue_s(1, j + 1);
      }
      if (CL2) {  // the upper pair's two extra key tiles: release them for the peer, no MMAs
        for (int j = n_kv; j < n_load; ++j) {
          const int st = j & 1;
          dev::mbar_wait_w(&k_full[st], (j >> 1) & 1);
          dev::mma_commit_mc_w(&k_empty[st], 0x3);
          dev::mbar_wait_w(&v_full[st], (j >> 1) & 1);
          dev::mma_commit_mc_w(&v_empty[st], 0x3);
        }
      }
      FWD_PROF(if (lane == 0) {
        atomicAdd(&g_fwd_prof[16], static_cast<unsigned long long>(pf_p));
        atomicAdd(&g_fwd_prof[17], static_cast<unsigned long long>(pf_kv));
        atomicAdd(&g_fwd_prof[18], static_cast<unsigned long long>(clock64() - pf_total));
      })
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    const int g = (warp - 4) >> 2;  // softmax group: 0 -> tile A, 1 -> tile B
    const uint32_t q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int qt = qt0 + g;
    const int qidx = qt * TILE + row;
    const int n_my = qt + 1;
    const uint32_t lane_off = (q4 * 32) << 16;
    const uint32_t t_s = tmem + g * 128 + lane_off;
    const uint32_t t_o = tmem + 256 + g * D + lane_off;
    float m = -INFINITY, l = 0.f;
    FWD_PROF(const bool pf_on = (q4 == 0 && lane == 0); long long pf[4] = {0, 0, 0, 0}; long long pf_t1 = 0;)
    for (int j = 0; j < n_my; ++j) {
      FWD_PROF(long long pf_t0 = clock64();)
      dev::mbar_wait(&s_full[g], j & 1);
      FWD_PROF(pf_t1 = clock64(); pf[0] += pf_t1 - pf_t0;)
      dev::tc_fence_after();
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) dev::tmem_ld32(t_s + c * 32, r[c]);
      if (!LDSB) dev::tmem_ld_wait_regs(r[0], r[1], r[2], r[3]);
      bool any = false;
      float factor = 1.f;
      uint32_t p[64];
      auto tile = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        if (DIAG) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i > row) r[i >> 5][i & 31] = __float_as_uint(-INFINITY);
        }
        // row max: 8 independent chains of 3-input FMNMX3 (68 instructions, not 134)
        auto rv = [&](int i) { return NULL_SM ? 0.f : __uint_as_float(r[i >> 5][i & 31]); };
        float mx8[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmaxf(rv(k2), rv(8 + k2));
#pragma unroll
        for (int i = 16; i < 128; i += 16)
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmax3f(mx8[k2], rv(i + k2), rv(i + 8 + k2));
        const float mxa = fmax3f(mx8[0], mx8[1], mx8[2]);
        const float mxb = fmax3f(mx8[3], mx8[4], mx8[5]);
        const float mxr = fmax3f(mxa, mxb, fmaxf(mx8[6], mx8[7]));
        const float cand = fmaxf(m, mxr * scale_log2);
        const bool need = j == 0 || cand > m + kRescaleThreshold;
        any = __any_sync(0xffffffffu, need);
        float m_new = m;
        if (any) {
          m_new = cand;
          factor = j == 0 ? 0.f : dev::ex2(m - m_new);
        }
        if constexpr (!QSTORE) {
        // P in two key halves: the first half's P (keys [0,64)) is stored and
        // released before the second half's exponentials, so the tensor pipe
        // can run PV over the first half while the second is computed (ptxas
        // interleaves the two halves' exponentials; tools/fwd_prof.py).
        uint64_t sum4[4] = {0, 0, 0, 0};
        auto exps = [&](int i0) {
#pragma unroll
          for (int i = i0; i < i0 + 32; ++i) {
            const uint64_t x2 = ffma2(f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                              __uint_as_float(r[i >> 4][(2 * i + 1) & 31])),
                                      scale_log2, -m_new);
            float a, b;
            if (NULL_SM) {
              a = f2_lo(x2);
              b = f2_hi(x2);
            } else if (EMU_EVERY > 0 && (i % (EMU_EVERY > 0 ? EMU_EVERY : 1)) == EMU_EVERY - 1) {
              const uint64_t e2 = exp2_fma2(x2);
              a = f2_lo(e2);
              b = f2_hi(e2);
            } else {
              a = dev::ex2(f2_lo(x2));
              b = dev::ex2(f2_hi(x2));
            }
            sum4[i & 3] = fadd2(sum4[i & 3], f2_pack(a, b));
            p[i] = dev::pack_bf16(a, b);
          }
        };
        exps(0);
        dev::tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&p[0]));
        if (any && j > 0) {
          // O_g holds P(j-1)V(j-1) (PV_g(j-1) completed before s_full_g(j)
          // fired); rescaled before PV_g(j) may start, i.e. before half 0 is released
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            dev::tmem_ld32(t_o + c * 32, o);
            dev::tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
            dev::tmem_st32(t_o + c * 32, o);
          }
        }
        if (SPLIT_P) {
          dev::tmem_st_wait();
          dev::tc_fence_before();
          dev::mbar_arrive(&p_full[2 * g]);
          FWD_PROF(pf[1] += clock64() - pf_t1;)
        }
        exps(32);
        dev::tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&p[32]));
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&p_full[2 * g + (SPLIT_P ? 1 : 0)]);
        FWD_PROF(long long pf_t3 = clock64(); pf[2] += pf_t3 - pf_t1;)
        const uint64_t s01 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l = l * factor + (f2_lo(s01) + f2_hi(s01));
        m = m_new;
        FWD_PROF(pf[3] += clock64() - pf_t3;)
        } else {
        // P in four key quarters, each stored (tcgen05.st, asynchronous) as soon
        // as it is packed.  Keys [0,64) are released after the third quarter's
        // exponentials, when their stores have long landed (no exposed store
        // wait), so PV over them overlaps the last quarter; keys [64,128) at the
        // end.  The exponentials overwrite their logits in r: the row sum is
        // taken after the release, off the S -> P critical path.
        auto exq = [&](int q, float neg_m) {  // column pairs [16q, 16q+16)
#pragma unroll
          for (int i = 16 * q; i < 16 * q + 16; ++i) {
            const uint64_t x2 = ffma2(f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                              __uint_as_float(r[i >> 4][(2 * i + 1) & 31])),
                                      scale_log2, neg_m);
            float a, b;
            if (NULL_SM) {
              a = f2_lo(x2);
              b = f2_hi(x2);
            } else if (EMU_EVERY > 0 && (i % (EMU_EVERY > 0 ? EMU_EVERY : 1)) == EMU_EVERY - 1) {
              const uint64_t e2 = exp2_fma2(x2);
              a = f2_lo(e2);
              b = f2_hi(e2);
            } else {
              a = dev::ex2(f2_lo(x2));
              b = dev::ex2(f2_hi(x2));
            }
            r[i >> 4][(2 * i) & 31] = __float_as_uint(a);
            r[i >> 4][(2 * i + 1) & 31] = __float_as_uint(b);
            p[i] = dev::pack_bf16(a, b);
          }
        };
        auto st_q = [&](int q) { dev::tmem_st16(t_s + 16 * q, *reinterpret_cast<uint32_t(*)[16]>(&p[16 * q])); };
        if (any && j > 0) {
          // O_g holds P(j-1)V(j-1) (PV_g(j-1) completed before s_full_g(j)
          // fired); rescaled before any P of this tile is released
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            dev::tmem_ld32(t_o + c * 32, o);
            dev::tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
            dev::tmem_st32(t_o + c * 32, o);
          }
        }
        // The same ordering problem for the stores: ptxas keeps the volatile
        // tcgen05.st in program order but would hoist the next quarters'
        // exponentials above them, issuing every store just before the wait.  A
        // clock read after each store (ordered with it) seeds the next quarter's
        // bias with a signed zero.
        auto after_store = [&]() {
          uint32_t c;
          asm volatile("mov.u32 %0, %%clock;" : "=r"(c)::"memory");
          return -m_new + __uint_as_float(c & 0x80000000u) * 0.f;
        };
        // turn: A(j) waits for B(j-1), B(j) waits for A(j) (B's last tile has no A(j))
        float neg_m0 = -m_new;
        if (SEQ && (g == 1 ? j + 1 < n_my : j > 0)) {
          named_bar(g == 0 ? 5 + q4 : 1 + q4, 64);
          neg_m0 = after_store();  // clock read after the barrier: the exponentials stay below it
        }
        exq(0, neg_m0);
        st_q(0);
        exq(1, after_store());
        st_q(1);
        exq(2, after_store());
        // ptxas would otherwise schedule the last quarter's exponentials above
        // the release (no data dependency keeps them below it): their bias
        // carries a signed zero derived from the arrive's state token.
        float neg_m3 = -m_new;
        if (SPLIT_P) {
          dev::tmem_st_wait();
          dev::tc_fence_before();
          const uint64_t tok0 = dev::mbar_arrive_token(&p_full[2 * g]);
          neg_m3 += __uint_as_float(static_cast<uint32_t>(tok0) & 0x80000000u) * 0.f;
          FWD_PROF(pf[1] += clock64() - pf_t1;)
        }
        st_q(2);
        exq(3, neg_m3);
        if (SEQ) {  // pass the turn: A(j) -> B(j) always; B(j) -> A(j+1) if A has tile j+1
          if (g == 0)
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + q4), "r"(64) : "memory");
          else if (j + 1 < n_my - 1)
            asm volatile("bar.arrive %0, %1;" ::"r"(5 + q4), "r"(64) : "memory");
        }
        st_q(3);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        const uint64_t tok = dev::mbar_arrive_token(&p_full[2 * g + (SPLIT_P ? 1 : 0)]);
        FWD_PROF(long long pf_t3 = clock64(); pf[2] += pf_t3 - pf_t1;)
        // Row sum, same pairing and order as when it ran inside the exponential
        // loop (bitwise equal).  Its four chains start from a signed zero derived
        // from the arrive's state token, so ptxas cannot hoist the adds back
        // above the arrive (onto the S -> P critical path).
        const float z = __uint_as_float(static_cast<uint32_t>(tok) & 0x80000000u) * 0.f;
        uint64_t sum4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) sum4[k] = f2_pack(z, z);
#pragma unroll
        for (int i = 0; i < 64; ++i)
          sum4[i & 3] = fadd2(sum4[i & 3], f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                                   __uint_as_float(r[i >> 4][(2 * i + 1) & 31])));
        const uint64_t s01 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l = l * factor + (f2_lo(s01) + f2_hi(s01));
        m = m_new;
        FWD_PROF(pf[3] += clock64() - pf_t3;)
        }
      };
      if (j == qt)
        tile(std::true_type{});
      else
        tile(std::false_type{});
    }
    FWD_PROF(if (pf_on) {
      for (int k = 0; k < 4; ++k) atomicAdd(&g_fwd_prof[8 * g + k], static_cast<unsigned long long>(pf[k]));
      atomicAdd(&g_fwd_prof[8 * g + 4], static_cast<unsigned long long>(n_my));
    })
    dev::mbar_wait(&o_done[g], 0);  // committed once, after the group's last PV
    dev::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + static_cast<long long>(qidx) * H * D + hh * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      dev::tmem_ld32(t_o + c * 32, o);
      dev::tmem_ld_wait_regs(o);
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        u.x = dev::pack_bf16(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv);
        u.y = dev::pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv);
        u.z = dev::pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv);
        u.w = dev::pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv);
        dst[i] = u;
      }
    }
    lse[static_cast<long long>(hh) * S + qidx] = (m + log2f(l)) * kLn2;
    dev::tc_fence_before();
  }
  if (CL2)
    dev::cluster_sync();  // no multicast or remote release still targets this CTA
  else
    __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

#ifdef MEMO_ATTN_ABLATIONS  // CTA-pair ping-pong forward (ablation build only)
// ------------------------------------------------- forward, ping-pong over a CTA pair
// attn_fwd_pp_kernel's schedule on a CTA pair (cta_group::2): the pair holds
// four query tiles (CTA r, group g -> tile 4q + 2g + r) and every MMA spans
// both CTAs (M = 256).  S_g = Q_g K_j^T reads each CTA's own Q rows and half
// of K_j (keys [64r, 64r+64)) from that CTA's shared memory; O_g += P_g V_j
// reads P from each CTA's TMEM and half of V_j (head-dim columns [64r, 64r+64)).
// Per SM that is 96 instead of 128 B/cycle of operand reads for S and 32
// instead of 64 for PV, and half the K/V TMA bytes: the one-CTA kernel's S
// runs at the 128 B/cycle shared-memory cap (tools/ubench_mma.cu).  The
// leader CTA issues the MMAs; both CTAs' softmax warps release P to barriers
// in the leader.  A group's two tiles need different key ranges (4q+2g+1 vs
// +2): the lower tile's last key tile is fully masked and only writes P = 0.
// Measured (ablation variants 42/44): bitwise equal to attn_fwd_pp_kernel,
// 131.9 ms at 128K against 111.4 ms -- both CTAs' softmax must release P
// before each pair MMA, and the cross-CTA arrivals lengthen the S -> P -> PV
// chain -- while its MMA-side ceiling (P = 0) is the same 95 ms as the
// one-CTA kernel's: the shared-memory operand rate was not what bounds it.
struct FwdPairSmem {
  static constexpr int Q_BYTES = 2 * CHUNK_BYTES;   // one 128-row Q tile, D = 128
  static constexpr int KV_BYTES = CHUNK_BYTES;      // half a K tile (64 rows x 128) / half a V tile (128 x 64)
  static constexpr int STAGES = 3;
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = Q_BYTES;
  static constexpr int K_OFF = 2 * Q_BYTES;
  static constexpr int V_OFF = K_OFF + STAGES * KV_BYTES;
  static constexpr int BAR_OFF = V_OFF + STAGES * KV_BYTES;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

template <int EMU_EVERY, bool NULL_SM = false>  // NULL_SM (ablation): P = 0 everywhere, the MMA-side ceiling
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k64,
                         const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ out,
                         float* __restrict__ lse, int S, int H, float scale_log2) {
  constexpr int D = 128;
  using L = FwdPairSmem;
  constexpr int NST = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;                 // leader: both CTAs' Q tiles
  uint64_t* k_full = bars + 1;                 // [NST] leader: both halves of K_j
  uint64_t* k_empty = k_full + NST;            // [NST] each CTA (leader's multicast commit)
  uint64_t* v_full = k_empty + NST;            // [NST] leader
  uint64_t* v_empty = v_full + NST;            // [NST] each CTA
  uint64_t* s_full = v_empty + NST;            // [2] each CTA
  uint64_t* p_full = s_full + 2;               // [2 groups][2 key halves] leader, 256 arrivals
  uint64_t* o_done = p_full + 4;               // [2] each CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const uint32_t rank = dev::cluster_ctarank();
  const int n_quads = S / (4 * TILE);
  const int quad = n_quads - 1 - static_cast<int>(blockIdx.x >> 1);  // heavy quads first
  const int hh = blockIdx.y;
  const int nA = 4 * quad + 2;  // key tiles of group A (its upper tile 4q+1 is diagonal at nA-1)
  const int n_kv = 4 * quad + 4;
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_k64);
    dev::tma_prefetch_desc(&map_v);
    dev::mbar_init(q_full, 1);
    for (int s2 = 0; s2 < NST; ++s2) {
      dev::mbar_init(&k_full[s2], 1);
      dev::mbar_init(&k_empty[s2], 1);
      dev::mbar_init(&v_full[s2], 1);
      dev::mbar_init(&v_empty[s2], 1);
    }
    for (int g = 0; g < 2; ++g) {
      dev::mbar_init(&s_full[g], 1);
      dev::mbar_init(&p_full[2 * g], 256);
      dev::mbar_init(&p_full[2 * g + 1], 256);
      dev::mbar_init(&o_done[g], 1);
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc_cg2(tmem_slot, 512);
  dev::tc_fence_before();
  dev::cluster_sync();  // both CTAs' barriers initialised before any remote arrival
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      if (lane == 0) {
        // ---- TMA producer (both CTAs): own Q tiles, own halves of K_j and V_j,
        // completion on the leader's barriers
        const uint32_t qf = dev::mapa(dev::smem_u32(q_full), 0);
        if (rank == 0) dev::mbar_expect_tx(q_full, 4 * L::Q_BYTES);
        for (int g = 0; g < 2; ++g)
          for (int c = 0; c < 2; ++c)
            dev::tma_load_2d_cg2(smem + (g ? L::QB_OFF : L::QA_OFF) + c * CHUNK_BYTES, &map_q, qf,
                                 hh * D + c * 64, (4 * quad + 2 * g + static_cast<int>(rank)) * TILE);
        for (int j = 0; j < n_kv; ++j) {
          const int st = j % NST;
          const uint32_t ph = (j / NST) & 1;
          dev::mbar_wait(&k_empty[st], ph ^ 1);
          if (rank == 0) dev::mbar_expect_tx(&k_full[st], 2 * L::KV_BYTES);
          for (int c = 0; c < 2; ++c)  // keys [64 rank, +64) of K_j, both 64-col chunks
            dev::tma_load_2d_cg2(smem + L::K_OFF + st * L::KV_BYTES + c * (L::KV_BYTES / 2), &map_k64,
                                 dev::mapa(dev::smem_u32(&k_full[st]), 0), hh * D + c * 64,
                                 j * TILE + static_cast<int>(rank) * 64);
          dev::mbar_wait(&v_empty[st], ph ^ 1);
          if (rank == 0) dev::mbar_expect_tx(&v_full[st], 2 * L::KV_BYTES);
          // head-dim columns [64 rank, +64) of V_j, all 128 keys
          dev::tma_load_2d_cg2(smem + L::V_OFF + st * L::KV_BYTES, &map_v, dev::mapa(dev::smem_u32(&v_full[st]), 0),
                               hh * D + static_cast<int>(rank) * 64, j * TILE);
        }
      }
    } else if (warp == 1 && rank == 0) {
      // ---- MMA issuer (leader only; whole warp converged, elect.sync issues)
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(256, 128, false, false);
      constexpr uint32_t idesc_o = dev::idesc_bf16_f32(256, D, false, true);
      const uint64_t qd[2] = {kmajor_base(dev::smem_u32(smem + L::QA_OFF)),
                              kmajor_base(dev::smem_u32(smem + L::QB_OFF))};
      dev::mbar_wait_cluster_w(q_full, 0);
      dev::tc_fence_after();
      auto issue_s = [&](int g, int j) {  // S_g(j), both CTAs' rows
        const int st = j % NST;
        if (g == 0 || j == nA) {
          dev::mbar_wait_cluster_w(&k_full[st], (j / NST) & 1);
          dev::tc_fence_after();
        }
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + L::K_OFF + st * L::KV_BYTES));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma2_bf16_ss_w(tmem + g * 128, kmajor_step(g ? qd[1] : qd[0], kk),
                              kmajor_step_c<L::KV_BYTES / 2>(kd, kk), idesc_s, kk > 0);
        dev::mma2_commit_mc_w(&s_full[g], 0x3);
        if (g == 1) dev::mma2_commit_mc_w(&k_empty[st], 0x3);  // B is the last reader of K_j
      };
      auto issue_pv = [&](int g, int j) {  // O_g += P_g(j) V_j, one key half at a time
        const int st = j % NST;
        dev::mbar_wait_cluster_w(&p_full[2 * g], j & 1);
        if (g == 0 || j == nA) dev::mbar_wait_cluster_w(&v_full[st], (j / NST) & 1);
        dev::tc_fence_after();
        const uint64_t vd = mnmajor_base(dev::smem_u32(smem + L::V_OFF + st * L::KV_BYTES));
#pragma unroll
        for (int kk = 0; kk < TILE / 32; ++kk)
          dev::mma2_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + kk * 8, mnmajor_step(vd, kk), idesc_o,
                              (j | kk) != 0);
        dev::mbar_wait_cluster_w(&p_full[2 * g + 1], j & 1);
        dev::tc_fence_after();
#pragma unroll
        for (int kk = TILE / 32; kk < TILE / 16; ++kk)
          dev::mma2_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + kk * 8, mnmajor_step(vd, kk), idesc_o, true);
        if (j == (g ? n_kv - 1 : nA - 1)) dev::mma2_commit_mc_w(&o_done[g], 0x3);
        if (g == 1) dev::mma2_commit_mc_w(&v_empty[st], 0x3);
      };
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j < nA) {
          issue_pv(0, j);
          if (j + 1 < nA) issue_s(0, j + 1);
        }
        issue_pv(1, j);
        if (j + 1 < n_kv) issue_s(1, j + 1);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    const int g = (warp - 4) >> 2;  // softmax group: 0 -> tile A, 1 -> tile B
    const uint32_t q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int qt = 4 * quad + 2 * g + static_cast<int>(rank);
    const int qidx = qt * TILE + row;
    const int n_my = g ? n_kv : nA;
    const uint32_t lane_off = (q4 * 32) << 16;
    const uint32_t t_s = tmem + g * 128 + lane_off;
    const uint32_t t_o = tmem + 256 + g * D + lane_off;
    const uint32_t pf0 = dev::mapa(dev::smem_u32(&p_full[2 * g]), 0);
    const uint32_t pf1 = dev::mapa(dev::smem_u32(&p_full[2 * g + 1]), 0);
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_my; ++j) {
      dev::mbar_wait(&s_full[g], j & 1);
      dev::tc_fence_after();
      if (NULL_SM || j > qt) {  // the group's other tile reaches one key tile further: all masked, P = 0
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0u;
        dev::tmem_st32(t_s, z);
        dev::tmem_st32(t_s + 32, z);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive_cluster(pf0);
        dev::mbar_arrive_cluster(pf1);
        continue;
      }
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) dev::tmem_ld32(t_s + c * 32, r[c]);
      // no wait::ld: consumers wait on the registers' scoreboard (attn_fwd_pp_kernel LDSB)
      bool any = false;
      float factor = 1.f;
      uint32_t p[64];
      auto tile = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        if (DIAG) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i > row) r[i >> 5][i & 31] = __float_as_uint(-INFINITY);
        }
        auto rv = [&](int i) { return __uint_as_float(r[i >> 5][i & 31]); };
        float mx8[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmaxf(rv(k2), rv(8 + k2));
#pragma unroll
        for (int i = 16; i < 128; i += 16)
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmax3f(mx8[k2], rv(i + k2), rv(i + 8 + k2));
        const float mxa = fmax3f(mx8[0], mx8[1], mx8[2]);
        const float mxb = fmax3f(mx8[3], mx8[4], mx8[5]);
        const float mxr = fmax3f(mxa, mxb, fmaxf(mx8[6], mx8[7]));
        const float cand = fmaxf(m, mxr * scale_log2);
        const bool need = j == 0 || cand > m + kRescaleThreshold;
        any = __any_sync(0xffffffffu, need);
        float m_new = m;
        if (any) {
          m_new = cand;
          factor = j == 0 ? 0.f : dev::ex2(m - m_new);
        }
        uint64_t sum4[4] = {0, 0, 0, 0};
        auto exps = [&](int i0) {
#pragma unroll
          for (int i = i0; i < i0 + 32; ++i) {
            const uint64_t x2 = ffma2(f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                              __uint_as_float(r[i >> 4][(2 * i + 1) & 31])),
                                      scale_log2, -m_new);
            float a, b;
            if (EMU_EVERY > 0 && (i % (EMU_EVERY > 0 ? EMU_EVERY : 1)) == EMU_EVERY - 1) {
              const uint64_t e2 = exp2_fma2(x2);
              a = f2_lo(e2);
              b = f2_hi(e2);
            } else {
              a = dev::ex2(f2_lo(x2));
              b = dev::ex2(f2_hi(x2));
            }
            sum4[i & 3] = fadd2(sum4[i & 3], f2_pack(a, b));
            p[i] = dev::pack_bf16(a, b);
          }
        };
        exps(0);
        dev::tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&p[0]));
        if (any && j > 0) {
          // O_g holds P(j-1)V(j-1) (PV_g(j-1) completed before s_full_g(j) fired)
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            dev::tmem_ld32(t_o + c * 32, o);
            dev::tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
            dev::tmem_st32(t_o + c * 32, o);
          }
        }
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive_cluster(pf0);
        exps(32);
        dev::tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&p[32]));
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive_cluster(pf1);
        const uint64_t s01 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l = l * factor + (f2_lo(s01) + f2_hi(s01));
        m = m_new;
      };
      if (j == qt)
        tile(std::true_type{});
      else
        tile(std::false_type{});
    }
    dev::mbar_wait(&o_done[g], 0);  // committed once, after the group's last PV
    dev::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + static_cast<long long>(qidx) * H * D + hh * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      dev::tmem_ld32(t_o + c * 32, o);
      dev::tmem_ld_wait_regs(o);
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        u.x = dev::pack_bf16(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv);
        u.y = dev::pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv);
        u.z = dev::pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv);
        u.w = dev::pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv);
        dst[i] = u;
      }
    }
    lse[static_cast<long long>(hh) * S + qidx] = (m + log2f(l)) * kLn2;
  }
  dev::tc_fence_before();
  dev::cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc_cg2(tmem, 512);
  }
}
#endif  // MEMO_ATTN_ABLATIONS

#ifdef MEMO_ATTN_ABLATIONS  // split-row ping-pong forward (ablation build only)
// ------------------------------------------------------- forward, ping-pong, split rows
// The ping-pong schedule of attn_fwd_pp_kernel (two query tiles A/B per CTA,
// TMEM S_A | S_B | O_A | O_B, one MMA warp alternating PV_A S_A PV_B S_B), with
// each query row's softmax split over two warps: warpgroup (g, hf) handles key
// columns [64hf, 64hf+64) of group g's tile, so every SMSP runs four softmax
// warps instead of two.  The per-tile softmax latency (S ready -> P released)
// is what sets the tensor pipe's idle time in the one-warp-per-row kernel
// (tools/fwd_prof.py: ~1650 of a ~2800-cycle step); halving each warp's share
// of the row shortens it.  The two halves exchange their row maxima through
// shared memory behind a 64-thread named barrier (one per group and lane
// quarter) and release their P halves independently: P of keys [0,64) lands in
// S columns [0,32) (half 0's own columns), keys [64,128) in columns [64,96).
// Only the hf = 0 warp rescales O (all 128 columns, before it releases the
// first P half, which is what starts PV_g(j)).
struct FwdPp2wSmem {
  static constexpr int TILE_BYTES = 2 * CHUNK_BYTES;  // D = 128
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = TILE_BYTES;
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;  // 2-stage K and V rings
  static constexpr int X_OFF = V_OFF + 2 * TILE_BYTES;  // [2 parity][2 g][2 hf][128] f32
  static constexpr int BAR_OFF = X_OFF + 2 * 2 * 2 * 128 * 4;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};
constexpr int PP2W_THREADS = 32 * 20;

// SEQ: the groups take turns on the exponential phase (mbarriers per lane
// quarter, 64 arrivals = the group's two warps), so a tile's softmax gets the
// SMSP's MUFU/issue to itself: A(j) -> B(j) -> A(j+1) ...
template <int EMU_EVERY, bool SEQ = false>
__global__ void __launch_bounds__(PP2W_THREADS, 1)
    attn_fwd_pp2w_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                         const __grid_constant__ CUtensorMap map_v, __nv_bfloat16* __restrict__ out,
                         float* __restrict__ lse, int S, int H, float scale_log2) {
  constexpr int D = 128;
  constexpr bool NULL_MMA = false;
  using L = FwdPp2wSmem;
  constexpr int NC = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2] per group
  uint64_t* p_full = bars + 11;  // [2 groups][2 key halves], one warpgroup each
  uint64_t* o_done = bars + 15;  // [2] per group
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  uint64_t* turn_ab = bars + 18;  // [4] per lane quarter: A's exponentials of tile j done
  uint64_t* turn_ba = bars + 22;  // [4]: B's exponentials of tile j done
  const uint32_t xchg_s = dev::smem_u32(smem + L::X_OFF);

  const int n_pairs = S / (2 * TILE);
  const int pp = n_pairs - 1 - static_cast<int>(blockIdx.x);  // heavy pairs first
  const int hh = blockIdx.y;
  const int qt0 = 2 * pp;
  const int n_kv = qt0 + 2;  // key tiles of group B; group A uses n_kv - 1
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::mbar_init(q_full, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&k_full[s2], 1);
      dev::mbar_init(&k_empty[s2], 1);
      dev::mbar_init(&v_full[s2], 1);
      dev::mbar_init(&v_empty[s2], 1);
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&p_full[2 * s2], 128);
      dev::mbar_init(&p_full[2 * s2 + 1], 128);
      dev::mbar_init(&o_done[s2], 1);
    }
    for (int q = 0; q < 4; ++q) {
      dev::mbar_init(&turn_ab[q], 64);
      dev::mbar_init(&turn_ba[q], 64);
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      if (lane == 0) {
        dev::mbar_expect_tx(q_full, 2 * L::TILE_BYTES);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::QA_OFF + c * CHUNK_BYTES, &map_q, q_full, hh * D + c * 64, qt0 * TILE);
          dev::tma_load_2d(smem + L::QB_OFF + c * CHUNK_BYTES, &map_q, q_full, hh * D + c * 64, (qt0 + 1) * TILE);
        }
        for (int j = 0; j < n_kv; ++j) {
          const int st = j & 1;
          const uint32_t ph = (j >> 1) & 1;
          dev::mbar_wait(&k_empty[st], ph ^ 1);
          dev::mbar_expect_tx(&k_full[st], L::TILE_BYTES);
          for (int c = 0; c < NC; ++c)
            dev::tma_load_2d(smem + L::K_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_k, &k_full[st],
                             hh * D + c * 64, j * TILE);
          dev::mbar_wait(&v_empty[st], ph ^ 1);
          dev::mbar_expect_tx(&v_full[st], L::TILE_BYTES);
          for (int c = 0; c < NC; ++c)
            dev::tma_load_2d(smem + L::V_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_v, &v_full[st],
                             hh * D + c * 64, j * TILE);
        }
      }
    } else if (warp == 1) {
      // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_o = dev::idesc_bf16_f32(128, D, false, true);
      const uint64_t qd[2] = {kmajor_base(dev::smem_u32(smem + L::QA_OFF)),
                              kmajor_base(dev::smem_u32(smem + L::QB_OFF))};
      const int nA = n_kv - 1;
      FWD_PROF(long long pf_total = clock64(); long long pf_kv = 0, pf_p = 0;)
      dev::mbar_wait_w(q_full, 0);
      auto issue_s = [&](int g, int j) {  // S_g(j) = Q_g K_j^T ; group A always issues first for tile j
        const int st = j & 1;
        if (g == 0 || j == nA) {
          FWD_PROF(long long t = clock64();)
          dev::mbar_wait_w(&k_full[st], (j >> 1) & 1);
          FWD_PROF(pf_kv += clock64() - t;)
          dev::tc_fence_after();
        }
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + L::K_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          if (!NULL_MMA)
            dev::mma_bf16_ss_w(tmem + g * 128, kmajor_step(g ? qd[1] : qd[0], kk), kmajor_step(kd, kk), idesc_s,
                               kk > 0);
        dev::mma_commit_w(&s_full[g]);
        if (g == 1) dev::mma_commit_w(&k_empty[st]);  // B is the last reader of K_j
      };
      auto issue_pv = [&](int g, int j) {  // O_g += P_g(j) V_j, one key half at a time
        const int st = j & 1;
        FWD_PROF(long long t = clock64();)
        dev::mbar_wait_w(&p_full[2 * g], j & 1);
        FWD_PROF(long long t2 = clock64(); pf_p += t2 - t;)
        if (g == 0 || j == nA) dev::mbar_wait_w(&v_full[st], (j >> 1) & 1);
        FWD_PROF(pf_kv += clock64() - t2;)
        dev::tc_fence_after();
        const uint64_t vd = mnmajor_base(dev::smem_u32(smem + L::V_OFF + st * L::TILE_BYTES));
#pragma unroll
        for (int kk = 0; kk < TILE / 32; ++kk)  // keys [0,64): P in S cols [0,32)
          dev::mma_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + kk * 8, mnmajor_step(vd, kk), idesc_o,
                             (j | kk) != 0);
        FWD_PROF(long long t3 = clock64();)
        dev::mbar_wait_w(&p_full[2 * g + 1], j & 1);
        FWD_PROF(pf_p += clock64() - t3;)
        dev::tc_fence_after();
#pragma unroll
        for (int kk = TILE / 32; kk < TILE / 16; ++kk)  // keys [64,128): P in S cols [64,96)
          dev::mma_bf16_ts_w(tmem + 256 + g * D, tmem + g * 128 + 32 + kk * 8, mnmajor_step(vd, kk), idesc_o,
                             true);
        if (j == (g ? n_kv - 1 : nA - 1)) dev::mma_commit_w(&o_done[g]);
        if (g == 1) dev::mma_commit_w(&v_empty[st]);
      };
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j < nA) {
          issue_pv(0, j);
          if (j + 1 < nA) issue_s(0, j + 1);
        }
        issue_pv(1, j);
        if (j + 1 < n_kv) issue_s(1, j + 1);
      }
      FWD_PROF(if (lane == 0) {
        atomicAdd(&g_fwd_prof[16], static_cast<unsigned long long>(pf_p));
        atomicAdd(&g_fwd_prof[17], static_cast<unsigned long long>(pf_kv));
        atomicAdd(&g_fwd_prof[18], static_cast<unsigned long long>(clock64() - pf_total));
      })
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    const int wg = (warp - 4) >> 2;
    const int g = wg >> 1;   // softmax group: 0 -> tile A, 1 -> tile B
    const int hf = wg & 1;   // key columns [64hf, 64hf+64) of every S tile
    const uint32_t q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int qt = qt0 + g;
    const int qidx = qt * TILE + row;
    const int n_my = qt + 1;
    const uint32_t lane_off = (q4 * 32) << 16;
    const uint32_t t_s = tmem + g * 128 + lane_off;
    const uint32_t t_o = tmem + 256 + g * D + lane_off;
    const int bar_id = 1 + 4 * g + q4;  // the two warps holding these rows of this group
    const uint32_t xmine = xchg_s + ((g * 2 + hf) * 128 + row) * 4;
    const uint32_t xother = xchg_s + ((g * 2 + (hf ^ 1)) * 128 + row) * 4;
    float m = -INFINITY, l = 0.f;
    FWD_PROF(const bool pf_on = (q4 == 0 && lane == 0 && hf == 0); long long pf[4] = {0, 0, 0, 0};)
    for (int j = 0; j < n_my; ++j) {
      FWD_PROF(long long pf_t0 = clock64();)
      dev::mbar_wait(&s_full[g], j & 1);
      FWD_PROF(long long pf_t1 = clock64(); pf[0] += pf_t1 - pf_t0;)
      dev::tc_fence_after();
      uint32_t r[2][32];
      dev::tmem_ld32(t_s + 64 * hf, r[0]);
      dev::tmem_ld32(t_s + 64 * hf + 32, r[1]);
      dev::tmem_ld_wait_regs(r[0], r[1]);
      auto tile = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        if (DIAG) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (64 * hf + i > row) r[i >> 5][i & 31] = __float_as_uint(-INFINITY);
        }
        auto rv = [&](int i) { return __uint_as_float(r[i >> 5][i & 31]); };
        float mx8[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmaxf(rv(k2), rv(8 + k2));
#pragma unroll
        for (int i = 16; i < 64; i += 16)
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) mx8[k2] = fmax3f(mx8[k2], rv(i + k2), rv(i + 8 + k2));
        const float mxa = fmax3f(mx8[0], mx8[1], mx8[2]);
        const float mxb = fmax3f(mx8[3], mx8[4], mx8[5]);
        const float mxh = fmax3f(mxa, mxb, fmaxf(mx8[6], mx8[7]));
        // row max across the two halves (parity-double-buffered slot: the
        // partner has read slot j&1 before it passes the barrier of tile j+1)
        const uint32_t par = (j & 1) * (2 * 2 * 128 * 4);
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(xmine + par), "f"(mxh) : "memory");
        named_bar(bar_id, 64);
        float other;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xother + par) : "memory");
        const float cand = fmaxf(m, fmaxf(mxh, other) * scale_log2);
        const bool need = j == 0 || cand > m + kRescaleThreshold;
        const bool any = __any_sync(0xffffffffu, need);  // same rows, same vote in both halves
        float m_new = m, factor = 1.f;
        if (any) {
          m_new = cand;
          factor = j == 0 ? 0.f : dev::ex2(m - m_new);
        }
        if (hf == 0 && any && j > 0) {
          // O_g holds P(j-1)V(j-1) (PV_g(j-1) completed before s_full_g(j)
          // fired); rescaled before this warp releases keys [0,64), which
          // starts PV_g(j)
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            dev::tmem_ld32(t_o + c * 32, o);
            dev::tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
            dev::tmem_st32(t_o + c * 32, o);
          }
        }
        float neg_m = -m_new;
        if (SEQ && (g == 1 ? j + 1 < n_my : j > 0)) {
          // A(j) waits for B(j-1), B(j) for A(j) (B's last tile has no A(j));
          // a clock read after the wait keeps ptxas from hoisting the exponentials
          dev::mbar_wait(g == 0 ? &turn_ba[q4] : &turn_ab[q4], g == 0 ? (j - 1) & 1 : j & 1);
          uint32_t c;
          asm volatile("mov.u32 %0, %%clock;" : "=r"(c)::"memory");
          neg_m += __uint_as_float(c & 0x80000000u) * 0.f;
        }
        uint64_t sum4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {  // 16 column pairs per store
          uint32_t p[16];
#pragma unroll
          for (int i = 16 * qq; i < 16 * qq + 16; ++i) {
            const uint64_t x2 = ffma2(f2_pack(__uint_as_float(r[i >> 4][(2 * i) & 31]),
                                              __uint_as_float(r[i >> 4][(2 * i + 1) & 31])),
                                      scale_log2, neg_m);
            float a, b;
            const int gi = 32 * hf + i;  // pair index within the row: same exponentials emulated as the pp kernel
            if (EMU_EVERY > 0 && (gi % (EMU_EVERY > 0 ? EMU_EVERY : 1)) == EMU_EVERY - 1) {
              const uint64_t e2 = exp2_fma2(x2);
              a = f2_lo(e2);
              b = f2_hi(e2);
            } else {
              a = dev::ex2(f2_lo(x2));
              b = dev::ex2(f2_hi(x2));
            }
            sum4[i & 3] = fadd2(sum4[i & 3], f2_pack(a, b));
            p[i - 16 * qq] = dev::pack_bf16(a, b);
          }
          if (SEQ && qq == 1) {  // pass the turn once this warp's exponentials are done
            if (g == 0)
              dev::mbar_arrive(&turn_ab[q4]);
            else if (j + 1 < n_my - 1)
              dev::mbar_arrive(&turn_ba[q4]);
          }
          dev::tmem_st16(t_s + 64 * hf + 16 * qq, p);  // inside this warp's own S columns
        }
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&p_full[2 * g + hf]);
        FWD_PROF(pf[2] += clock64() - pf_t1;)
        const uint64_t s01 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l = l * factor + (f2_lo(s01) + f2_hi(s01));
        m = m_new;
      };
      if (j == qt)
        tile(std::true_type{});
      else
        tile(std::false_type{});
    }
    FWD_PROF(if (pf_on) {
      for (int k = 0; k < 4; ++k) atomicAdd(&g_fwd_prof[8 * g + k], static_cast<unsigned long long>(pf[k]));
      atomicAdd(&g_fwd_prof[8 * g + 4], static_cast<unsigned long long>(n_my));
    })
    // epilogue: combine the two partial row sums, write O columns [64hf, 64hf+64) and the LSE
    const uint32_t par = (n_my & 1) * (2 * 2 * 128 * 4);
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(xmine + par), "f"(l) : "memory");
    named_bar(bar_id, 64);
    float l_other;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(l_other) : "r"(xother + par) : "memory");
    const float lt = hf == 0 ? l + l_other : l_other + l;  // same sum in both halves
    dev::mbar_wait(&o_done[g], 0);  // committed once, after the group's last PV
    dev::tc_fence_after();
    const float inv = 1.f / lt;
    __nv_bfloat16* orow = out + static_cast<long long>(qidx) * H * D + hh * D + 64 * hf;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      dev::tmem_ld32(t_o + 64 * hf + c * 32, o);
      dev::tmem_ld_wait_regs(o);
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        u.x = dev::pack_bf16(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv);
        u.y = dev::pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv);
        u.z = dev::pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv);
        u.w = dev::pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv);
        dst[i] = u;
      }
    }
    if (hf == 0) lse[static_cast<long long>(hh) * S + qidx] = (m + log2f(lt)) * kLn2;
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}
#endif  // MEMO_ATTN_ABLATIONS

// ============================================================== backward
// ndelta[h][t] = -sum_d dO*O ; nlse2[h][t] = -lse * log2(e)  (the delta / lse2 workspace)
// D/8 threads per (t, head) row, each loading 16 bytes of O and of dO (one
// 128-bit load each, whole rows per warp), then a shuffle tree over the row's
// lanes.  HBM-bound: 4·D bytes read and 8 written per row.
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                     const __nv_bfloat16* __restrict__ dout,
                                     const float* __restrict__ lse, float* __restrict__ delta,
                                     float* __restrict__ lse2, int S, int H, int D) {
  const int tpr = D / 8;  // threads per row (16 at D = 128, 8 at D = 64)
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gtid / tpr;  // row = t*H + hh
  const int sub = gtid - row * tpr;
  const bool live = row < S * H;
  float acc = 0.f;
  if (live) {
    const long long base = static_cast<long long>(row) * D + sub * 8;  // [S][H][D] contiguous
    const uint4 a = *reinterpret_cast<const uint4*>(o + base);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + base);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&av[i]);
      const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(&bv[i]);
      acc += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
    }
  }
  for (int off = tpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (live && sub == 0) {
    const int t = row / H, hh = row - t * H;
    const long long i = static_cast<long long>(hh) * S + t;
    delta[i] = -acc;            // stored negated: consumers add (FFMA2/FADD2, no negation)
    lse2[i] = -lse[i] * kLog2e;
  }
}

template <int D>
struct BwdSmem {
  static constexpr int NC = D / 64;
  static constexpr int TILE_BYTES = NC * CHUNK_BYTES;
  static constexpr int A0_OFF = 0;                        // K (dkdv)
  static constexpr int A1_OFF = A0_OFF + TILE_BYTES;      // V (dkdv)
  static constexpr int R0_OFF = A1_OFF + TILE_BYTES;      // ring: Q (dkdv) | K (dq)  [2]
  static constexpr int R1_OFF = R0_OFF + 2 * TILE_BYTES;  // ring: dO (dkdv) | V (dq) [2]
  static constexpr int VEC_OFF = R1_OFF + 2 * TILE_BYTES;  // [2][2][128] f32 (lse2, delta)
  static constexpr int BAR_OFF = VEC_OFF + 2 * 2 * 128 * 4;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};
constexpr int HALF = 64;             // rows of the partner tile per pipeline step
// Compute warps 4..11: two per SMSP (warps w and w+4 share TMEM lane quarter
// w%4), each owning one 32-column chunk of the 64-row half, so dependent
// TMEM-load / MUFU chains of one warp hide behind the other.
constexpr int BWD_COMPUTE_WARPS = 8;
constexpr int BWD_THREADS = 32 * (4 + BWD_COMPUTE_WARPS);
constexpr int HALF_BYTES = HALF * 128;  // byte offset of the second half inside a 64-col chunk

// Writes 32 consecutive columns of a dq/dk row: scale, inverse RoPE, bf16.
__device__ __forceinline__ void store_grad32(__nv_bfloat16* dst, float (&x)[32], float scale,
                                             const float2* cs) {
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] *= scale;
  if (cs) {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const float2 t = cs[p];
      const float a = x[2 * p], b = x[2 * p + 1];
      x[2 * p] = a * t.x + b * t.y;
      x[2 * p + 1] = -a * t.y + b * t.x;
    }
  }
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

#ifdef MEMO_ATTN_ABLATIONS  // K/V-in-shared-memory dK/dV (ablation build only)
template <int D>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap map_q,
                         const __grid_constant__ CUtensorMap map_k,
                         const __grid_constant__ CUtensorMap map_v,
                         const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                         const float* __restrict__ delta, __nv_bfloat16* __restrict__ dk,
                         __nv_bfloat16* __restrict__ dv, long long ld, const float2* __restrict__ rope,
                         long long pos0, int S, float scale, float scale_log2) {
  using L = BwdSmem<D>;
  constexpr int NC = L::NC;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* in_full = bars + 1;   // [2]
  uint64_t* in_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2] per TMEM buffer
  uint64_t* p_ready = bars + 7;   // [2]
  uint64_t* fin = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF);  // [stage][lse2|delta][128]

  const int n_tiles = S / TILE;
  const int kt = blockIdx.x;  // key tile
  const int hh = blockIdx.y;
  const int n_q = n_tiles - kt;  // query tiles kt..n_tiles-1
  const int n_g = 2 * n_q;       // 64-query halves
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::tma_prefetch_desc(&map_do);
    dev::mbar_init(kv_full, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&in_full[s2], 1);
      dev::mbar_init(&in_empty[s2], 1);
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&p_ready[s2], 32 * BWD_COMPUTE_WARPS);
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // buffer b: S^T half at b*128, dP^T half at b*128 + 64
  const uint32_t t_dv = tmem + 256, t_dk = tmem + 256 + D;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_expect_tx(kv_full, 2 * L::TILE_BYTES);
      for (int c = 0; c < NC; ++c) {
        dev::tma_load_2d(smem + L::A0_OFF + c * CHUNK_BYTES, &map_k, kv_full, hh * D + c * 64, kt * TILE);
        dev::tma_load_2d(smem + L::A1_OFF + c * CHUNK_BYTES, &map_v, kv_full, hh * D + c * 64, kt * TILE);
      }
      for (int i = 0; i < n_q; ++i) {
        const int qt = kt + i, st = i & 1;
        dev::mbar_wait(&in_empty[st], ((i >> 1) & 1) ^ 1);
        dev::mbar_expect_tx(&in_full[st], 2 * L::TILE_BYTES + 1024);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::R0_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_q,
                           &in_full[st], hh * D + c * 64, qt * TILE);
          dev::tma_load_2d(smem + L::R1_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_do,
                           &in_full[st], hh * D + c * 64, qt * TILE);
        }
        const long long off = static_cast<long long>(hh) * S + qt * TILE;
        dev::bulk_load(vec + st * 256, lse2 + off, 512, &in_full[st]);
        dev::bulk_load(vec + st * 256 + 128, delta + off, 512, &in_full[st]);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, HALF, false, false);
      constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
      const uint64_t kd0 = kmajor_base(dev::smem_u32(smem + L::A0_OFF));
      const uint64_t vd0 = kmajor_base(dev::smem_u32(smem + L::A1_OFF));
      dev::mbar_wait_w(kv_full, 0);
      auto issue_sd = [&](int g) {
        const int i = g >> 1, half = g & 1, st = i & 1, b = g & 1;
        if (half == 0) {
          dev::mbar_wait_w(&in_full[st], (i >> 1) & 1);
          dev::tc_fence_after();
        }
        const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::R0_OFF + st * L::TILE_BYTES) + half * HALF_BYTES);
        const uint64_t dod = kmajor_base(dev::smem_u32(smem + L::R1_OFF + st * L::TILE_BYTES) + half * HALF_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ss_w(tmem + b * 128, kmajor_step(kd0, kk), kmajor_step(qd, kk), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ss_w(tmem + b * 128 + 64, kmajor_step(vd0, kk), kmajor_step(dod, kk), idesc_s,
                           kk > 0);
        dev::mma_commit_w(&s_full[b]);
      };
      issue_sd(0);
      for (int g = 0; g < n_g; ++g) {
        if (g + 1 < n_g) issue_sd(g + 1);
        const int i = g >> 1, half = g & 1, st = i & 1, b = g & 1;
        dev::mbar_wait_w(&p_ready[b], (g >> 1) & 1);
        dev::tc_fence_after();
        const uint64_t qm = mnmajor_base(dev::smem_u32(smem + L::R0_OFF + st * L::TILE_BYTES) + half * HALF_BYTES);
        const uint64_t dom = mnmajor_base(dev::smem_u32(smem + L::R1_OFF + st * L::TILE_BYTES) + half * HALF_BYTES);
#pragma unroll
        for (int kk = 0; kk < HALF / 16; ++kk)
          dev::mma_bf16_ts_w(t_dv, tmem + b * 128 + 32 * (kk >> 1) + 8 * (kk & 1), mnmajor_step(dom, kk),
                             idesc_g, (g | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < HALF / 16; ++kk)
          dev::mma_bf16_ts_w(t_dk, tmem + b * 128 + 64 + 32 * (kk >> 1) + 8 * (kk & 1), mnmajor_step(qm, kk),
                             idesc_g, (g | kk) != 0);
        if (half == 1) dev::mma_commit_w(&in_empty[st]);
      }
      dev::mma_commit_w(fin);
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int ch = (warp - 4) >> 2;  // which 32-column chunk of each half this warp owns
    const int r = q4 * 32 + lane;  // key row in tile
    const int kidx = kt * TILE + r;
    const uint32_t lane_off = (q4 * 32) << 16;
    for (int g = 0; g < n_g; ++g) {
      const int i = g >> 1, half = g & 1, st = i & 1, b = g & 1;
      const bool diag = i == 0;
      if (half == 0) dev::mbar_wait(&in_full[st], (i >> 1) & 1);
      dev::mbar_wait(&s_full[b], (g >> 1) & 1);
      dev::tc_fence_after();
      // lse2 / delta of this half's queries, read with ld.shared (a generic
      // pointer here compiles to LD.E, which stalls on the LSU global path)
      const uint32_t l2 = dev::smem_u32(vec + st * 256 + half * HALF);
      const uint32_t dl = l2 + 128 * 4;
      const uint32_t t_st = tmem + b * 128 + lane_off, t_dpt = t_st + 64;
      // The causal mask only touches the diagonal tile; keep it out of the hot loop.
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        {
          const int c = ch;
          uint32_t sr[32], dr[32];
          dev::tmem_ld32(t_st + c * 32, sr);
          dev::tmem_ld32(t_dpt + c * 32, dr);
          dev::tmem_ld_wait_regs(sr, dr);
          uint32_t pp[16], dd[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 lv = dev::lds_f4(l2 + (c * 32 + 4 * j4) * 4);
            const float4 dv4 = dev::lds_f4(dl + (c * 32 + 4 * j4) * 4);
            const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
            const float dq[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
            float p4[4], d4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int qc = c * 32 + 4 * j4 + e;
              float p = dev::ex2(fmaf(__uint_as_float(sr[4 * j4 + e]), scale_log2, lq[e]));
              if (DIAG && half * HALF + qc < r) p = 0.f;
              p4[e] = p;
              d4[e] = p * (__uint_as_float(dr[4 * j4 + e]) + dq[e]);
            }
            pp[2 * j4] = dev::pack_bf16(p4[0], p4[1]);
            pp[2 * j4 + 1] = dev::pack_bf16(p4[2], p4[3]);
            dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
            dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
          }
          // packed bf16 stays inside this warp's own 32-column slice (the
          // other warp of the lane quarter may still be reading its slice)
          dev::tmem_st16(t_st + c * 32, pp);
          dev::tmem_st16(t_dpt + c * 32, dd);
        }
      };
      if (diag)
        body(std::true_type{});
      else
        body(std::false_type{});
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_ready[b]);
    }
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    __nv_bfloat16* dvrow = dv + static_cast<long long>(kidx) * ld + hh * D;
    __nv_bfloat16* dkrow = dk + static_cast<long long>(kidx) * ld + hh * D;
#pragma unroll 1
    for (int c = ch * (D / 64); c < (ch + 1) * (D / 64); ++c) {
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dv + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dvrow + c * 32, x, 1.f, nullptr);
      dev::tmem_ld32(t_dk + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dkrow + c * 32, x, scale,
                   rope ? rope + (pos0 + kidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}
#endif  // MEMO_ATTN_ABLATIONS

// Optional stall accounting of the dK/dV kernel (build with -DMEMO_DKDV_PROF):
// [0] MMA warp waiting for Q/dO tiles, [1] MMA warp waiting for P/dS (compute),
// [2] compute warp 4 waiting for S/dP (tensor), [3] compute warp 4 busy per step,
// [4] steps (MMA warp), [5] total kernel cycles of the MMA warp.
#ifdef MEMO_DKDV_PROF
__device__ unsigned long long g_dkdv_prof[16];
#define MEMO_PROF(x) x
#else
#define MEMO_PROF(x)
#endif

// ------------------------------------------------------------ dK/dV, K/V in TMEM
// Same math as attn_bwd_dkdv_kernel, but K and V (fixed for the CTA) sit in
// TMEM as the A operands of S^T = K Q^T and dP^T = V dO^T, so those MMAs read
// only the 32-query B slice from shared memory instead of re-reading the whole
// K/V tile per step (the SS form at N=64 ran at ~2/3 rate, smem-bound).  The
// TMEM budget then gives 32-query steps, double-buffered:
//   [0,128) dV | [128,256) dK | [256,320) K | [320,384) V | [384,448) buf0 | [448,512) buf1
//   buf: S^T [0,32) | dP^T [32,64); warp ch writes P^T into [16ch,+8), dS^T into [32+16ch,+8)
// K and V never touch shared memory; the ring holds 3 full Q/dO tiles.
constexpr int KV_NS = 3;
constexpr int QSTEP = 32;  // queries per pipeline step

template <int D>
struct DkdvTmSmem {
  static constexpr int NC = D / 64;
  static constexpr int CH_BYTES = CHUNK_BYTES;
  static constexpr int STAGE_BYTES = NC * CHUNK_BYTES;
  static constexpr int TILE_BYTES = NC * CHUNK_BYTES;
  static constexpr int RQ_OFF = 0;                             // [KV_NS] Q tiles
  static constexpr int RD_OFF = KV_NS * TILE_BYTES;            // [KV_NS] dO tiles
  static constexpr int VEC_OFF = 2 * KV_NS * TILE_BYTES;       // [KV_NS][lse2 128 | delta 128]
  static constexpr int BAR_OFF = VEC_OFF + KV_NS * 1024;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

// One-step stages (attn_bwd_dkdv_tm_kernel TS > 0): [TS] Q slices of QSTEP rows,
// [TS] dO slices, [TS][lse2 32 | delta 32] f32.
template <int D, int TSN>
struct DkdvTsSmem {
  static constexpr int NC = D / 64;
  static constexpr int CH_BYTES = QSTEP * 128;             // one 64-col chunk of a QSTEP-row slice
  static constexpr int STAGE_BYTES = NC * CH_BYTES;
  static constexpr int TILE_BYTES = STAGE_BYTES;
  static constexpr int RQ_OFF = 0;
  static constexpr int RD_OFF = TSN * STAGE_BYTES;
  static constexpr int VEC_OFF = 2 * TSN * STAGE_BYTES;
  static constexpr int BAR_OFF = VEC_OFF + TSN * 256;
  static constexpr int BYTES = BAR_OFF + 512 + 1024;
};

// WPQ: softmax-gradient warps per TMEM lane quarter (2: 16 query columns each;
// 4: 8 columns each, compacted P/dS write-back behind a per-quarter named barrier).
// EMU: every EMU-th column pair's exponentials run on the FMA pipe (exp2_fma)
// instead of MUFU.EX2 (0: none).  The MUFU is the largest single item of the
// compute warps' per-step critical path (tools/dkdv_prof.py).
// CL2 (the default for an even tile count): CTA pairs (clusters of 2) on key
// tiles 2p, 2p+1 of one head share each Q/dO tile by TMA multicast (each CTA
// loads one 64-column chunk of both, for both CTAs); the upper key tile walks
// query tile 2p too, fully masked (P = 0, dS = 0), so both CTAs consume the
// same stages.  A stage is refilled once both CTAs' MMAs have released it.
// QH (ablation build): P^T/dS^T released per 16-query half (warp ch = 0 / 1 of
// each lane quarter on its own barrier), so dV/dK over the first half can run
// under the second half's math; QH = 2 also makes the two warps of an SMSP take
// turns on the exponentials (ch 1 starts its MUFU work when ch 0 has issued
// its own).  Bitwise equal; at 128K QH = 1 is within noise of the default
// (205.4-206.1 vs 205.6-207.0 ms) and QH = 2 is 3 % slower (210.7-212.5 ms).
template <int D, int WPQ, int EMU = 0, bool SPLIT = false, int TS = 0, bool CL2 = false, int QH = 0,
          bool CLNOMC = false>
__global__ void __launch_bounds__(32 * (4 + 4 * WPQ), 1)
    attn_bwd_dkdv_tm_kernel(const __nv_bfloat16* __restrict__ kg, const __nv_bfloat16* __restrict__ vg,
                            const __grid_constant__ CUtensorMap map_q,
                            const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                            const float* __restrict__ delta, __nv_bfloat16* __restrict__ dk,
                            __nv_bfloat16* __restrict__ dv, long long ld, const float2* __restrict__ rope,
                            long long pos0, int S, int H, float scale, float scale_log2) {
  // TS > 0: the Q/dO ring holds TS one-step (QSTEP-query) stages instead of
  // KV_NS whole 128-query tiles (same shared memory), so a stage is released
  // and refilled every step and the loads run TS-1 steps ahead.
  using L = std::conditional_t<(TS > 0), DkdvTsSmem<D, (TS > 0 ? TS : 1)>, DkdvTmSmem<D>>;
  constexpr int NC = L::NC;
  constexpr int NS = TS > 0 ? TS : KV_NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_ready = bars + 0;
  uint64_t* in_full = bars + 1;        // [NS]
  uint64_t* in_empty = in_full + NS;   // [NS]
  uint64_t* s_full = in_empty + NS;    // [2]
  uint64_t* p_ready = s_full + 2;      // [2]  (SPLIT: P^T written; else P^T and dS^T)
  uint64_t* fin = p_ready + 2;
  uint64_t* ds_ready = fin + 1;        // [2]  SPLIT: dS^T written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ds_ready + 2);
  constexpr int CW = 32 * 4 * WPQ;
  constexpr int COLS = QSTEP / WPQ;  // query columns per compute warp per step

  const int n_tiles = S / TILE;
  const int kt = blockIdx.x;  // key tile
  const int hh = blockIdx.y;
  // rank in the 1-D cluster of 2 = blockIdx.x & 1 (rank 1 holds the upper key tile); derived from
  // blockIdx (not %cluster_ctarank) so ptxas keeps the loop state uniform
  const uint32_t crank = CL2 ? (blockIdx.x & 1u) : 0u;
  const int q_first = kt - static_cast<int>(crank);          // first query tile walked
  const int n_q = n_tiles - q_first;
  const int n_g = n_q * (TILE / QSTEP);
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_do);
    dev::mbar_init(kv_ready, CW);
    for (int s2 = 0; s2 < NS; ++s2) {
      dev::mbar_init(&in_full[s2], 1);
      dev::mbar_init(&in_empty[s2], CL2 ? 2 : 1);  // CL2: both CTAs' MMAs release a stage
    }
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&p_ready[s2], QH ? CW / 2 : CW);   // QH: queries [0,16) of the step
      dev::mbar_init(&ds_ready[s2], QH ? CW / 2 : CW);  // QH: queries [16,32); SPLIT: dS^T written
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  if (CL2)
    dev::cluster_sync();  // the peer's barriers exist before its first multicast lands here
  else
    __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dv = tmem, t_dk = tmem + 128, t_k = tmem + 256, t_v = tmem + 320;
  auto buf = [&](int b) { return tmem + 384 + 64 * b; };

  MEMO_PROF(__shared__ volatile long long pf_issue[4];)
  if (warp == 0) {
    if (lane == 0) {
      MEMO_PROF(long long pe_acc = 0;)
      if constexpr (TS > 0) {
        for (int g = 0; g < n_g; ++g) {
          const int st = g % NS;
          const int q0 = (q_first + (g >> 2)) * TILE + (g & 3) * QSTEP;  // first query of the step
          dev::mbar_wait(&in_empty[st], ((g / NS) & 1) ^ 1);
          dev::mbar_expect_tx(&in_full[st], 2 * L::STAGE_BYTES + 2 * QSTEP * 4);
          for (int c = CL2 ? static_cast<int>(crank) : 0; c < (CL2 ? static_cast<int>(crank) + 1 : NC); ++c) {
            if (CL2) {  // this CTA's 64-column chunk of the step's Q and dO slices, to both CTAs
              dev::tma_load_2d_mc(smem + L::RQ_OFF + st * L::STAGE_BYTES + c * L::CH_BYTES, &map_q, &in_full[st],
                                  hh * D + c * 64, q0, 0x3);
              dev::tma_load_2d_mc(smem + L::RD_OFF + st * L::STAGE_BYTES + c * L::CH_BYTES, &map_do, &in_full[st],
                                  hh * D + c * 64, q0, 0x3);
              continue;
            }
            dev::tma_load_2d(smem + L::RQ_OFF + st * L::STAGE_BYTES + c * L::CH_BYTES, &map_q, &in_full[st],
                             hh * D + c * 64, q0);
            dev::tma_load_2d(smem + L::RD_OFF + st * L::STAGE_BYTES + c * L::CH_BYTES, &map_do, &in_full[st],
                             hh * D + c * 64, q0);
          }
          float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF + st * 256);
          const long long off = static_cast<long long>(hh) * S + q0;
          dev::bulk_load(vec, lse2 + off, QSTEP * 4, &in_full[st]);
          dev::bulk_load(vec + 32, delta + off, QSTEP * 4, &in_full[st]);
        }
      } else
      for (int i = 0; i < n_q; ++i) {
        const int qt = q_first + i, st = i % NS;
        MEMO_PROF(long long pe = clock64();)
        dev::mbar_wait(&in_empty[st], ((i / NS) & 1) ^ 1);
        MEMO_PROF(if (i >= NS) pe_acc += clock64() - pe;)
        dev::mbar_expect_tx(&in_full[st], 2 * L::TILE_BYTES + 1024);
        MEMO_PROF(pf_issue[st] = clock64();)
        if (CL2 && !CLNOMC) {  // half of Q_qt and dO_qt, to both CTAs (CLNOMC: ablation, each loads all)
          if (NC == 2) {  // D = 128: this CTA's 64-column chunk of each
            const int c = static_cast<int>(crank);
            dev::tma_load_2d_mc(smem + L::RQ_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_q, &in_full[st],
                                hh * D + c * 64, qt * TILE, 0x3);
            dev::tma_load_2d_mc(smem + L::RD_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_do, &in_full[st],
                                hh * D + c * 64, qt * TILE, 0x3);
          } else if (crank == 0) {  // D = 64: one CTA loads Q, the other dO
            dev::tma_load_2d_mc(smem + L::RQ_OFF + st * L::TILE_BYTES, &map_q, &in_full[st], hh * D, qt * TILE,
                                0x3);
          } else {
            dev::tma_load_2d_mc(smem + L::RD_OFF + st * L::TILE_BYTES, &map_do, &in_full[st], hh * D, qt * TILE,
                                0x3);
          }
        } else
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::RQ_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_q, &in_full[st],
                           hh * D + c * 64, qt * TILE);
          dev::tma_load_2d(smem + L::RD_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_do, &in_full[st],
                           hh * D + c * 64, qt * TILE);
        }
        float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF + st * 1024);
        const long long off = static_cast<long long>(hh) * S + qt * TILE;
        dev::bulk_load(vec, lse2 + off, 512, &in_full[st]);
        dev::bulk_load(vec + 128, delta + off, 512, &in_full[st]);
      }
      if (CL2) {  // producer tail: the peer's releases of the last stages land here asynchronously
        const int n_fill = TS > 0 ? n_g : n_q;
        for (int i = n_fill; i < n_fill + NS; ++i) dev::mbar_wait(&in_empty[i % NS], ((i / NS) & 1) ^ 1);
      }
      MEMO_PROF(atomicAdd(&g_dkdv_prof[14], static_cast<unsigned long long>(pe_acc));)
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, QSTEP, false, false);
      constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
      dev::mbar_wait_w(kv_ready, 0);
      dev::tc_fence_after();
      MEMO_PROF(long long pf_acc[16] = {};)
      auto issue_sd = [&](int g) {
        const int i = g >> 2, qq = g & 3, b = g & 1;
        const int st = TS > 0 ? g % NS : i % NS;
        if constexpr (TS > 0) {
          dev::mbar_wait_w(&in_full[st], (g / NS) & 1);
          dev::tc_fence_after();
        } else if (qq == 0) {
          MEMO_PROF(long long prof_b = clock64();)
          dev::mbar_wait_w(&in_full[st], (i / NS) & 1);
          MEMO_PROF({  // per-CTA register sums, one atomic each at the end (no per-step atomics)
            const long long w = clock64() - prof_b;
            pf_acc[0] += w;
            if (i == 0) pf_acc[8] += w;  // first tile of the CTA
            if (i > 0 && w > 200) {
              pf_acc[9] += w;
              pf_acc[10] += 1;
              pf_acc[12] += clock64() - pf_issue[st];
            }
            if (i > 0) pf_acc[11] += 1;
          })
          dev::tc_fence_after();
        }
        if constexpr (TS > 0) {
          const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::RQ_OFF + st * L::STAGE_BYTES));
          const uint64_t dod = kmajor_base(dev::smem_u32(smem + L::RD_OFF + st * L::STAGE_BYTES));
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            dev::mma_bf16_ts_w(buf(b), t_k + kk * 8, kmajor_step_c<L::CH_BYTES>(qd, kk), idesc_s, kk > 0);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            dev::mma_bf16_ts_w(buf(b) + 32, t_v + kk * 8, kmajor_step_c<L::CH_BYTES>(dod, kk), idesc_s, kk > 0);
        } else {
        const uint32_t roff = qq * QSTEP * 128;  // 32 rows of 128 B inside every 64-col chunk
        const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::RQ_OFF + st * L::TILE_BYTES) + roff);
        const uint64_t dod = kmajor_base(dev::smem_u32(smem + L::RD_OFF + st * L::TILE_BYTES) + roff);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ts_w(buf(b), t_k + kk * 8, kmajor_step(qd, kk), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ts_w(buf(b) + 32, t_v + kk * 8, kmajor_step(dod, kk), idesc_s, kk > 0);
        }
        dev::mma_commit_w(&s_full[b]);
      };
      MEMO_PROF(long long prof_s = clock64();)
      issue_sd(0);
      for (int g = 0; g < n_g; ++g) {
        if (g + 1 < n_g) issue_sd(g + 1);
        const int i = g >> 2, qq = g & 3, b = g & 1;
        const int st = TS > 0 ? g % NS : i % NS;
        MEMO_PROF(long long prof_a = clock64();)
        dev::mbar_wait_w(&p_ready[b], (g >> 1) & 1);
        MEMO_PROF(pf_acc[1] += clock64() - prof_a;)
        dev::tc_fence_after();
        const uint32_t roff = TS > 0 ? 0u : qq * QSTEP * 128;
        const uint32_t sbytes = TS > 0 ? L::STAGE_BYTES : L::TILE_BYTES;
        const uint64_t qm = mnmajor_base_c<L::CH_BYTES>(dev::smem_u32(smem + L::RQ_OFF + st * sbytes) + roff);
        const uint64_t dom = mnmajor_base_c<L::CH_BYTES>(dev::smem_u32(smem + L::RD_OFF + st * sbytes) + roff);
        if constexpr (QH) {  // one query half at a time: dV then dK per 16-query k-step
#pragma unroll
          for (int kk = 0; kk < QSTEP / 16; ++kk) {
            if (kk > 0) {
              dev::mbar_wait_w(&ds_ready[b], (g >> 1) & 1);
              dev::tc_fence_after();
            }
            dev::mma_bf16_ts_w(t_dv, buf(b) + 16 * kk, mnmajor_step(dom, kk), idesc_g, (g | kk) != 0);
            dev::mma_bf16_ts_w(t_dk, buf(b) + 32 + 16 * kk, mnmajor_step(qm, kk), idesc_g, (g | kk) != 0);
          }
        } else {
#pragma unroll
        for (int kk = 0; kk < QSTEP / 16; ++kk)
          dev::mma_bf16_ts_w(t_dv, buf(b) + (WPQ == 4 ? 8 : 16) * kk, mnmajor_step(dom, kk), idesc_g, (g | kk) != 0);
        if constexpr (SPLIT) {  // dV(g) above overlaps the dS^T math of the compute warps
          dev::mbar_wait_w(&ds_ready[b], (g >> 1) & 1);
          dev::tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < QSTEP / 16; ++kk)
          dev::mma_bf16_ts_w(t_dk, buf(b) + 32 + (WPQ == 4 ? 8 : 16) * kk, mnmajor_step(qm, kk), idesc_g,
                             (g | kk) != 0);
        }
        if (TS > 0 || qq == 3) {
          if (CL2)
            dev::mma_commit_mc_w(&in_empty[st], 0x3);  // the stage holds both CTAs' chunks
          else
            dev::mma_commit_w(&in_empty[st]);
        }
      }
      dev::mma_commit_w(fin);
      MEMO_PROF(if (lane == 0) {
        pf_acc[5] += clock64() - prof_s;
        pf_acc[4] += n_g;
        for (int k = 0; k < 16; ++k)
          if (k != 2 && k != 3 && k != 6 && k != 7 && k != 14)
            atomicAdd(&g_dkdv_prof[k], static_cast<unsigned long long>(pf_acc[k]));
      })
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int ch = (warp - 4) >> 2;  // COLS-query slice of each 32-query step
    const int r = q4 * 32 + lane;    // key row in tile
    const int kidx = kt * TILE + r;
    const uint32_t lane_off = (q4 * 32) << 16;
    const long long hcols = static_cast<long long>(H) * D;
    // K (ch 0) / V (ch 1) row r -> TMEM A operand
    if (ch < 2) row_to_tmem<D>((ch == 0 ? kg : vg) + kidx * hcols + hh * D, (ch == 0 ? t_k : t_v) + lane_off);
    dev::tmem_st_wait();
    dev::tc_fence_before();
    dev::mbar_arrive(kv_ready);
    MEMO_PROF(long long cp_acc[8] = {};)
    // CL2: the upper key tile's first query tile (shared with the lower one) is
    // fully masked: P^T = dS^T = 0, peeled off so the main loop has no branch
    const int g_start = CL2 ? static_cast<int>(crank) * (TILE / QSTEP) : 0;
    for (int g = 0; g < g_start; ++g) {
      static_assert(!CL2 || (COLS == 16 && !SPLIT), "CL2: the default compute layout only");
      const int b = g & 1;
      dev::mbar_wait(&s_full[b], (g >> 1) & 1);
      dev::tc_fence_after();
      uint32_t z[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) z[e] = 0u;
      dev::tmem_st8(buf(b) + lane_off + 16 * ch, z);
      dev::tmem_st8(buf(b) + lane_off + 32 + 16 * ch, z);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_ready[b]);
    }
    for (int g = g_start; g < n_g; ++g) {
      const int i = g >> 2, qq = g & 3, b = g & 1;
      const int st = TS > 0 ? g % NS : i % NS;
      const bool diag = i == static_cast<int>(crank);
      if (TS > 0 || qq == 0) dev::mbar_wait(&in_full[st], TS > 0 ? (g / NS) & 1 : (i / NS) & 1);
      const uint32_t l2 = TS > 0 ? dev::smem_u32(smem + L::VEC_OFF + st * 256) + (COLS * ch) * 4
                                 : dev::smem_u32(smem + L::VEC_OFF + st * 1024) + (qq * QSTEP + COLS * ch) * 4;
      const uint32_t dl = l2 + (TS > 0 ? 128 : 512);
      // lse2 / delta of this step's columns, loaded before the S/dP wait so the
      // shared-memory latency is off the critical path
      float4 lvv[COLS / 4], dvv[COLS / 4];
#pragma unroll
      for (int j4 = 0; j4 < COLS / 4; ++j4) {
        lvv[j4] = dev::lds_f4(l2 + 16 * j4);
        dvv[j4] = dev::lds_f4(dl + 16 * j4);
      }
      MEMO_PROF(long long prof_t0 = clock64();)
      dev::mbar_wait(&s_full[b], (g >> 1) & 1);
      MEMO_PROF(long long prof_t1 = clock64(); cp_acc[2] += prof_t1 - prof_t0;)
      dev::tc_fence_after();
      uint32_t sr[COLS], dr[COLS];
      if constexpr (COLS == 16) {
        dev::tmem_ld16(buf(b) + lane_off + 16 * ch, sr);
        dev::tmem_ld16(buf(b) + lane_off + 32 + 16 * ch, dr);
      } else {
        dev::tmem_ld8(buf(b) + lane_off + 8 * ch, sr);
        dev::tmem_ld8(buf(b) + lane_off + 32 + 8 * ch, dr);
      }
      // COLS 16: no wait::ld, the consumers wait on the registers' scoreboard
      // (this warp's P^T/dS^T stores depend on every loaded value, and nothing
      // else reuses these columns first).  COLS 8 writes into other warps'
      // columns behind a named barrier, which needs the loads complete.
      if constexpr (COLS != 16) dev::tmem_ld_wait_regs(sr, dr);
      MEMO_PROF(cp_acc[6] += clock64() - prof_t1;)
      uint32_t pp[COLS / 2], dd[COLS / 2];
      float scl = scale_log2;
      const int turn_bar = 1 + static_cast<int>(q4) + 4 * (g & 1);  // per SMSP, alternating by step parity
      if constexpr (QH) {
        static_assert(!QH || (COLS == 16 && !SPLIT && TS == 0), "QH: the default compute layout only");
        if (QH == 2 && ch == 1) {  // ch 0's exponentials first: every exponential below depends on this barrier
          uint32_t zero;
          asm volatile("bar.sync %1, 64;\n\tmov.b32 %0, 0;" : "=r"(zero) : "r"(turn_bar) : "memory");
          scl += __uint_as_float(zero);
        }
      }
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
        for (int j4 = 0; j4 < COLS / 4; ++j4) {
          const float4 lv = lvv[j4];
          const float4 dv4 = dvv[j4];
          const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
          const float dq4[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
          float p4[4], d4[4];
#pragma unroll
          for (int e = 0; e < 4; e += 2) {  // column pairs: FFMA2 / FADD2 / FMUL2
            const uint64_t x2 = ffma2_v(f2_pack(__uint_as_float(sr[4 * j4 + e]), __uint_as_float(sr[4 * j4 + e + 1])),
                                        scl, f2_pack(lq[e], lq[e + 1]));
            float pa, pb;
            if (EMU && ((2 * j4 + (e >> 1)) % (EMU ? EMU : 1)) == EMU - 1) {
              const uint64_t e2 = exp2_fma2(x2);
              pa = f2_lo(e2);
              pb = f2_hi(e2);
            } else {
              pa = dev::ex2(f2_lo(x2));
              pb = dev::ex2(f2_hi(x2));
            }
            if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e < r) pa = 0.f;
            if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e + 1 < r) pb = 0.f;
            const uint64_t d2 = fmul2(f2_pack(pa, pb),
                                      fadd2(f2_pack(__uint_as_float(dr[4 * j4 + e]), __uint_as_float(dr[4 * j4 + e + 1])),
                                            f2_pack(dq4[e], dq4[e + 1])));
            p4[e] = pa;
            p4[e + 1] = pb;
            d4[e] = f2_lo(d2);
            d4[e + 1] = f2_hi(d2);
          }
          pp[2 * j4] = dev::pack_bf16(p4[0], p4[1]);
          pp[2 * j4 + 1] = dev::pack_bf16(p4[2], p4[3]);
          dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
          dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
        }
      };
      if constexpr (SPLIT && COLS == 16) {
        // P^T first (its own barrier, so dV(g) can start), then dS^T.
        float pf[COLS];
        auto pbody = [&](auto diag_tag) {
          constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
          for (int j4 = 0; j4 < COLS / 4; ++j4) {
            const float4 lv = lvv[j4];
            const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const uint64_t x2 = ffma2_v(f2_pack(__uint_as_float(sr[4 * j4 + e]), __uint_as_float(sr[4 * j4 + e + 1])),
                                          scale_log2, f2_pack(lq[e], lq[e + 1]));
              float pa, pb;
              if (EMU && ((2 * j4 + (e >> 1)) % (EMU ? EMU : 1)) == EMU - 1) {
                const uint64_t e2 = exp2_fma2(x2);
                pa = f2_lo(e2);
                pb = f2_hi(e2);
              } else {
                pa = dev::ex2(f2_lo(x2));
                pb = dev::ex2(f2_hi(x2));
              }
              if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e < r) pa = 0.f;
              if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e + 1 < r) pb = 0.f;
              pf[4 * j4 + e] = pa;
              pf[4 * j4 + e + 1] = pb;
            }
            pp[2 * j4] = dev::pack_bf16(pf[4 * j4], pf[4 * j4 + 1]);
            pp[2 * j4 + 1] = dev::pack_bf16(pf[4 * j4 + 2], pf[4 * j4 + 3]);
          }
        };
        if (diag)
          pbody(std::true_type{});
        else
          pbody(std::false_type{});
        dev::tmem_st8(buf(b) + lane_off + 16 * ch, pp);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&p_ready[b]);
#pragma unroll
        for (int j4 = 0; j4 < COLS / 4; ++j4) {
          const float4 dv4 = dvv[j4];
          const float dq4[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
          float d4[4];
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const uint64_t d2 = fmul2(f2_pack(pf[4 * j4 + e], pf[4 * j4 + e + 1]),
                                      fadd2(f2_pack(__uint_as_float(dr[4 * j4 + e]), __uint_as_float(dr[4 * j4 + e + 1])),
                                            f2_pack(dq4[e], dq4[e + 1])));
            d4[e] = f2_lo(d2);
            d4[e + 1] = f2_hi(d2);
          }
          dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
          dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
        }
        dev::tmem_st8(buf(b) + lane_off + 32 + 16 * ch, dd);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&ds_ready[b]);
        continue;
      }
      if (diag)
        body(std::true_type{});
      else
        body(std::false_type{});
      if constexpr (QH) {
        if (QH == 2 && ch == 0)  // after its last exponential (the packed P depends on all of them)
          asm volatile("bar.arrive %0, 64;" ::"r"(turn_bar), "r"(pp[COLS / 2 - 1]) : "memory");
      }
      if constexpr (COLS == 16) {
        // packed bf16 stays inside this warp's own 16-column slice
        dev::tmem_st8(buf(b) + lane_off + 16 * ch, pp);
        dev::tmem_st8(buf(b) + lane_off + 32 + 16 * ch, dd);
      } else {
        // compacted: queries 8ch..8ch+7 -> cols 4ch..4ch+3, contiguous per 16-query
        // k-step.  Those columns belong to another warp's slice, so every warp of
        // this lane quarter must have finished its loads first.
        named_bar(1 + q4, 128);
        dev::tmem_st4(buf(b) + lane_off + 4 * ch, pp);
        dev::tmem_st4(buf(b) + lane_off + 32 + 4 * ch, dd);
      }
      MEMO_PROF(long long prof_t2 = clock64();)
      dev::tmem_st_wait();
      MEMO_PROF(cp_acc[7] += clock64() - prof_t2;)
      dev::tc_fence_before();
      dev::mbar_arrive(QH && ch == 1 ? &ds_ready[b] : &p_ready[b]);
      MEMO_PROF(cp_acc[3] += clock64() - prof_t1;)
    }
    MEMO_PROF(if (warp == 4 && lane == 0) for (int k2 : {2, 3, 6, 7})
                atomicAdd(&g_dkdv_prof[k2], static_cast<unsigned long long>(cp_acc[k2]));)
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    __nv_bfloat16* dvrow = dv + static_cast<long long>(kidx) * ld + hh * D;
    __nv_bfloat16* dkrow = dk + static_cast<long long>(kidx) * ld + hh * D;
#pragma unroll 1
    for (int c = ch; c < D / 32; c += WPQ) {  // 32-column chunks of dV/dK spread over the quarter's warps
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dv + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dvrow + c * 32, x, 1.f, nullptr);
      dev::tmem_ld32(t_dk + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dkrow + c * 32, x, scale, rope ? rope + (pos0 + kidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  if (CL2)
    dev::cluster_sync();  // no multicast or remote release still targets this CTA
  else
    __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

#ifdef MEMO_ATTN_ABLATIONS  // 16-query and decoupled P/dS dK/dV (ablation build only)
// ------------------------------------------------------------ dK/dV, 16-query steps
// Ablation: bitwise equal, 268 vs 206 ms at 128K (M128 N16 MMAs run at 79 %).
// Same math and operands as attn_bwd_dkdv_tm_kernel<D, 2>, with the pipeline cut
// finer: 16-query steps and FOUR S^T/dP^T buffers in the same 128 TMEM columns
//   [0,128) dV | [128,256) dK | [256,320) K | [320,384) V | [384 + 32b, +32) buf b
//   buf: S^T [0,16) | dP^T [16,32); P^T packed into [0,8), dS^T into [16,24)
// so the MMA warp queues S/dP three steps ahead of the dV/dK that wait for the
// compute warps (768 tensor cycles of slack instead of 512).  The compute warps
// form two groups of four (one per TMEM lane quarter) taking alternate steps,
// each warp all 16 columns of its rows, so a warp has two steps' time per step.
constexpr int Q16 = 16;

template <int D>
__global__ void __launch_bounds__(32 * 12, 1)
    attn_bwd_dkdv_q16_kernel(const __nv_bfloat16* __restrict__ kg, const __nv_bfloat16* __restrict__ vg,
                             const __grid_constant__ CUtensorMap map_q,
                             const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                             const float* __restrict__ delta, __nv_bfloat16* __restrict__ dk,
                             __nv_bfloat16* __restrict__ dv, long long ld, const float2* __restrict__ rope,
                             long long pos0, int S, int H, float scale, float scale_log2) {
  using L = DkdvTmSmem<D>;
  constexpr int NC = L::NC;
  constexpr int NS = KV_NS;
  constexpr int NB = 4;                // S^T/dP^T buffers
  constexpr int SPT = TILE / Q16;      // steps per query tile
  constexpr int AHEAD = NB - 1;        // S/dP issued this many steps ahead
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_ready = bars + 0;
  uint64_t* in_full = bars + 1;        // [NS]
  uint64_t* in_empty = in_full + NS;   // [NS]
  uint64_t* s_full = in_empty + NS;    // [NB]
  uint64_t* p_ready = s_full + NB;     // [NB]
  uint64_t* fin = p_ready + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);

  const int n_tiles = S / TILE;
  const int kt = blockIdx.x;  // key tile
  const int hh = blockIdx.y;
  const int n_q = n_tiles - kt;
  const int n_g = n_q * SPT;
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_do);
    dev::mbar_init(kv_ready, 256);
    for (int s2 = 0; s2 < NS; ++s2) {
      dev::mbar_init(&in_full[s2], 1);
      dev::mbar_init(&in_empty[s2], 1);
    }
    for (int s2 = 0; s2 < NB; ++s2) {
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&p_ready[s2], 128);
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dv = tmem, t_dk = tmem + 128, t_k = tmem + 256, t_v = tmem + 320;
  auto buf = [&](int b) { return tmem + 384 + 32 * b; };

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n_q; ++i) {
        const int qt = kt + i, st = i % NS;
        dev::mbar_wait(&in_empty[st], ((i / NS) & 1) ^ 1);
        dev::mbar_expect_tx(&in_full[st], 2 * L::TILE_BYTES + 1024);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::RQ_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_q, &in_full[st],
                           hh * D + c * 64, qt * TILE);
          dev::tma_load_2d(smem + L::RD_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_do, &in_full[st],
                           hh * D + c * 64, qt * TILE);
        }
        float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF + st * 1024);
        const long long off = static_cast<long long>(hh) * S + qt * TILE;
        dev::bulk_load(vec, lse2 + off, 512, &in_full[st]);
        dev::bulk_load(vec + 128, delta + off, 512, &in_full[st]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, Q16, false, false);
    constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
    dev::mbar_wait_w(kv_ready, 0);
    dev::tc_fence_after();
    auto issue_sd = [&](int g) {
      const int i = g / SPT, qq = g % SPT, b = g % NB, st = i % NS;
      if (qq == 0) {
        dev::mbar_wait_w(&in_full[st], (i / NS) & 1);
        dev::tc_fence_after();
      }
      const uint32_t roff = qq * Q16 * 128;  // 16 rows of 128 B inside every 64-col chunk
      const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::RQ_OFF + st * L::TILE_BYTES) + roff);
      const uint64_t dod = kmajor_base(dev::smem_u32(smem + L::RD_OFF + st * L::TILE_BYTES) + roff);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        dev::mma_bf16_ts_w(buf(b), t_k + kk * 8, kmajor_step(qd, kk), idesc_s, kk > 0);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        dev::mma_bf16_ts_w(buf(b) + 16, t_v + kk * 8, kmajor_step(dod, kk), idesc_s, kk > 0);
      dev::mma_commit_w(&s_full[b]);
    };
    for (int g = 0; g < AHEAD && g < n_g; ++g) issue_sd(g);
    for (int g = 0; g < n_g; ++g) {
      if (g + AHEAD < n_g) issue_sd(g + AHEAD);  // into the buffer dK(g-1) read: in order behind it
      const int i = g / SPT, qq = g % SPT, b = g % NB, st = i % NS;
      dev::mbar_wait_w(&p_ready[b], (g / NB) & 1);
      dev::tc_fence_after();
      const uint32_t roff = qq * Q16 * 128;
      const uint64_t qm = mnmajor_base_c<CHUNK_BYTES>(dev::smem_u32(smem + L::RQ_OFF + st * L::TILE_BYTES) + roff);
      const uint64_t dom = mnmajor_base_c<CHUNK_BYTES>(dev::smem_u32(smem + L::RD_OFF + st * L::TILE_BYTES) + roff);
      dev::mma_bf16_ts_w(t_dv, buf(b), dom, idesc_g, g != 0);
      dev::mma_bf16_ts_w(t_dk, buf(b) + 16, qm, idesc_g, g != 0);
      if (qq == SPT - 1) dev::mma_commit_w(&in_empty[st]);
    }
    dev::mma_commit_w(fin);
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int grp = (warp - 4) >> 2;  // this group takes steps g with g % 2 == grp
    const int r = q4 * 32 + lane;     // key row in tile
    const int kidx = kt * TILE + r;
    const uint32_t lane_off = (q4 * 32) << 16;
    const long long hcols = static_cast<long long>(H) * D;
    // K (group 0) / V (group 1) row r -> TMEM A operand
    row_to_tmem<D>((grp == 0 ? kg : vg) + kidx * hcols + hh * D, (grp == 0 ? t_k : t_v) + lane_off);
    dev::tmem_st_wait();
    dev::tc_fence_before();
    dev::mbar_arrive(kv_ready);
    for (int g = grp; g < n_g; g += 2) {
      const int i = g / SPT, qq = g % SPT, b = g % NB, st = i % NS;
      if (qq < 2) dev::mbar_wait(&in_full[st], (i / NS) & 1);
      const uint32_t l2 = dev::smem_u32(smem + L::VEC_OFF + st * 1024) + (qq * Q16) * 4;
      const uint32_t dl = l2 + 512;
      float4 lvv[4], dvv[4];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        lvv[j4] = dev::lds_f4(l2 + 16 * j4);
        dvv[j4] = dev::lds_f4(dl + 16 * j4);
      }
      dev::mbar_wait(&s_full[b], (g / NB) & 1);
      dev::tc_fence_after();
      uint32_t sr[16], dr[16];
      dev::tmem_ld16(buf(b) + lane_off, sr);
      dev::tmem_ld16(buf(b) + lane_off + 16, dr);
      // no wait::ld: the P^T/dS^T stores below depend on every loaded value
      uint32_t pp[8], dd[8];
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 lv = lvv[j4];
          const float4 dv4 = dvv[j4];
          const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
          const float dq4[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
          float p4[4], d4[4];
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const uint64_t x2 = ffma2_v(f2_pack(__uint_as_float(sr[4 * j4 + e]), __uint_as_float(sr[4 * j4 + e + 1])),
                                        scale_log2, f2_pack(lq[e], lq[e + 1]));
            float pa = dev::ex2(f2_lo(x2));
            float pb = dev::ex2(f2_hi(x2));
            if (DIAG && qq * Q16 + 4 * j4 + e < r) pa = 0.f;
            if (DIAG && qq * Q16 + 4 * j4 + e + 1 < r) pb = 0.f;
            const uint64_t d2 = fmul2(f2_pack(pa, pb),
                                      fadd2(f2_pack(__uint_as_float(dr[4 * j4 + e]), __uint_as_float(dr[4 * j4 + e + 1])),
                                            f2_pack(dq4[e], dq4[e + 1])));
            p4[e] = pa;
            p4[e + 1] = pb;
            d4[e] = f2_lo(d2);
            d4[e + 1] = f2_hi(d2);
          }
          pp[2 * j4] = dev::pack_bf16(p4[0], p4[1]);
          pp[2 * j4 + 1] = dev::pack_bf16(p4[2], p4[3]);
          dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
          dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
        }
      };
      if (i == 0)
        body(std::true_type{});
      else
        body(std::false_type{});
      dev::tmem_st8(buf(b) + lane_off, pp);
      dev::tmem_st8(buf(b) + lane_off + 16, dd);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_ready[b]);
    }
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    __nv_bfloat16* dvrow = dv + static_cast<long long>(kidx) * ld + hh * D;
    __nv_bfloat16* dkrow = dk + static_cast<long long>(kidx) * ld + hh * D;
#pragma unroll 1
    for (int c = grp; c < D / 32; c += 2) {  // 32-column chunks of dV/dK spread over the two groups
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dv + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dvrow + c * 32, x, 1.f, nullptr);
      dev::tmem_ld32(t_dk + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dkrow + c * 32, x, scale, rope ? rope + (pos0 + kidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------ dK/dV, decoupled P/dS
// Ablation (measured 12 % SLOWER at 128K than attn_bwd_dkdv_tm_kernel<D, 2>:
// 231-232 vs 206-207 ms, H=32, D=128, interleaved runs).  Same math and operands as attn_bwd_dkdv_tm_kernel
// (K, V resident in TMEM as the A operands of S^T = K Q^T and dP^T = V dO^T,
// 32-query steps, two compute warps per TMEM lane quarter), but P^T / dS^T no
// longer overwrite their S^T / dP^T columns: they go to one of two separate
// 32-column regions, and S^T / dP^T use a single buffer that is released as
// soon as the compute warps have loaded it into registers.  The tensor pipe
// therefore computes S^T(g+1), dP^T(g+1) while the compute warps still work on
// step g, and the loop that limited the old layout -- P/dS(g) -> dV, dK(g) ->
// S, dP(g+2) into the freed buffer -> compute(g+2) -- is gone:
//   [0,128) dV | [128,256) dK | [256,320) K | [320,384) V | [384,416) S^T |
//   [416,448) dP^T | [448+32b, +16) P^T(b) | [464+32b, +16) dS^T(b), b = g % 2
// (warp ch of a quarter owns queries 16ch..16ch+15: 8 packed columns of each).
template <int D>
__global__ void __launch_bounds__(32 * 12, 1)
    attn_bwd_dkdv_tm2_kernel(const __nv_bfloat16* __restrict__ kg, const __nv_bfloat16* __restrict__ vg,
                             const __grid_constant__ CUtensorMap map_q,
                             const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                             const float* __restrict__ delta, __nv_bfloat16* __restrict__ dk,
                             __nv_bfloat16* __restrict__ dv, long long ld, const float2* __restrict__ rope,
                             long long pos0, int S, int H, float scale, float scale_log2) {
  using L = DkdvTmSmem<D>;
  constexpr int NC = L::NC;
  constexpr int NS = KV_NS;
  constexpr int CW = 32 * 8;   // compute threads
  constexpr int COLS = 16;     // query columns per compute warp per step
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_ready = bars + 0;
  uint64_t* in_full = bars + 1;        // [NS]
  uint64_t* in_empty = in_full + NS;   // [NS]
  uint64_t* s_full = in_empty + NS;    // S^T(g), dP^T(g) computed
  uint64_t* sd_free = s_full + 1;      // ... and loaded by every compute thread
  uint64_t* p_ready = sd_free + 1;     // [2] P^T / dS^T of region b written
  uint64_t* pds_free = p_ready + 2;    // [2] dV / dK MMAs done with region b
  uint64_t* fin = pds_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);

  const int n_tiles = S / TILE;
  const int kt = blockIdx.x;  // key tile
  const int hh = blockIdx.y;
  const int n_q = n_tiles - kt;
  const int n_g = n_q * (TILE / QSTEP);
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_do);
    dev::mbar_init(kv_ready, CW);
    for (int s2 = 0; s2 < NS; ++s2) {
      dev::mbar_init(&in_full[s2], 1);
      dev::mbar_init(&in_empty[s2], 1);
    }
    dev::mbar_init(s_full, 1);
    dev::mbar_init(sd_free, CW);
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&p_ready[s2], CW);
      dev::mbar_init(&pds_free[s2], 1);
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dv = tmem, t_dk = tmem + 128, t_k = tmem + 256, t_v = tmem + 320;
  const uint32_t t_s = tmem + 384, t_dp = tmem + 416;
  auto region = [&](int b) { return tmem + 448 + 32 * b; };

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n_q; ++i) {
        const int qt = kt + i, st = i % NS;
        dev::mbar_wait(&in_empty[st], ((i / NS) & 1) ^ 1);
        dev::mbar_expect_tx(&in_full[st], 2 * L::TILE_BYTES + 1024);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::RQ_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_q, &in_full[st],
                           hh * D + c * 64, qt * TILE);
          dev::tma_load_2d(smem + L::RD_OFF + st * L::TILE_BYTES + c * CHUNK_BYTES, &map_do, &in_full[st],
                           hh * D + c * 64, qt * TILE);
        }
        float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF + st * 1024);
        const long long off = static_cast<long long>(hh) * S + qt * TILE;
        dev::bulk_load(vec, lse2 + off, 512, &in_full[st]);
        dev::bulk_load(vec + 128, delta + off, 512, &in_full[st]);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, QSTEP, false, false);
      constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
      dev::mbar_wait_w(kv_ready, 0);
      dev::tc_fence_after();
      auto issue_sd = [&](int g) {
        const int i = g >> 2, qq = g & 3, st = i % NS;
        if (qq == 0) {
          dev::mbar_wait_w(&in_full[st], (i / NS) & 1);
          dev::tc_fence_after();
        }
        const uint32_t roff = qq * QSTEP * 128;  // 32 rows of 128 B inside every 64-col chunk
        const uint64_t qd = kmajor_base(dev::smem_u32(smem + L::RQ_OFF + st * L::TILE_BYTES) + roff);
        const uint64_t dod = kmajor_base(dev::smem_u32(smem + L::RD_OFF + st * L::TILE_BYTES) + roff);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ts_w(t_s, t_k + kk * 8, kmajor_step(qd, kk), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ts_w(t_dp, t_v + kk * 8, kmajor_step(dod, kk), idesc_s, kk > 0);
        dev::mma_commit_w(s_full);
      };
      issue_sd(0);
      for (int g = 0; g < n_g; ++g) {
        const int i = g >> 2, qq = g & 3, st = i % NS, b = g & 1;
        if (g + 1 < n_g) {
          dev::mbar_wait_w(sd_free, g & 1);  // S^T(g), dP^T(g) are in registers
          dev::tc_fence_after();
          issue_sd(g + 1);
        }
        dev::mbar_wait_w(&p_ready[b], (g >> 1) & 1);
        dev::tc_fence_after();
        const uint32_t roff = qq * QSTEP * 128;
        const uint64_t qm = mnmajor_base(dev::smem_u32(smem + L::RQ_OFF + st * L::TILE_BYTES) + roff);
        const uint64_t dom = mnmajor_base(dev::smem_u32(smem + L::RD_OFF + st * L::TILE_BYTES) + roff);
#pragma unroll
        for (int kk = 0; kk < QSTEP / 16; ++kk)
          dev::mma_bf16_ts_w(t_dv, region(b) + 8 * kk, mnmajor_step(dom, kk), idesc_g, (g | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < QSTEP / 16; ++kk)
          dev::mma_bf16_ts_w(t_dk, region(b) + 16 + 8 * kk, mnmajor_step(qm, kk), idesc_g, (g | kk) != 0);
        dev::mma_commit_w(&pds_free[b]);
        if (qq == 3) dev::mma_commit_w(&in_empty[st]);
      }
      dev::mma_commit_w(fin);
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int ch = (warp - 4) >> 2;  // 16-query slice of each 32-query step
    const int r = q4 * 32 + lane;    // key row in tile
    const int kidx = kt * TILE + r;
    const uint32_t lane_off = (q4 * 32) << 16;
    const long long hcols = static_cast<long long>(H) * D;
    // K (ch 0) / V (ch 1) row r -> TMEM A operand
    row_to_tmem<D>((ch == 0 ? kg : vg) + kidx * hcols + hh * D, (ch == 0 ? t_k : t_v) + lane_off);
    dev::tmem_st_wait();
    dev::tc_fence_before();
    dev::mbar_arrive(kv_ready);
    for (int g = 0; g < n_g; ++g) {
      const int i = g >> 2, qq = g & 3, st = i % NS, b = g & 1;
      const bool diag = i == 0;
      if (qq == 0) dev::mbar_wait(&in_full[st], (i / NS) & 1);
      const uint32_t l2 = dev::smem_u32(smem + L::VEC_OFF + st * 1024) + (qq * QSTEP + COLS * ch) * 4;
      const uint32_t dl = l2 + 512;
      // lse2 / delta of this step's columns, loaded before the S/dP wait
      float4 lvv[COLS / 4], dvv[COLS / 4];
#pragma unroll
      for (int j4 = 0; j4 < COLS / 4; ++j4) {
        lvv[j4] = dev::lds_f4(l2 + 16 * j4);
        dvv[j4] = dev::lds_f4(dl + 16 * j4);
      }
      dev::mbar_wait(s_full, g & 1);
      dev::tc_fence_after();
      uint32_t sr[COLS], dr[COLS];
      dev::tmem_ld16(t_s + lane_off + 16 * ch, sr);
      dev::tmem_ld16(t_dp + lane_off + 16 * ch, dr);
      dev::tmem_ld_wait_regs(sr, dr);
      dev::tc_fence_before();
      dev::mbar_arrive(sd_free);  // the tensor pipe may overwrite S^T / dP^T now
      uint32_t pp[COLS / 2], dd[COLS / 2];
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
        for (int j4 = 0; j4 < COLS / 4; ++j4) {
          const float4 lv = lvv[j4];
          const float4 dv4 = dvv[j4];
          const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
          const float dq4[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
          float p4[4], d4[4];
#pragma unroll
          for (int e = 0; e < 4; e += 2) {  // column pairs: FFMA2 / FADD2 / FMUL2
            const uint64_t x2 = ffma2_v(f2_pack(__uint_as_float(sr[4 * j4 + e]), __uint_as_float(sr[4 * j4 + e + 1])),
                                        scale_log2, f2_pack(lq[e], lq[e + 1]));
            float pa = dev::ex2(f2_lo(x2));
            float pb = dev::ex2(f2_hi(x2));
            if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e < r) pa = 0.f;
            if (DIAG && qq * QSTEP + COLS * ch + 4 * j4 + e + 1 < r) pb = 0.f;
            const uint64_t d2 = fmul2(f2_pack(pa, pb),
                                      fadd2(f2_pack(__uint_as_float(dr[4 * j4 + e]), __uint_as_float(dr[4 * j4 + e + 1])),
                                            f2_pack(dq4[e], dq4[e + 1])));
            p4[e] = pa;
            p4[e + 1] = pb;
            d4[e] = f2_lo(d2);
            d4[e + 1] = f2_hi(d2);
          }
          pp[2 * j4] = dev::pack_bf16(p4[0], p4[1]);
          pp[2 * j4 + 1] = dev::pack_bf16(p4[2], p4[3]);
          dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
          dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
        }
      };
      if (diag)
        body(std::true_type{});
      else
        body(std::false_type{});
      if (g >= 2) {  // region b was last read by dV / dK of step g - 2
        dev::mbar_wait(&pds_free[b], ((g - 2) >> 1) & 1);
        dev::tc_fence_after();
      }
      dev::tmem_st8(region(b) + lane_off + 8 * ch, pp);
      dev::tmem_st8(region(b) + lane_off + 16 + 8 * ch, dd);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_ready[b]);
    }
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    __nv_bfloat16* dvrow = dv + static_cast<long long>(kidx) * ld + hh * D;
    __nv_bfloat16* dkrow = dk + static_cast<long long>(kidx) * ld + hh * D;
#pragma unroll 1
    for (int c = ch; c < D / 32; c += 2) {  // 32-column chunks of dV/dK spread over the quarter's warps
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dv + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dvrow + c * 32, x, 1.f, nullptr);
      dev::tmem_ld32(t_dk + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dkrow + c * 32, x, scale, rope ? rope + (pos0 + kidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}


// AT: Q and dO live in TMEM (A operands) instead of shared memory.
#endif  // MEMO_ATTN_ABLATIONS

// CL2: CTA pairs (clusters of 2) on query tiles qt+1, qt of one head share
// each K/V tile by TMA multicast: every CTA loads one 64-column chunk of K_j
// and of V_j for both, halving the L2->SM traffic (1.1 TB per 128K launch
// without it).  A stage is refilled once both CTAs have released it; the lower
// tile's extra key tile (qt+1) is fully masked and contributes dS = 0.
template <int D, bool AT, bool CL2 = false>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dout,
                       const __grid_constant__ CUtensorMap map_q,
                       const __grid_constant__ CUtensorMap map_do,
                       const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_v, const float* __restrict__ lse2,
                       const float* __restrict__ delta, __nv_bfloat16* __restrict__ dq, long long ld,
                       const float2* __restrict__ rope, long long pos0, int S, int H, float scale,
                       float scale_log2) {
  using L = BwdSmem<D>;
  constexpr int NC = L::NC;
  // With Q/dO in TMEM the A0/A1 region joins the K/V ring as a third stage.
  constexpr int NS = AT ? 3 : 2;
  auto k_off = [](int st) { return AT ? st * 2 * L::TILE_BYTES : L::R0_OFF + st * L::TILE_BYTES; };
  auto v_off = [](int st) { return AT ? st * 2 * L::TILE_BYTES + L::TILE_BYTES : L::R1_OFF + st * L::TILE_BYTES; };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* qd_ready = bars + 0;
  uint64_t* kv_full = bars + 1;   // [3]
  uint64_t* kv_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;    // [2]
  uint64_t* ds_ready = bars + 9;  // [2]
  uint64_t* fin = bars + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int n_tiles = S / TILE;
  const int qt = n_tiles - 1 - static_cast<int>(blockIdx.x);  // heavy tiles first
  const int hh = blockIdx.y;
  // rank in the 1-D cluster of 2 = blockIdx.x & 1 (rank 1 holds the lower tile); derived from
  // blockIdx (not %cluster_ctarank) so ptxas keeps the loop state uniform
  const uint32_t crank = CL2 ? (blockIdx.x & 1u) : 0u;
  const int n_kv = qt + 1 + static_cast<int>(crank);
  const int n_g = 2 * n_kv;
  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::mbar_init(qd_ready, AT ? 128 : 1);
    for (int s2 = 0; s2 < NS; ++s2) {
      dev::mbar_init(&kv_full[s2], 1);
      dev::mbar_init(&kv_empty[s2], CL2 ? 2 : 1);  // CL2: both CTAs' MMAs release a stage
    }
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&ds_ready[s2], 32 * BWD_COMPUTE_WARPS);
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  if (CL2)
    dev::cluster_sync();  // the peer's barriers exist before its first multicast lands here
  else
    __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // buffer b: S half at b*128, dP half at b*128 + 64; dQ at 256; Q, dO as A operands after it
  const uint32_t t_dq = tmem + 256, t_q = tmem + 256 + D, t_do = t_q + D / 2;

  if (warp == 0) {
    if (lane == 0) {
      if (!AT) {
        dev::mbar_expect_tx(qd_ready, 2 * L::TILE_BYTES);
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + L::A0_OFF + c * CHUNK_BYTES, &map_q, qd_ready, hh * D + c * 64, qt * TILE);
          dev::tma_load_2d(smem + L::A1_OFF + c * CHUNK_BYTES, &map_do, qd_ready, hh * D + c * 64, qt * TILE);
        }
      }
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NS;
        dev::mbar_wait(&kv_empty[st], ((j / NS) & 1) ^ 1);
        dev::mbar_expect_tx(&kv_full[st], 2 * L::TILE_BYTES);
        if (CL2) {  // half of K_j and V_j, to both CTAs
          if (NC == 2) {  // D = 128: this CTA's 64-column chunk of each
            const int c = static_cast<int>(crank);
            dev::tma_load_2d_mc(smem + k_off(st) + c * CHUNK_BYTES, &map_k, &kv_full[st], hh * D + c * 64,
                                j * TILE, 0x3);
            dev::tma_load_2d_mc(smem + v_off(st) + c * CHUNK_BYTES, &map_v, &kv_full[st], hh * D + c * 64,
                                j * TILE, 0x3);
          } else if (crank == 0) {  // D = 64: one CTA loads K, the other V
            dev::tma_load_2d_mc(smem + k_off(st), &map_k, &kv_full[st], hh * D, j * TILE, 0x3);
          } else {
            dev::tma_load_2d_mc(smem + v_off(st), &map_v, &kv_full[st], hh * D, j * TILE, 0x3);
          }
          continue;
        }
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(smem + k_off(st) + c * CHUNK_BYTES, &map_k, &kv_full[st], hh * D + c * 64,
                           j * TILE);
          dev::tma_load_2d(smem + v_off(st) + c * CHUNK_BYTES, &map_v, &kv_full[st], hh * D + c * 64,
                           j * TILE);
        }
      }
      if (CL2) {  // producer tail: the peer's releases of the last stages land here asynchronously
        for (int j = n_kv; j < n_kv + NS; ++j) dev::mbar_wait(&kv_empty[j % NS], ((j / NS) & 1) ^ 1);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, HALF, false, false);
      constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
      dev::mbar_wait_w(qd_ready, 0);
      const uint64_t qa0 = kmajor_base(dev::smem_u32(smem + L::A0_OFF));
      const uint64_t doa0 = kmajor_base(dev::smem_u32(smem + L::A1_OFF));
      auto issue_s = [&](int g) {
        const int j = g >> 1, half = g & 1, st = j % NS, b = g & 1;
        if (half == 0) {
          dev::mbar_wait_w(&kv_full[st], (j / NS) & 1);
          dev::tc_fence_after();
        }
        const uint64_t kd = kmajor_base(dev::smem_u32(smem + k_off(st)) + half * HALF_BYTES);
        const uint64_t vd = kmajor_base(dev::smem_u32(smem + v_off(st)) + half * HALF_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          if (AT)
            dev::mma_bf16_ts_w(tmem + b * 128, t_q + kk * 8, kmajor_step(kd, kk), idesc_s, kk > 0);
          else
            dev::mma_bf16_ss_w(tmem + b * 128, kmajor_step(qa0, kk), kmajor_step(kd, kk), idesc_s, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          if (AT)
            dev::mma_bf16_ts_w(tmem + b * 128 + 64, t_do + kk * 8, kmajor_step(vd, kk), idesc_s, kk > 0);
          else
            dev::mma_bf16_ss_w(tmem + b * 128 + 64, kmajor_step(doa0, kk), kmajor_step(vd, kk), idesc_s,
                             kk > 0);
        }
        dev::mma_commit_w(&s_full[b]);
      };
      issue_s(0);
      for (int g = 0; g < n_g; ++g) {
        if (g + 1 < n_g) issue_s(g + 1);
        const int j = g >> 1, half = g & 1, st = j % NS, b = g & 1;
        dev::mbar_wait_w(&ds_ready[b], (g >> 1) & 1);
        dev::tc_fence_after();
        const uint64_t km = mnmajor_base(dev::smem_u32(smem + k_off(st)) + half * HALF_BYTES);
#pragma unroll
        for (int kk = 0; kk < HALF / 16; ++kk)
          dev::mma_bf16_ts_w(t_dq, tmem + b * 128 + 32 * (kk >> 1) + 8 * (kk & 1), mnmajor_step(km, kk),
                             idesc_g, (g | kk) != 0);
        if (half == 1) {
          if (CL2)
            dev::mma_commit_mc_w(&kv_empty[st], 0x3);  // the stage holds both CTAs' chunks
          else
            dev::mma_commit_w(&kv_empty[st]);
        }
      }
      dev::mma_commit_w(fin);
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int ch = (warp - 4) >> 2;  // which 32-column chunk of each half this warp owns
    const int r = q4 * 32 + lane;
    const int qidx = qt * TILE + r;
    const uint32_t lane_off = (q4 * 32) << 16;
    const long long rowoff = static_cast<long long>(qidx) * H * D + hh * D;
    if (AT && ch == 0) {
      row_to_tmem<D>(q + rowoff, t_q + lane_off);
      row_to_tmem<D>(dout + rowoff, t_do + lane_off);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(qd_ready);
    }
    const long long vi = static_cast<long long>(hh) * S + qidx;
    const float my_lse2 = lse2[vi];
    const float my_delta = delta[vi];
    for (int g = 0; g < n_g; ++g) {
      const int j = g >> 1, half = g & 1, b = g & 1;
      const bool diag = j == qt;
      dev::mbar_wait(&s_full[b], (g >> 1) & 1);
      dev::tc_fence_after();
      const uint32_t t_s = tmem + b * 128 + lane_off, t_dp = t_s + 64;
      if (CL2 && j > qt) {  // the pair's extra key tile: fully masked, dS = 0
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        dev::tmem_st16(t_s + ch * 32, z);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&ds_ready[b]);
        continue;
      }
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
        {
          const int c = ch;
          uint32_t sr[32], dr[32];
          dev::tmem_ld32(t_s + c * 32, sr);
          dev::tmem_ld32(t_dp + c * 32, dr);
          // no wait::ld: the consumers wait on the registers' scoreboard (the dS
          // stores below depend on every loaded value, nothing reuses S/dP first)
          uint32_t dd[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {  // key pairs: FFMA2 / FADD2 / FMUL2
            const int kc = half * HALF + c * 32 + 2 * jj;
            const uint64_t x2 = ffma2(f2_pack(__uint_as_float(sr[2 * jj]), __uint_as_float(sr[2 * jj + 1])),
                                      scale_log2, my_lse2);
            float pa = dev::ex2(f2_lo(x2)), pb = dev::ex2(f2_hi(x2));
            if (DIAG && kc > r) pa = 0.f;
            if (DIAG && kc + 1 > r) pb = 0.f;
            const uint64_t d2 = fmul2(f2_pack(pa, pb),
                                      fadd2(f2_pack(__uint_as_float(dr[2 * jj]), __uint_as_float(dr[2 * jj + 1])),
                                            f2_pack(my_delta, my_delta)));
            dd[jj] = dev::pack_bf16(f2_lo(d2), f2_hi(d2));
          }
          dev::tmem_st16(t_s + c * 32, dd);  // inside this warp's own slice
        }
      };
      if (diag)
        body(std::true_type{});
      else
        body(std::false_type{});
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&ds_ready[b]);
    }
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    __nv_bfloat16* dqrow = dq + static_cast<long long>(qidx) * ld + hh * D;
#pragma unroll 1
    for (int c = ch * (D / 64); c < (ch + 1) * (D / 64); ++c) {
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dq + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dqrow + c * 32, x, scale,
                   rope ? rope + (pos0 + qidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  if (CL2)
    dev::cluster_sync();  // no multicast or remote release still targets this CTA
  else
    __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

#ifdef MEMO_ATTN_ABLATIONS  // fused 5-unit backward (ablation build only)
// ------------------------------------------------------------ fused backward
// One CTA per (key tile kt, head): S^T, dP^T, dV += P^T dO, dK += dS^T Q and
// dQ^T_partial = K^T dS^T for every 64-query half of the query tiles kt..n-1,
// so S and dP are computed once (5 GEMM units instead of the split kernels' 7).
// dQ partials are summed in an f32 accumulator [H][S][D] at L2 in a FIXED order
// (key tile 0 stores, then 1, 2, … add): a per-(head, 64-query chunk) counter
// orders the contributions, and CTAs take (kt, head) from an atomic ticket in
// ascending kt, so a CTA only ever waits for CTAs that are already resident.
// The sum order never depends on scheduling -> bitwise deterministic dQ.
//
// TMEM (512 cols): [0,128) dV | [128,256) dK | [256,320) S^T buf0 | [320,384)
// S^T buf1 | [384,448) dP^T | [448,512) dQ^T.  P^T and dS^T (bf16) are written
// back into their S^T buffer (warp ch: cols 32ch..+16 P^T, 32ch+16..+32 dS^T)
// and feed dV/dK as TMEM A operands; dS^T also goes to shared memory as the B
// operand of dQ^T (the A operand is K itself read MN-major).
// Warps: 0 TMA, 1 MMA issue, 2 dQ ordering + bulk reduce, 4..11 softmax-grad math.
constexpr int FB_NS = 3;              // Q/dO half-tile ring stages
constexpr int FB_NSTG = 1;            // dQ^T staging buffers
constexpr int FB_HALF_BYTES = HALF * 64 * 2;  // [64 rows][64 cols] bf16 chunk = 8 KiB

template <int D>
struct FusedBwdSmem {
  static constexpr int NC = D / 64;
  static constexpr int TILE_BYTES = NC * CHUNK_BYTES;          // K or V [128][D]
  static constexpr int HT_BYTES = NC * FB_HALF_BYTES;          // Q or dO half [64][D]
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE_BYTES;
  static constexpr int RING_OFF = 2 * TILE_BYTES;              // stage: Q half | dO half
  static constexpr int DS_OFF = RING_OFF + FB_NS * 2 * HT_BYTES;  // 2 x [128 keys][64 q] bf16
  static constexpr int DS_BYTES = TILE * HALF * 2;
  static constexpr int STG_OFF = DS_OFF + 2 * DS_BYTES;        // dQ^T half staged [64 q][D] f32
  static constexpr int STG_BYTES = HALF * D * 4;
  static constexpr int VEC_OFF = STG_OFF + FB_NSTG * STG_BYTES;  // stage: lse2[64] | delta[64]
  static constexpr int BAR_OFF = VEC_OFF + FB_NS * 512;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

template <int D, int PEND>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap map_q,
                          const __grid_constant__ CUtensorMap map_k,
                          const __grid_constant__ CUtensorMap map_v,
                          const __grid_constant__ CUtensorMap map_do, const float* __restrict__ lse2,
                          const float* __restrict__ delta, float* __restrict__ dq_acc,
                          uint32_t* __restrict__ counters, uint32_t* __restrict__ ticket,
                          __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, long long ld,
                          const float2* __restrict__ rope, long long pos0, int S, int H, float scale,
                          float scale_log2, int G) {
  static_assert(D == 128, "fused backward needs M = D = 128 for the dQ^T MMA");
  using L = FusedBwdSmem<D>;
  constexpr int NC = L::NC;
  constexpr int NS = FB_NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* in_full = bars + 1;          // [NS]
  uint64_t* in_empty = in_full + NS;     // [NS]
  uint64_t* s_full = in_empty + NS;      // [2] (per S^T buffer)
  uint64_t* dp_full = s_full + 2;        // [2] (by half parity; one dP^T buffer)
  uint64_t* dp_free = dp_full + 2;       // [2]
  uint64_t* ds_ready = dp_free + 2;      // [2]
  uint64_t* dq_full = ds_ready + 2;      // [2]
  uint64_t* dq_free = dq_full + 2;       // [2]
  uint64_t* staged = dq_free + 2;        // [2] dQ^T(g) is in the staging buffer
  uint64_t* stg_free = staged + 2;       // [2] the bulk reduce of g has read it
  uint64_t* fin = stg_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);
  uint32_t* tick_slot = tmem_slot + 1;
  constexpr int CW = 32 * BWD_COMPUTE_WARPS;  // compute threads

  const uint32_t warp = dev::warp_id();
  const uint32_t lane = dev::lane_id();
  const int n_tiles = S / TILE;
  const int n_chunks = S / HALF;

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&map_q);
    dev::tma_prefetch_desc(&map_k);
    dev::tma_prefetch_desc(&map_v);
    dev::tma_prefetch_desc(&map_do);
    dev::mbar_init(kv_full, 1);
    for (int s2 = 0; s2 < NS; ++s2) {
      dev::mbar_init(&in_full[s2], 1);
      dev::mbar_init(&in_empty[s2], 1);
    }
    for (int s2 = 0; s2 < 2; ++s2) {
      dev::mbar_init(&s_full[s2], 1);
      dev::mbar_init(&dp_full[s2], 1);
      dev::mbar_init(&dp_free[s2], CW);
      dev::mbar_init(&ds_ready[s2], CW);
      dev::mbar_init(&dq_full[s2], 1);
      dev::mbar_init(&dq_free[s2], CW);
      dev::mbar_init(&staged[s2], CW);
      dev::mbar_init(&stg_free[s2], 1);
    }
    dev::mbar_init(fin, 1);
    dev::fence_barrier_init();
    *tick_slot = atomicAdd(ticket, 1u);
  }
  if (warp == 1) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Tickets: heads in groups of G; inside a group ascending key tile (heavy
  // first), heads innermost.  Every CTA with a smaller kt of the same head
  // holds a smaller ticket, so it is resident or done: waits cannot deadlock.
  const int tick = static_cast<int>(*tick_slot);
  const int grp = tick / (G * n_tiles);
  const int rem = tick - grp * G * n_tiles;
  const int kt = rem / G;
  const int hh = grp * G + rem % G;
  const int n_q = n_tiles - kt;
  const int n_g = 2 * n_q;
  // Query halves are walked from the last tile down to the diagonal, so the
  // CTAs of a wave sweep the same dQ chunks together (L2-resident reduces).
  auto chunk_of = [&](int g) { return 2 * (n_tiles - 1 - (g >> 1)) + (g & 1); };
  const uint32_t t_dv = tmem, t_dk = tmem + 128, t_dp = tmem + 384, t_dq = tmem + 448;
  auto t_s = [&](int b) { return tmem + 256 + 64 * b; };

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_expect_tx(kv_full, 2 * L::TILE_BYTES);
      for (int c = 0; c < NC; ++c) {
        dev::tma_load_2d(smem + L::K_OFF + c * CHUNK_BYTES, &map_k, kv_full, hh * D + c * 64, kt * TILE);
        dev::tma_load_2d(smem + L::V_OFF + c * CHUNK_BYTES, &map_v, kv_full, hh * D + c * 64, kt * TILE);
      }
      for (int g = 0; g < n_g; ++g) {
        const int st = g % NS;
        const int q0 = chunk_of(g) * HALF;
        dev::mbar_wait(&in_empty[st], ((g / NS) & 1) ^ 1);
        dev::mbar_expect_tx(&in_full[st], 2 * L::HT_BYTES + 512);
        uint8_t* sq = smem + L::RING_OFF + st * 2 * L::HT_BYTES;
        for (int c = 0; c < NC; ++c) {
          dev::tma_load_2d(sq + c * FB_HALF_BYTES, &map_q, &in_full[st], hh * D + c * 64, q0);
          dev::tma_load_2d(sq + L::HT_BYTES + c * FB_HALF_BYTES, &map_do, &in_full[st], hh * D + c * 64, q0);
        }
        const long long off = static_cast<long long>(hh) * S + q0;
        float* vec = reinterpret_cast<float*>(smem + L::VEC_OFF + st * 512);
        dev::bulk_load(vec, lse2 + off, 256, &in_full[st]);
        dev::bulk_load(vec + 64, delta + off, 256, &in_full[st]);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, converged: MMAs/commits elect one lane
      constexpr uint32_t idesc_s = dev::idesc_bf16_f32(128, HALF, false, false);
      constexpr uint32_t idesc_g = dev::idesc_bf16_f32(128, D, false, true);
      constexpr uint32_t idesc_q = dev::idesc_bf16_f32(D, HALF, true, true);
      const uint32_t k_addr = dev::smem_u32(smem + L::K_OFF);
      const uint64_t kd0 = kmajor_base(k_addr);
      const uint64_t vd0 = kmajor_base(dev::smem_u32(smem + L::V_OFF));
      const uint64_t ktd0 = dev::umma_desc_sw128(k_addr, CHUNK_BYTES, 1024);  // K^T, MN-major A
      // half-tile operands: 64-col chunks are FB_HALF_BYTES apart
      auto kmaj_half = [](uint64_t d, int kk) {
        return d + static_cast<uint64_t>(((kk >> 2) * FB_HALF_BYTES + (kk & 3) * 32) >> 4);
      };
      auto stage_addr = [&](int g) { return dev::smem_u32(smem + L::RING_OFF + (g % NS) * 2 * L::HT_BYTES); };
      dev::mbar_wait_w(kv_full, 0);
      auto issue_s = [&](int g) {
        const int st = g % NS;
        dev::mbar_wait_w(&in_full[st], (g / NS) & 1);
        dev::tc_fence_after();
        const uint64_t qd = dev::umma_desc_sw128(stage_addr(g), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ss_w(t_s(g & 1), kmajor_step(kd0, kk), kmaj_half(qd, kk), idesc_s, kk > 0);
        dev::mma_commit_w(&s_full[g & 1]);
      };
      auto issue_dp = [&](int g) {
        const uint64_t dod = dev::umma_desc_sw128(stage_addr(g) + L::HT_BYTES, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          dev::mma_bf16_ss_w(t_dp, kmajor_step(vd0, kk), kmaj_half(dod, kk), idesc_s, kk > 0);
        dev::mma_commit_w(&dp_full[g & 1]);
      };
      issue_s(0);
      issue_dp(0);
      for (int g = 0; g < n_g; ++g) {
        const int b = g & 1;
        const uint32_t par = (g >> 1) & 1;
        if (g + 1 < n_g) {
          issue_s(g + 1);
          dev::mbar_wait_w(&dp_free[b], par);  // softmax warps hold dP^T(g) in registers
          dev::tc_fence_after();
          issue_dp(g + 1);
        }
        dev::mbar_wait_w(&ds_ready[b], par);
        dev::tc_fence_after();
        const uint32_t sa = stage_addr(g);
        const uint64_t qm = dev::umma_desc_sw128(sa, FB_HALF_BYTES, 1024);
        const uint64_t dom = dev::umma_desc_sw128(sa + L::HT_BYTES, FB_HALF_BYTES, 1024);
#pragma unroll
        for (int kk = 0; kk < HALF / 16; ++kk)
          dev::mma_bf16_ts_w(t_dv, t_s(b) + 32 * (kk >> 1) + 8 * (kk & 1), mnmajor_step(dom, kk), idesc_g,
                           (g | kk) != 0);
#pragma unroll
        for (int kk = 0; kk < HALF / 16; ++kk)
          dev::mma_bf16_ts_w(t_dk, t_s(b) + 32 * (kk >> 1) + 16 + 8 * (kk & 1), mnmajor_step(qm, kk), idesc_g,
                           (g | kk) != 0);
        dev::mma_commit_w(&in_empty[g % NS]);
        if (g > 0) {
          dev::mbar_wait_w(&dq_free[b ^ 1], ((g - 1) >> 1) & 1);
          dev::tc_fence_after();
        }
        const uint64_t dsd = dev::umma_desc_sw128(dev::smem_u32(smem + L::DS_OFF + b * L::DS_BYTES), CHUNK_BYTES, 1024);
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          dev::mma_bf16_ss_w(t_dq, mnmajor_step(ktd0, kk), mnmajor_step(dsd, kk), idesc_q, kk > 0);
        dev::mma_commit_w(&dq_full[b]);
      }
      dev::mma_commit_w(fin);
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // dQ^T(g) staged -> wait for this chunk's turn -> one bulk f32 reduce at
      // L2 (key tile 0 stores) -> release the chunk once the reduce completed.
      const uint32_t stg0 = dev::smem_u32(smem + L::STG_OFF);
      uint32_t* ctr0 = counters + static_cast<long long>(hh) * n_chunks;
      float* acc0 = dq_acc + static_cast<long long>(hh) * S * D;
      for (int g = 0; g < n_g; ++g) {
        const int b = g & 1;
        const int ck = chunk_of(g);
        dev::mbar_wait(&staged[b], (g >> 1) & 1);
        if (kt > 0) {
          while (dev::ld_acquire_u32(ctr0 + ck) != static_cast<uint32_t>(kt)) __nanosleep(32);
        }
        dev::fence_proxy_async_global();
        const uint32_t stg = stg0 + (g % FB_NSTG) * L::STG_BYTES;
        if (kt == 0)
          dev::bulk_store(acc0 + static_cast<long long>(ck) * HALF * D, stg, L::STG_BYTES);
        else
          dev::bulk_reduce_add_f32(acc0 + static_cast<long long>(ck) * HALF * D, stg, L::STG_BYTES);
        dev::bulk_commit();
        dev::bulk_wait_read<0>();
        dev::mbar_arrive(&stg_free[b]);
        // keep PEND reduces in flight; release each chunk once its reduce completed
        if (g >= PEND) {
          dev::bulk_wait<PEND>();
          dev::fence_proxy_async_global();
          dev::st_release_u32(ctr0 + chunk_of(g - PEND), static_cast<uint32_t>(kt + 1));
        }
      }
      dev::bulk_wait<0>();
      dev::fence_proxy_async_global();
      for (int g = n_g > PEND ? n_g - PEND : 0; g < n_g; ++g)
        dev::st_release_u32(ctr0 + chunk_of(g), static_cast<uint32_t>(kt + 1));
    }
  } else if (warp >= 4) {
    const uint32_t q4 = warp & 3;
    const int ch = (warp - 4) >> 2;  // which 32-query slice of each half this warp owns
    const int r = q4 * 32 + lane;    // key row in tile (TMEM lane); also D index for dQ^T
    const uint32_t lane_off = (q4 * 32) << 16;
    const uint32_t ds_row = dev::smem_u32(smem + L::DS_OFF) + (r >> 3) * 1024 + (r & 7) * 128;
    // dQ^T(g): TMEM -> registers -> staging buffer [64 q][D] f32 (warp 2 reduces it)
    const uint32_t stg_col = dev::smem_u32(smem + L::STG_OFF) + (32 * ch) * (D * 4) + r * 4;
    auto drain = [&](int g) {
      const int b = g & 1;
      const uint32_t par = (g >> 1) & 1;
      dev::mbar_wait(&dq_full[b], par);
      dev::tc_fence_after();
      uint32_t x[32];
      dev::tmem_ld32(t_dq + lane_off + 32 * ch, x);
      dev::tmem_ld_wait_regs(x);
      dev::tc_fence_before();
      dev::mbar_arrive(&dq_free[b]);
      // staging buffer g % FB_NSTG was last read by the bulk reduce of g - FB_NSTG
      if (g >= FB_NSTG) dev::mbar_wait(&stg_free[(g - FB_NSTG) & 1], ((g - FB_NSTG) >> 1) & 1);
      const uint32_t sc = stg_col + (g % FB_NSTG) * L::STG_BYTES;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(sc + j * (D * 4)), "r"(x[j]) : "memory");
      dev::fence_proxy_async();
      dev::mbar_arrive(&staged[b]);
    };
    for (int g = 0; g < n_g; ++g) {
      const int b = g & 1, st = g % NS;
      const uint32_t par = (g >> 1) & 1;
      const bool diag = g >= n_g - 2;  // query tile == key tile
      const uint32_t vec = dev::smem_u32(smem + L::VEC_OFF + st * 512) + 32 * ch * 4;
      dev::mbar_wait(&in_full[st], (g / NS) & 1);
      dev::mbar_wait(&s_full[b], par);
      dev::mbar_wait(&dp_full[b], par);
      dev::tc_fence_after();
      uint32_t sr[32], dr[32];
      dev::tmem_ld32(t_s(b) + lane_off + 32 * ch, sr);
      dev::tmem_ld32(t_dp + lane_off + 32 * ch, dr);
      dev::tmem_ld_wait_regs(sr, dr);
      dev::tc_fence_before();
      dev::mbar_arrive(&dp_free[b]);
      uint32_t pp[16], dd[16];
      auto body = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 lv = dev::lds_f4(vec + 16 * j4);
          const float4 dv4 = dev::lds_f4(vec + 256 + 16 * j4);
          const float lq[4] = {lv.x, lv.y, lv.z, lv.w};
          const float dq4[4] = {dv4.x, dv4.y, dv4.z, dv4.w};
          float p4[4], d4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int qc = (g & 1) * HALF + 32 * ch + 4 * j4 + e;  // query within tile
            float p = dev::ex2(fmaf(__uint_as_float(sr[4 * j4 + e]), scale_log2, lq[e]));
            if (DIAG && qc < r) p = 0.f;
            p4[e] = p;
            d4[e] = p * (__uint_as_float(dr[4 * j4 + e]) + dq4[e]);
          }
          pp[2 * j4] = dev::pack_bf16(p4[0], p4[1]);
          pp[2 * j4 + 1] = dev::pack_bf16(p4[2], p4[3]);
          dd[2 * j4] = dev::pack_bf16(d4[0], d4[1]);
          dd[2 * j4 + 1] = dev::pack_bf16(d4[2], d4[3]);
        }
      };
      if (diag)
        body(std::true_type{});
      else
        body(std::false_type{});
      dev::tmem_st16(t_s(b) + lane_off + 32 * ch, pp);
      dev::tmem_st16(t_s(b) + lane_off + 32 * ch + 16, dd);
      // dS^T row r, queries 32ch..32ch+31 -> 16-byte chunks 4ch..4ch+3 (128-byte swizzle)
      const uint32_t row = ds_row + b * L::DS_BYTES;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dev::sts_u4(row + (((4 * ch + j) ^ (r & 7)) << 4), dd[4 * j], dd[4 * j + 1], dd[4 * j + 2],
                    dd[4 * j + 3]);
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::fence_proxy_async();
      dev::mbar_arrive(&ds_ready[b]);
      if (g > 0) drain(g - 1);
    }
    drain(n_g - 1);
    dev::mbar_wait(fin, 0);
    dev::tc_fence_after();
    const int kidx = kt * TILE + r;
    __nv_bfloat16* dvrow = dv + static_cast<long long>(kidx) * ld + hh * D;
    __nv_bfloat16* dkrow = dk + static_cast<long long>(kidx) * ld + hh * D;
#pragma unroll 1
    for (int c = ch * (D / 64); c < (ch + 1) * (D / 64); ++c) {
      uint32_t r32[32];
      float x[32];
      dev::tmem_ld32(t_dv + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dvrow + c * 32, x, 1.f, nullptr);
      dev::tmem_ld32(t_dk + lane_off + c * 32, r32);
      dev::tmem_ld_wait_regs(r32);
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(r32[e]);
      store_grad32(dkrow + c * 32, x, scale, rope ? rope + (pos0 + kidx) * (D / 2) + c * 16 : nullptr);
    }
    dev::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

// dq [S, ld] bf16 = inverse-RoPE(scale * acc [H][S][D] f32); 8 columns per thread.
__global__ void attn_dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                       long long ld, const float2* __restrict__ rope, long long pos0,
                                       int S, int H, int D, float scale) {
  const long long hc = static_cast<long long>(H) * D;
  const long long n8 = static_cast<long long>(S) * hc / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = i / (hc / 8);
    const int col = static_cast<int>(i - t * (hc / 8)) * 8;
    const float* src = acc + (static_cast<long long>(col / D) * S + t) * D + col % D;  // [H][S][D]
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *reinterpret_cast<const float4*>(src + 4);
    float x[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale,
                  b.x * scale, b.y * scale, b.z * scale, b.w * scale};
    if (rope) {
      const int d = col % D;
      const float2* cs = rope + (pos0 + t) * (D / 2) + d / 2;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 c = cs[p];
        const float u = x[2 * p], w = x[2 * p + 1];
        x[2 * p] = u * c.x + w * c.y;
        x[2 * p + 1] = -u * c.y + w * c.x;
      }
    }
    uint4 o;
    o.x = dev::pack_bf16(x[0], x[1]);
    o.y = dev::pack_bf16(x[2], x[3]);
    o.z = dev::pack_bf16(x[4], x[5]);
    o.w = dev::pack_bf16(x[6], x[7]);
    *reinterpret_cast<uint4*>(dq + t * ld + col) = o;
  }
}
#endif  // MEMO_ATTN_ABLATIONS

#ifdef MEMO_ATTN_ABLATIONS
// Ablation build only (make -C csrc ablations -> _lib_ablations/libmemo.so,
// selected by tools through MEMO_LIB_PATH): environment-selected variants whose
// measurements DESIGN §4 and profiles/README.md record.  The product library
// contains none of these kernels and reads no environment variable here.
int abl_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
bool bwd_fused() {
  const char* e = getenv("MEMO_ATTN_BWD");
  return e && std::string(e) == "fused";
}

cudaError_t launch_bwd_fused(const AttnBwdArgs& a, cudaStream_t stream) {
  constexpr int D = 128;
  using L = FusedBwdSmem<D>;
  const int h = a.H * D;
  CUtensorMap mq, mk, mv, mdo;
  bool ok = make_tma_2d_bf16(&mq, a.q, h, a.S, h, 64, HALF) &&
            make_tma_2d_bf16(&mk, a.k, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mv, a.v, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mdo, a.dout, h, a.S, h, 64, HALF);
  if (!ok) return cudaErrorInvalidValue;
  static std::once_flag f;
  std::call_once(f, [] {
    cudaFuncSetAttribute(attn_bwd_fused_kernel<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    cudaFuncSetAttribute(attn_bwd_fused_kernel<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    cudaFuncSetAttribute(attn_bwd_fused_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
    cudaFuncSetAttribute(attn_bwd_fused_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
  });
  const int pend = abl_env("MEMO_FB_PEND", 0);
  // heads per ticket group: the accumulator of a group should stay L2-resident
  int G = abl_env("MEMO_FB_GROUP", 0);
  if (G <= 0) G = 4;
  while (G > 1 && a.H % G != 0) --G;
  const long long HS = static_cast<long long>(a.H) * a.S;
  float* delta = a.delta;
  float* lse2 = a.delta + HS;
  float* acc = a.delta + 2 * HS;
  uint32_t* counters = reinterpret_cast<uint32_t*>(acc + HS * D);
  const long long n_ctr = HS / HALF;
  uint32_t* ticket = counters + n_ctr;
  if (a.ev[0]) record_timing_event(a.ev[0], stream);
  cudaMemsetAsync(counters, 0, (n_ctr + 4) * sizeof(uint32_t), stream);
  attn_bwd_prep_kernel<<<(a.S * a.H * (D / 8) + 255) / 256, 256, 0, stream>>>(a.o, a.dout, a.lse, delta, lse2, a.S,
                                                                              a.H, D);
  if (a.ev[1]) record_timing_event(a.ev[1], stream);
  const float2* rope = reinterpret_cast<const float2*>(a.rope);
  auto kern = pend >= 4 ? attn_bwd_fused_kernel<D, 4>
             : pend == 2 ? attn_bwd_fused_kernel<D, 2>
             : pend == 1 ? attn_bwd_fused_kernel<D, 1>
                         : attn_bwd_fused_kernel<D, 0>;
  kern<<<(a.S / TILE) * a.H, BWD_THREADS, L::BYTES, stream>>>(
      mq, mk, mv, mdo, lse2, delta, acc, counters, ticket, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S,
      a.H, a.softmax_scale, a.softmax_scale * kLog2e, G);
  if (a.ev[2]) record_timing_event(a.ev[2], stream);
  const long long n8 = HS * D / 8;
  const int blocks = static_cast<int>(std::min<long long>((n8 + 255) / 256, 148LL * 16));
  attn_dq_convert_kernel<<<blocks, 256, 0, stream>>>(acc, a.dq, a.ld_dqkv, rope, a.pos0, a.S, a.H, D,
                                                     a.softmax_scale);
  if (a.ev[3]) record_timing_event(a.ev[3], stream);
  return cudaGetLastError();
}
#endif  // MEMO_ATTN_ABLATIONS

// Deterministic split backward: prep (delta, log2 LSE), dK/dV (K/V resident in
// TMEM, one CTA per key tile) and dQ (Q/dO resident in TMEM, one CTA per query
// tile); no atomics, so every output is bitwise repeatable.
template <int D>
cudaError_t launch_bwd(const AttnBwdArgs& a, cudaStream_t stream) {
  const int h = a.H * a.D;
  CUtensorMap mq, mk, mv, mdo;
  bool ok = make_tma_2d_bf16(&mq, a.q, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mk, a.k, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mv, a.v, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mdo, a.dout, h, a.S, h, 64, TILE);
  if (!ok) return cudaErrorInvalidValue;
  static std::once_flag f;
  std::call_once(f, [] {
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dq_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         BwdSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, DkdvTmSmem<D>::BYTES);
#ifdef MEMO_ATTN_ABLATIONS
    cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         BwdSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, true, 0, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, false, 2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, false, 1>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dkdv_tm2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DkdvTmSmem<D>::BYTES);
    cudaFuncSetAttribute(attn_bwd_dq_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         BwdSmem<D>::BYTES);
#endif
  });
  float* delta = a.delta;
  float* lse2 = a.delta + static_cast<long long>(a.H) * a.S;
  const int rows = a.S * a.H;
  if (a.ev[0]) record_timing_event(a.ev[0], stream);
  attn_bwd_prep_kernel<<<(rows * (D / 8) + 255) / 256, 256, 0, stream>>>(a.o, a.dout, a.lse, delta, lse2, a.S,
                                                            a.H, D);
  const float scale_log2 = a.softmax_scale * kLog2e;
  const float2* rope = reinterpret_cast<const float2*>(a.rope);
  dim3 grid(a.S / TILE, a.H);
  // dK/dV: CTA pairs on key tiles 2p, 2p+1 sharing each Q/dO tile by multicast
  // whenever the tile count is even (bitwise equal; 3-4 % faster at 128K: half
  // the L2 reads buys clock under the power cap).  Ablation build:
  // MEMO_ATTN_DKDV_CL2=0 -> one CTA per key tile, 2 -> pairs without multicast,
  // 3 -> the single-CTA kernel launched as clusters (placement only).
  bool dkdv_cl2 = (a.S / TILE) % 2 == 0;
  int clm = 1;
#ifdef MEMO_ATTN_ABLATIONS
  clm = abl_env("MEMO_ATTN_DKDV_CL2", 1);
  dkdv_cl2 = dkdv_cl2 && clm >= 1;
#endif
  if (a.ev[1]) record_timing_event(a.ev[1], stream);
#ifdef MEMO_ATTN_ABLATIONS
  // MEMO_ATTN_DKDV_VARIANT: 1 K/V in shared memory, 2 four warps per lane
  // quarter, 3 P^T/dS^T behind separate barriers, 4/5 every 2nd/4th column
  // pair's exponentials on the FMA pipe, 7 P^T/dS^T decoupled from a single
  // S^T/dP^T buffer (attn_bwd_dkdv_tm2_kernel: 231-232 vs 206-207 ms at 128K),
  // 8/9 one-step Q/dO stages (TS = 12 / 8)
  switch (abl_env("MEMO_ATTN_DKDV_VARIANT", 0)) {
    case 13: {  // one-step Q/dO stages (TS = 12) on CTA pairs sharing them by multicast
      CUtensorMap mq32, mdo32;
      if (!make_tma_2d_bf16(&mq32, a.q, h, a.S, h, 64, QSTEP) || !make_tma_2d_bf16(&mdo32, a.dout, h, a.S, h, 64, QSTEP))
        return cudaErrorInvalidValue;
      if ((a.S / TILE) % 2 != 0) return cudaErrorInvalidValue;
      static std::once_flag f13;
      std::call_once(f13, [] {
        cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 12, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, DkdvTsSmem<D, 12>::BYTES);
      });
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(32 * (4 + 8));
      cfg.dynamicSmemBytes = DkdvTsSmem<D, 12>::BYTES;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 12, true>, a.k, a.v,
                                               mq32, mdo32, (const float*)lse2, (const float*)delta, a.dk, a.dv,
                                               a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale, scale_log2);
      if (e != cudaSuccess) return e;
      break;
    }
    case 12:
      attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, false, 1><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 11:
      attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, false, 2><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 10: {  // 16-query steps, four S/dP buffers (N=16 MMAs run at 79 %: 268 vs 206 ms)
      static std::once_flag f16;
      std::call_once(f16, [] {
        cudaFuncSetAttribute(attn_bwd_dkdv_q16_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DkdvTmSmem<D>::BYTES);
      });
      attn_bwd_dkdv_q16_kernel<D><<<grid, 32 * 12, DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    }
    case 8:
    case 9: {
      // one-step Q/dO stages (TS = 12 / 8): loads run TS-1 steps ahead
      CUtensorMap mq32, mdo32;
      if (!make_tma_2d_bf16(&mq32, a.q, h, a.S, h, 64, QSTEP) || !make_tma_2d_bf16(&mdo32, a.dout, h, a.S, h, 64, QSTEP))
        return cudaErrorInvalidValue;
      static std::once_flag fts;
      std::call_once(fts, [] {
        cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DkdvTsSmem<D, 12>::BYTES);
        cudaFuncSetAttribute(attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DkdvTsSmem<D, 8>::BYTES);
      });
      if (abl_env("MEMO_ATTN_DKDV_VARIANT", 0) == 8)
        attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 12><<<grid, 32 * (4 + 8), DkdvTsSmem<D, 12>::BYTES, stream>>>(
            a.k, a.v, mq32, mdo32, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
            scale_log2);
      else
        attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 8><<<grid, 32 * (4 + 8), DkdvTsSmem<D, 8>::BYTES, stream>>>(
            a.k, a.v, mq32, mdo32, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
            scale_log2);
      break;
    }
    case 7:
      attn_bwd_dkdv_tm2_kernel<D><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 1:
      attn_bwd_dkdv_kernel<D><<<grid, BWD_THREADS, BwdSmem<D>::BYTES, stream>>>(
          mq, mk, mv, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.softmax_scale, scale_log2);
      break;
    case 2:
      attn_bwd_dkdv_tm_kernel<D, 4><<<grid, 32 * (4 + 16), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 3:
      attn_bwd_dkdv_tm_kernel<D, 2, 0, true><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 4:
      attn_bwd_dkdv_tm_kernel<D, 2, 2><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    case 5:
      attn_bwd_dkdv_tm_kernel<D, 2, 4><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
          a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
          scale_log2);
      break;
    default:
#endif
      if (dkdv_cl2) {  // CTA pairs sharing each Q/dO tile by multicast
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(32 * (4 + 8));
        cfg.dynamicSmemBytes = DkdvTmSmem<D>::BYTES;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e;
#ifdef MEMO_ATTN_ABLATIONS
        if (clm == 3)  // the single-CTA kernel, launched as clusters of 2 (placement only)
          e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_tm_kernel<D, 2>, a.k, a.v, mq, mdo, (const float*)lse2,
                                 (const float*)delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H,
                                 a.softmax_scale, scale_log2);
        else if (clm == 2)  // pairs, each CTA loading whole tiles (no multicast)
          e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, true, 0, true>, a.k, a.v, mq,
                                 mdo, (const float*)lse2, (const float*)delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0,
                                 a.S, a.H, a.softmax_scale, scale_log2);
        else
#endif
          e = cudaLaunchKernelEx(&cfg, attn_bwd_dkdv_tm_kernel<D, 2, 0, false, 0, true>, a.k, a.v, mq, mdo,
                                 (const float*)lse2, (const float*)delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S,
                                 a.H, a.softmax_scale, scale_log2);
        if (e != cudaSuccess) return e;
      } else {
        attn_bwd_dkdv_tm_kernel<D, 2><<<grid, 32 * (4 + 8), DkdvTmSmem<D>::BYTES, stream>>>(
            a.k, a.v, mq, mdo, lse2, delta, a.dk, a.dv, a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale,
            scale_log2);
      }
#ifdef MEMO_ATTN_ABLATIONS
  }
#endif
  if (a.ev[2]) record_timing_event(a.ev[2], stream);
  // dQ: CTA pairs (clusters of 2) sharing each K/V tile by multicast whenever
  // the tile count is even (1 % faster at 128K, bitwise equal).  Ablation
  // build: MEMO_ATTN_DQ_CL2=0 -> one CTA per query tile, MEMO_ATTN_DQ_TMEM_A=0 ->
  // Q/dO as shared-memory operands.
  bool dq_cl2 = (a.S / TILE) % 2 == 0;
#ifdef MEMO_ATTN_ABLATIONS
  dq_cl2 = dq_cl2 && abl_env("MEMO_ATTN_DQ_CL2", 1) == 1;
  if (abl_env("MEMO_ATTN_DQ_TMEM_A", 1) == 0) {  // Q/dO as shared-memory operands
    attn_bwd_dq_kernel<D, false><<<grid, BWD_THREADS, BwdSmem<D>::BYTES, stream>>>(
        a.q, a.dout, mq, mdo, mk, mv, lse2, delta, a.dq, a.ld_dqkv, rope, a.pos0, a.S, a.H,
        a.softmax_scale, scale_log2);
    dq_cl2 = false;
  } else
#endif
  if (dq_cl2) {
    static std::once_flag fcl;
    std::call_once(fcl, [] {
      cudaFuncSetAttribute(attn_bwd_dq_kernel<D, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           BwdSmem<D>::BYTES);
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(BWD_THREADS);
    cfg.dynamicSmemBytes = BwdSmem<D>::BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_bwd_dq_kernel<D, true, true>, a.q, a.dout, mq, mdo, mk, mv,
                                             static_cast<const float*>(lse2), static_cast<const float*>(delta), a.dq,
                                             a.ld_dqkv, rope, a.pos0, a.S, a.H, a.softmax_scale, scale_log2);
    if (e != cudaSuccess) return e;
  } else {
    attn_bwd_dq_kernel<D, true><<<grid, BWD_THREADS, BwdSmem<D>::BYTES, stream>>>(
        a.q, a.dout, mq, mdo, mk, mv, lse2, delta, a.dq, a.ld_dqkv, rope, a.pos0, a.S, a.H,
        a.softmax_scale, scale_log2);
  }
  if (a.ev[3]) record_timing_event(a.ev[3], stream);
  return cudaGetLastError();
}

}  // namespace

template <int D, bool QT, bool EMU>
void launch_fwd(const AttnFwdArgs& a, const CUtensorMap& mq, const CUtensorMap& mk,
                const CUtensorMap& mv, float scale_log2, cudaStream_t stream) {
  using L = FwdSmem<D, QT>;
  static std::once_flag f;
  std::call_once(f, [] {
    cudaFuncSetAttribute(attn_fwd_kernel<D, QT, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         L::BYTES);
  });
  dim3 grid(a.S / TILE, a.H);
  attn_fwd_kernel<D, QT, EMU><<<grid, 256, L::BYTES, stream>>>(a.q, mq, mk, mv, a.o, a.lse, a.S,
                                                               a.H, scale_log2);
}

cudaError_t attn_fwd(const AttnFwdArgs& a, cudaStream_t stream) {
  if (a.S % TILE != 0 || (a.D != 64 && a.D != 128)) return cudaErrorInvalidValue;
  const int h = a.H * a.D;
  CUtensorMap mq, mk, mv;
  bool ok = make_tma_2d_bf16(&mq, a.q, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mk, a.k, h, a.S, h, 64, TILE) &&
            make_tma_2d_bf16(&mv, a.v, h, a.S, h, 64, TILE);
  if (!ok) return cudaErrorInvalidValue;
  const float scale_log2 = a.softmax_scale * kLog2e;
  if (a.ev[0]) record_timing_event(a.ev[0], stream);
#ifdef MEMO_ATTN_ABLATIONS
  // MEMO_ATTN_FWD_VARIANT: 0-3 one softmax warp per row (bit0 Q in TMEM, bit1
  // FMA exp2 share); 5-7 split rows (1/4, none, 1/8 FMA share); 8-12 ping-pong
  // with FMA share 1/3 (product), none, 1/8, 1/4, 1/2; 13 ping-pong without the
  // two-half P release (the round-1 product); 14, 15 ping-pong with share 1/6, 1/16;
  // 16 ping-pong with no softmax math (NULL_SM: the MMA/TMA/TMEM ceiling, wrong output);
  // 17-20 ping-pong with split rows (attn_fwd_pp2w_kernel), FMA share 1/3, 1/4, none, 1/8;
  // 21-23 ping-pong without MMAs (NULL_MMA: the softmax-throughput ceiling, wrong output), share 1/3, none, 1/4;
  // 24-26 ping-pong with the groups taking turns on the exponentials (SEQ), share 1/3, none, 1/4;
  // 27 ping-pong with quarter P stores and the row sum after the release (QSTORE);
  // 28-31 ping-pong without the wait::ld after the S loads (LDSB), share 1/3, 1/8, none, 1/4;
  // 32 LDSB + QSTORE, share 1/8; 33 the round-2 product before LDSB (wait::ld after the S loads);
  // 34-37 QSTORE (with LDSB), share 1/4, 1/6, 1/16, none; 42/43 CTA-pair ping-pong (share 1/3, 1/4), 44 its MMA-side ceiling (P = 0);
  // 38-41 split rows with the groups taking turns (attn_fwd_pp2w_kernel SEQ), share 1/4, 1/8, none, 1/16
  const int v = abl_env("MEMO_ATTN_FWD_VARIANT", 8);
  if (v != 8) {
    if ((v == 42 || v == 43 || v == 44) && a.D == 128 && a.S % (4 * TILE) == 0) {
      // CTA-pair ping-pong (attn_fwd_pair_kernel), FMA share 1/3 / 1/4
      CUtensorMap mk64;
      if (!make_tma_2d_bf16(&mk64, a.k, h, a.S, h, 64, 64)) return cudaErrorInvalidValue;
      static std::once_flag fpair;
      std::call_once(fpair, [] {
        cudaFuncSetAttribute(attn_fwd_pair_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPairSmem::BYTES);
        cudaFuncSetAttribute(attn_fwd_pair_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPairSmem::BYTES);
        cudaFuncSetAttribute(attn_fwd_pair_kernel<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FwdPairSmem::BYTES);
      });
      auto kern = v == 42 ? attn_fwd_pair_kernel<3> : v == 43 ? attn_fwd_pair_kernel<4> : attn_fwd_pair_kernel<3, true>;
      kern<<<dim3(2 * (a.S / (4 * TILE)), a.H), 384, FwdPairSmem::BYTES, stream>>>(mq, mk64, mv, a.o, a.lse, a.S, a.H,
                                                                                 scale_log2);
    } else if (((v >= 17 && v <= 20) || (v >= 38 && v <= 41)) && a.D == 128 && a.S % (2 * TILE) == 0) {
      static std::once_flag fw;
      std::call_once(fw, [] {
        for (auto k : {attn_fwd_pp2w_kernel<3>, attn_fwd_pp2w_kernel<4>, attn_fwd_pp2w_kernel<0>,
                       attn_fwd_pp2w_kernel<8>, attn_fwd_pp2w_kernel<4, true>, attn_fwd_pp2w_kernel<8, true>,
                       attn_fwd_pp2w_kernel<0, true>, attn_fwd_pp2w_kernel<16, true>})
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPp2wSmem::BYTES);
      });
      auto kern = v == 17 ? attn_fwd_pp2w_kernel<3> : v == 18 ? attn_fwd_pp2w_kernel<4>
                : v == 19 ? attn_fwd_pp2w_kernel<0> : v == 20 ? attn_fwd_pp2w_kernel<8>
                : v == 38 ? attn_fwd_pp2w_kernel<4, true> : v == 39 ? attn_fwd_pp2w_kernel<8, true>
                : v == 40 ? attn_fwd_pp2w_kernel<0, true> : attn_fwd_pp2w_kernel<16, true>;
      kern<<<dim3(a.S / (2 * TILE), a.H), PP2W_THREADS, FwdPp2wSmem::BYTES, stream>>>(mq, mk, mv, a.o, a.lse, a.S,
                                                                                     a.H, scale_log2);
    } else if (v >= 9 && a.D == 128 && a.S % (2 * TILE) == 0) {
      static std::once_flag fa;
      std::call_once(fa, [] {
        for (auto k : {attn_fwd_pp_kernel<0>, attn_fwd_pp_kernel<8>, attn_fwd_pp_kernel<4>, attn_fwd_pp_kernel<2>,
                       attn_fwd_pp_kernel<3, false>, attn_fwd_pp_kernel<6>, attn_fwd_pp_kernel<16>,
                       attn_fwd_pp_kernel<3, true, true>, attn_fwd_pp_kernel<3, true, false, true>,
                       attn_fwd_pp_kernel<0, true, false, true>, attn_fwd_pp_kernel<4, true, false, true>,
                       attn_fwd_pp_kernel<3, true, false, false, true, true>,
                       attn_fwd_pp_kernel<0, true, false, false, true, true>,
                       attn_fwd_pp_kernel<4, true, false, false, true, true>,
                       attn_fwd_pp_kernel<3, true, false, false, false, true>,
                       attn_fwd_pp_kernel<3, true, false, false, false, false, true>,
                       attn_fwd_pp_kernel<8, true, false, false, false, false, true>,
                       attn_fwd_pp_kernel<0, true, false, false, false, false, true>,
                       attn_fwd_pp_kernel<4, true, false, false, false, false, true>,
                       attn_fwd_pp_kernel<8, true, false, false, false, true, true>,
                       attn_fwd_pp_kernel<3, true, false, false, false, false, false>,
                       attn_fwd_pp_kernel<4, true, false, false, false, true>,
                       attn_fwd_pp_kernel<6, true, false, false, false, true>,
                       attn_fwd_pp_kernel<16, true, false, false, false, true>,
                       attn_fwd_pp_kernel<0, true, false, false, false, true>})
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPpSmem::BYTES);
      });
      auto kern = v == 9 ? attn_fwd_pp_kernel<0> : v == 10 ? attn_fwd_pp_kernel<8>
                : v == 11 ? attn_fwd_pp_kernel<4> : v == 12 ? attn_fwd_pp_kernel<2>
                : v == 14 ? attn_fwd_pp_kernel<6> : v == 15 ? attn_fwd_pp_kernel<16>
                : v == 16 ? attn_fwd_pp_kernel<3, true, true>
                : v == 21 ? attn_fwd_pp_kernel<3, true, false, true>
                : v == 22 ? attn_fwd_pp_kernel<0, true, false, true>
                : v == 23 ? attn_fwd_pp_kernel<4, true, false, true>
                : v == 24 ? attn_fwd_pp_kernel<3, true, false, false, true, true>
                : v == 25 ? attn_fwd_pp_kernel<0, true, false, false, true, true>
                : v == 26 ? attn_fwd_pp_kernel<4, true, false, false, true, true>
                : v == 27 ? attn_fwd_pp_kernel<3, true, false, false, false, true>
                : v == 28 ? attn_fwd_pp_kernel<3, true, false, false, false, false, true>
                : v == 29 ? attn_fwd_pp_kernel<8, true, false, false, false, false, true>
                : v == 30 ? attn_fwd_pp_kernel<0, true, false, false, false, false, true>
                : v == 31 ? attn_fwd_pp_kernel<4, true, false, false, false, false, true>
                : v == 32 ? attn_fwd_pp_kernel<8, true, false, false, false, true, true>
                : v == 33 ? attn_fwd_pp_kernel<3, true, false, false, false, false, false>
                : v == 34 ? attn_fwd_pp_kernel<4, true, false, false, false, true>
                : v == 35 ? attn_fwd_pp_kernel<6, true, false, false, false, true>
                : v == 36 ? attn_fwd_pp_kernel<16, true, false, false, false, true>
                : v == 37 ? attn_fwd_pp_kernel<0, true, false, false, false, true>
                : attn_fwd_pp_kernel<3, false>;
      kern<<<dim3(a.S / (2 * TILE), a.H), 384, FwdPpSmem::BYTES, stream>>>(mq, mk, mv, a.o, a.lse, a.S, a.H,
                                                                          scale_log2);
    } else if ((v == 5 || v == 6 || v == 7) && a.D == 128) {
      static std::once_flag fb;
      std::call_once(fb, [] {
        for (auto k : {attn_fwd_2w_kernel<4>, attn_fwd_2w_kernel<8>, attn_fwd_2w_kernel<0>})
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2wSmem::BYTES);
      });
      auto kern = v == 5 ? attn_fwd_2w_kernel<4> : v == 7 ? attn_fwd_2w_kernel<8> : attn_fwd_2w_kernel<0>;
      kern<<<dim3(a.S / TILE, a.H), 384, Fwd2wSmem::BYTES, stream>>>(a.q, mk, mv, a.o, a.lse, a.S, a.H, scale_log2);
    } else if (a.D == 128) {
      switch (v) {
        case 0: launch_fwd<128, false, false>(a, mq, mk, mv, scale_log2, stream); break;
        case 1: launch_fwd<128, true, false>(a, mq, mk, mv, scale_log2, stream); break;
        case 2: launch_fwd<128, false, true>(a, mq, mk, mv, scale_log2, stream); break;
        default: launch_fwd<128, true, true>(a, mq, mk, mv, scale_log2, stream); break;
      }
    } else {
      launch_fwd<64, true, true>(a, mq, mk, mv, scale_log2, stream);
    }
    if (a.ev[1]) record_timing_event(a.ev[1], stream);
    return cudaGetLastError();
  }
#endif
  bool fwd_cl2 = a.S % (4 * TILE) == 0;
#ifdef MEMO_ATTN_ABLATIONS
  fwd_cl2 = fwd_cl2 && abl_env("MEMO_ATTN_FWD_CL2", 1) == 1;
#endif
  if (a.D == 128 && fwd_cl2) {
    // ping-pong on CTA pairs (clusters of 2) sharing each K/V tile by multicast
    // whenever the query-tile pairs come in pairs: bitwise equal to one CTA per
    // pair, 0.7 % faster at 128K (ablation build: MEMO_ATTN_FWD_CL2=0 -> one CTA)
    static std::once_flag fcl;
    std::call_once(fcl, [] {
      cudaFuncSetAttribute(attn_fwd_pp_kernel<3, true, false, false, false, false, true, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPpSmem::BYTES);
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.S / (2 * TILE), a.H);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = FwdPpSmem::BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = attn_fwd_pp_kernel<3, true, false, false, false, false, true, true>;
#ifdef MEMO_ATTN_ABLATIONS
    // MEMO_ATTN_FWD_EMU=6/8/16: that share of the exponentials on the FMA pipe instead of 1/3
    switch (abl_env("MEMO_ATTN_FWD_EMU", 3)) {
      case 6: kern = attn_fwd_pp_kernel<6, true, false, false, false, false, true, true>; break;
      case 8: kern = attn_fwd_pp_kernel<8, true, false, false, false, false, true, true>; break;
      case 16: kern = attn_fwd_pp_kernel<16, true, false, false, false, false, true, true>; break;
      default: break;
    }
    static std::once_flag femu;
    std::call_once(femu, [] {
      for (auto k : {attn_fwd_pp_kernel<6, true, false, false, false, false, true, true>,
                     attn_fwd_pp_kernel<8, true, false, false, false, false, true, true>,
                     attn_fwd_pp_kernel<16, true, false, false, false, false, true, true>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPpSmem::BYTES);
    });
#endif
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, a.o, a.lse, a.S, a.H, scale_log2);
    if (e != cudaSuccess) return e;
  } else if (a.D == 128 && a.S % (2 * TILE) == 0) {
    // ping-pong: two query tiles per CTA, setmaxnreg, 1/3 of the exponentials
    // on the FMA pipe (paired exp2_fma2)
    static std::once_flag f8;
    std::call_once(f8, [] {
      cudaFuncSetAttribute(attn_fwd_pp_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPpSmem::BYTES);
    });
    attn_fwd_pp_kernel<3><<<dim3(a.S / (2 * TILE), a.H), 384, FwdPpSmem::BYTES, stream>>>(mq, mk, mv, a.o, a.lse,
                                                                                        a.S, a.H, scale_log2);
  } else if (a.D == 128) {  // an odd number of query tiles: one tile per CTA
    launch_fwd<128, true, true>(a, mq, mk, mv, scale_log2, stream);
  } else {
    launch_fwd<64, true, true>(a, mq, mk, mv, scale_log2, stream);
  }
  if (a.ev[1]) record_timing_event(a.ev[1], stream);
  return cudaGetLastError();
}

}  // namespace memo

namespace memo {
size_t attn_bwd_workspace_bytes(int S, int H, int D) {
  const size_t HS = static_cast<size_t>(H) * S;
  size_t b = 2 * HS * sizeof(float);  // delta, lse2
#ifdef MEMO_ATTN_ABLATIONS
  if (D == 128 && bwd_fused())  // f32 dQ accumulator, ordering counters, ticket
    b += HS * D * sizeof(float) + (HS / HALF + 4) * sizeof(uint32_t);
#endif
  return b;
}

cudaError_t attn_bwd(const AttnBwdArgs& a, cudaStream_t stream) {
  if (a.S % TILE != 0) return cudaErrorInvalidValue;
#ifdef MEMO_ATTN_ABLATIONS
  if (a.D == 128 && bwd_fused()) return launch_bwd_fused(a, stream);
#endif
  if (a.D == 128) return launch_bwd<128>(a, stream);
  if (a.D == 64) return launch_bwd<64>(a, stream);
  return cudaErrorInvalidValue;
}
#ifdef MEMO_FWD_PROF
extern "C" int memo_debug_fwd_prof(unsigned long long* out24, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out24, g_fwd_prof, 24 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(g_fwd_prof, z, sizeof(z));
  }
  return 0;
}
#endif
#ifdef MEMO_DKDV_PROF
extern "C" int memo_debug_dkdv_prof(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, g_dkdv_prof, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_dkdv_prof, z, sizeof(z));
  }
  return 0;
}
#endif
}  // namespace memo
