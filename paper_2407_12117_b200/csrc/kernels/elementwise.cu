// elementwise.cu — the HBM-bound kernels of the Llama block (sm_100a).
//
// All row kernels use one warp per token row with 16-byte vectorised,
// coalesced loads (lane l touches bytes [16l, 16l+16) of every 512-byte
// stripe) and warp-shuffle reductions; grids are sized in multiples of the SM
// count.  Column reductions (RMSNorm weight gradients, loss) are two-pass and
// order-fixed, so every result is bit-reproducible run to run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "elementwise.h"
#include "sm100.cuh"
#include "tma_util.h"

namespace memo {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void load_bf16x4(const __nv_bfloat16* p, float (&f)[4]) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  f[0] = __bfloat162float(a.x);
  f[1] = __bfloat162float(a.y);
  f[2] = __bfloat162float(b.x);
  f[3] = __bfloat162float(b.y);
}
__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  uint2 u;
  u.x = dev::pack_bf16(a, b);
  u.y = dev::pack_bf16(c, d);
  *reinterpret_cast<uint2*>(p) = u;
}

int grid_for_rows(long long rows, int rows_per_block) {
  long long g = (rows + rows_per_block - 1) / rows_per_block;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------ init
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Bit-identical to oc_init (oracle/llama_cpu.c): explicit _rn intrinsics keep
// nvcc from contracting the norm-weight expression into an FMA.
__global__ void init_uniform_kernel(__nv_bfloat16* __restrict__ w, float* __restrict__ master,
                                    long long n, uint64_t seed, uint64_t tid, int is_norm) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix64(seed * 0x9E3779B97F4A7C15ULL + tid * 0xD1B54A32D192ED03ULL +
                                  static_cast<uint64_t>(i));
    const float u = __fmul_rn(static_cast<float>(h >> 40), 1.0f / 16777216.0f);
    const float x = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
    const float v = is_norm ? __fadd_rn(1.0f, __fmul_rn(x, 0.1f)) : __fmul_rn(x, 0.0346410161513775f);
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    w[i] = b;
    if (master) master[i] = __bfloat162float(b);
  }
}

// ------------------------------------------------------------------ embedding
__global__ void embed_fwd_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ E,
                                 float* __restrict__ x, int S, int h) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= S) return;
  const __nv_bfloat16* e = E + static_cast<long long>(tok[row]) * h;
  float* o = x + static_cast<long long>(row) * h;
  for (int j = lane * 4; j < h; j += 128) {
    float f[4];
    load_bf16x4(e + j, f);
    *reinterpret_cast<float4*>(o + j) = make_float4(f[0], f[1], f[2], f[3]);
  }
}

// dE[v] = sum over positions p of token v (CSR order) of dx[p]; rows without
// tokens are written as zero.  Deterministic (fixed summation order).
__global__ void embed_bwd_kernel(const int* __restrict__ offsets, const int* __restrict__ pos,
                                 const float* __restrict__ dx, float* __restrict__ dE, int V,
                                 int h) {
  const int v = blockIdx.x;
  if (v >= V) return;
  const int b = offsets[v], e = offsets[v + 1];
  for (int j = threadIdx.x * 4; j < h; j += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = b; k < e; ++k) {
      const float4 g = *reinterpret_cast<const float4*>(dx + static_cast<long long>(pos[k]) * h + j);
      acc.x += g.x;
      acc.y += g.y;
      acc.z += g.z;
      acc.w += g.w;
    }
    *reinterpret_cast<float4*>(dE + static_cast<long long>(v) * h + j) = acc;
  }
}

// ------------------------------------------------------------------ RMSNorm
// y = bf16(xin * rstd(xin) * g), xin = x (+ bf16 a).  Optionally copies xin
// to `xcopy` (f32) — used to land the embedding output in its rounding buffer.
template <int NV>  // NV = h / 128 float4 vectors per lane
__global__ void rmsnorm_fwd_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ a,
                                   const __nv_bfloat16* __restrict__ g, __nv_bfloat16* __restrict__ y,
                                   int S, int h, float eps) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= S) return;
  const float* xr = x + static_cast<long long>(row) * h;
  float v[NV][4];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = i * 128 + lane * 4;
    const float4 t = *reinterpret_cast<const float4*>(xr + j);
    v[i][0] = t.x;
    v[i][1] = t.y;
    v[i][2] = t.z;
    v[i][3] = t.w;
    if (a) {
      float f[4];
      load_bf16x4(a + static_cast<long long>(row) * h + j, f);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[i][e] += f[e];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) ss += v[i][e] * v[i][e];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / static_cast<float>(h) + eps);
  __nv_bfloat16* yr = y + static_cast<long long>(row) * h;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = i * 128 + lane * 4;
    float gg[4];
    load_bf16x4(g + j, gg);
    store_bf16x4(yr + j, v[i][0] * r * gg[0], v[i][1] * r * gg[1], v[i][2] * r * gg[2],
                 v[i][3] * r * gg[3]);
  }
}

// Backward of y = xin * r * g:
//   dx = dres + r*(dy*g) - xin * r^3 * mean(dy*g*xin)    (f32, may alias dres)
//   dx_bf16 = bf16(dx) (optional), partial_dg[block][j] = sum_rows dy*xin*r
// Two streaming passes per row (reductions, then outputs) keep registers low
// for any h; per-warp column accumulators live in dynamic shared memory and
// are folded in fixed warp order, then across blocks by dg_reduce.
constexpr int NORM_BWD_ROWS = 64;
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(
    const float* __restrict__ x, const __nv_bfloat16* __restrict__ a,
    const __nv_bfloat16* __restrict__ g, const float* __restrict__ dy, const float* dres,
    float* dx, __nv_bfloat16* __restrict__ dx_bf16, float* __restrict__ partial, int S, int h,
    float eps) {
  extern __shared__ float acc[];  // [8][h]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* my = acc + warp * h;
  for (int j = lane; j < h; j += 32) my[j] = 0.f;
  __syncwarp();
  const int row0 = blockIdx.x * NORM_BWD_ROWS;
  for (int rr = warp; rr < NORM_BWD_ROWS; rr += 8) {
    const int row = row0 + rr;
    if (row >= S) break;
    const long long base = static_cast<long long>(row) * h;
    float ss = 0.f, dot = 0.f;
    for (int j = lane * 4; j < h; j += 128) {
      const float4 t = *reinterpret_cast<const float4*>(x + base + j);
      float xv[4] = {t.x, t.y, t.z, t.w};
      if (a) {
        float f[4];
        load_bf16x4(a + base + j, f);
#pragma unroll
        for (int e = 0; e < 4; ++e) xv[e] += f[e];
      }
      const float4 d = *reinterpret_cast<const float4*>(dy + base + j);
      const float dv[4] = {d.x, d.y, d.z, d.w};
      float gg[4];
      load_bf16x4(g + j, gg);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ss += xv[e] * xv[e];
        dot += dv[e] * gg[e] * xv[e];
      }
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    const float r = rsqrtf(ss / static_cast<float>(h) + eps);
    const float c = r * r * r * dot / static_cast<float>(h);
    for (int j = lane * 4; j < h; j += 128) {
      const float4 t = *reinterpret_cast<const float4*>(x + base + j);
      float xv[4] = {t.x, t.y, t.z, t.w};
      if (a) {
        float f[4];
        load_bf16x4(a + base + j, f);
#pragma unroll
        for (int e = 0; e < 4; ++e) xv[e] += f[e];
      }
      const float4 d = *reinterpret_cast<const float4*>(dy + base + j);
      const float dv[4] = {d.x, d.y, d.z, d.w};
      float gg[4];
      load_bf16x4(g + j, gg);
      const float4 rs =
          dres ? *reinterpret_cast<const float4*>(dres + base + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float rv[4] = {rs.x, rs.y, rs.z, rs.w};
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[e] = rv[e] + (r * dv[e] * gg[e] - c * xv[e]);
        my[j + e] += dv[e] * xv[e] * r;
      }
      *reinterpret_cast<float4*>(dx + base + j) = make_float4(o[0], o[1], o[2], o[3]);
      if (dx_bf16) store_bf16x4(dx_bf16 + base + j, o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < h; j += 256) {
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += acc[w * h + j];
    partial[static_cast<long long>(blockIdx.x) * h + j] = sum;
  }
}

// Same contract, one HBM pass: a 256-thread block owns NORM_BWD_ROWS rows and
// every thread a fixed slice of 4*V consecutive columns (h = 1024*V), so the
// row (x, a, dy, dres) stays in registers between the reduction and the
// output, g is loaded once, and the dg accumulators live in registers.  The
// per-row (sum x^2, sum dy*g*x) reduction goes warp-shuffle -> 8 partials in
// shared memory read back in fixed order (deterministic).
template <int V>
__global__ void __launch_bounds__(256) rmsnorm_bwd_reg_kernel(
    const float* __restrict__ x, const __nv_bfloat16* __restrict__ a,
    const __nv_bfloat16* __restrict__ g, const float* __restrict__ dy, const float* dres,
    float* dx, __nv_bfloat16* __restrict__ dx_bf16, float* __restrict__ partial, int S, float eps) {
  constexpr int h = 1024 * V;
  __shared__ float red[2][2][8];  // [row parity][ss|dot][warp]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = threadIdx.x * 4;  // columns c0 + 1024*v .. +3
  float gg[V][4], acc[V][4];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    load_bf16x4(g + c0 + 1024 * v, gg[v]);
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[v][e] = 0.f;
  }
  const int row0 = blockIdx.x * NORM_BWD_ROWS;
  for (int rr = 0; rr < NORM_BWD_ROWS; ++rr) {
    const int row = row0 + rr;
    if (row >= S) break;
    const long long base = static_cast<long long>(row) * h + c0;
    float xv[V][4], dv[V][4];
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float4 t = *reinterpret_cast<const float4*>(x + base + 1024 * v);
      const float4 d = *reinterpret_cast<const float4*>(dy + base + 1024 * v);
      xv[v][0] = t.x; xv[v][1] = t.y; xv[v][2] = t.z; xv[v][3] = t.w;
      dv[v][0] = d.x; dv[v][1] = d.y; dv[v][2] = d.z; dv[v][3] = d.w;
      if (a) {
        float f[4];
        load_bf16x4(a + base + 1024 * v, f);
#pragma unroll
        for (int e = 0; e < 4; ++e) xv[v][e] += f[e];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ss += xv[v][e] * xv[v][e];
        dot += dv[v][e] * gg[v][e] * xv[v][e];
      }
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    const int par = rr & 1;
    if (lane == 0) {
      red[par][0][warp] = ss;
      red[par][1][warp] = dot;
    }
    __syncthreads();  // the other parity buffer makes one barrier per row enough
    ss = 0.f;
    dot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      ss += red[par][0][w];
      dot += red[par][1][w];
    }
    const float r = rsqrtf(ss / static_cast<float>(h) + eps);
    const float c = r * r * r * dot / static_cast<float>(h);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float rv[4] = {0.f, 0.f, 0.f, 0.f};
      if (dres) {
        const float4 q = *reinterpret_cast<const float4*>(dres + base + 1024 * v);
        rv[0] = q.x; rv[1] = q.y; rv[2] = q.z; rv[3] = q.w;
      }
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[e] = rv[e] + (r * dv[v][e] * gg[v][e] - c * xv[v][e]);
        acc[v][e] += dv[v][e] * xv[v][e] * r;
      }
      *reinterpret_cast<float4*>(dx + base + 1024 * v) = make_float4(o[0], o[1], o[2], o[3]);
      if (dx_bf16) store_bf16x4(dx_bf16 + base + 1024 * v, o[0], o[1], o[2], o[3]);
    }
  }
  float* prow = partial + static_cast<long long>(blockIdx.x) * h + c0;
#pragma unroll
  for (int v = 0; v < V; ++v)
    *reinterpret_cast<float4*>(prow + 1024 * v) = make_float4(acc[v][0], acc[v][1], acc[v][2], acc[v][3]);
}

// dg[j] (=|+=) sum_p partial[p][j] in fixed order.
__global__ void dg_reduce_kernel(const float* __restrict__ partial, float* __restrict__ dg, int P,
                                 int h, int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= h) return;
  float s = 0.f;
  for (int p = 0; p < P; ++p) s += partial[static_cast<long long>(p) * h + j];
  dg[j] = accumulate ? dg[j] + s : s;
}

// ------------------------------------------------------------------ SwiGLU
// gu rows = [gate(F) | up(F)];  act = bf16(silu(g) * u)
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                  long long S, int F) {
  const long long n4 = S * F / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = i * 4;
    const long long t = e / F;
    const int j = static_cast<int>(e - t * F);
    float gv[4], uv[4];
    load_bf16x4(gu + t * 2 * F + j, gv);
    load_bf16x4(gu + t * 2 * F + F + j, uv);
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = gv[k] / (1.f + __expf(-gv[k])) * uv[k];
    store_bf16x4(act + e, o[0], o[1], o[2], o[3]);
  }
}

// Row-major variants (F % 8 == 0): blocks stride over rows, threads over
// 8-column vectors -- no 64-bit division per element, 16-byte accesses.  Same
// per-element formulas as the flat kernels (bitwise-identical results).
__device__ __forceinline__ void load_bf16x8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    f[2 * i] = __bfloat162float(v.x);
    f[2 * i + 1] = __bfloat162float(v.y);
  }
}
__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 u;
  u.x = dev::pack_bf16(f[0], f[1]);
  u.y = dev::pack_bf16(f[2], f[3]);
  u.z = dev::pack_bf16(f[4], f[5]);
  u.w = dev::pack_bf16(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

__global__ void swiglu_fwd_rows_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                       long long S, int F) {
  for (long long t = blockIdx.x; t < S; t += gridDim.x) {
    const __nv_bfloat16* g = gu + t * 2 * F;
    for (int j = threadIdx.x * 8; j < F; j += blockDim.x * 8) {
      float gv[8], uv[8], o[8];
      load_bf16x8(g + j, gv);
      load_bf16x8(g + F + j, uv);
#pragma unroll
      // silu(g) * u = g * u / (1 + e^-g); the approximate divide (2 ulp) is far
      // inside the bf16 output's rounding and keeps this kernel on HBM speed
      for (int k = 0; k < 8; ++k) o[k] = __fdividef(gv[k] * uv[k], 1.f + __expf(-gv[k]));
      store_bf16x8(act + t * F + j, o);
    }
  }
}

__global__ void swiglu_bwd_rows_kernel(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ dact,
                                       __nv_bfloat16* __restrict__ dgu, long long S, int F) {
  for (long long t = blockIdx.x; t < S; t += gridDim.x) {
    const __nv_bfloat16* g = gu + t * 2 * F;
    for (int j = threadIdx.x * 8; j < F; j += blockDim.x * 8) {
      float gv[8], uv[8], dv[8], dg[8], du[8];
      load_bf16x8(g + j, gv);
      load_bf16x8(g + F + j, uv);
      load_bf16x8(dact + t * F + j, dv);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float sg = __fdividef(1.f, 1.f + __expf(-gv[k]));
        du[k] = dv[k] * gv[k] * sg;
        dg[k] = dv[k] * uv[k] * sg * (1.f + gv[k] * (1.f - sg));
      }
      store_bf16x8(dgu + t * 2 * F + j, dg);
      store_bf16x8(dgu + t * 2 * F + F + j, du);
    }
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                  const __nv_bfloat16* __restrict__ dact,
                                  __nv_bfloat16* __restrict__ dgu, long long S, int F) {
  const long long n4 = S * F / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = i * 4;
    const long long t = e / F;
    const int j = static_cast<int>(e - t * F);
    float gv[4], uv[4], dv[4];
    load_bf16x4(gu + t * 2 * F + j, gv);
    load_bf16x4(gu + t * 2 * F + F + j, uv);
    load_bf16x4(dact + e, dv);
    float dg[4], du[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sg = 1.f / (1.f + __expf(-gv[k]));
      du[k] = dv[k] * gv[k] * sg;
      dg[k] = dv[k] * uv[k] * sg * (1.f + gv[k] * (1.f - sg));
    }
    store_bf16x4(dgu + t * 2 * F + j, dg[0], dg[1], dg[2], dg[3]);
    store_bf16x4(dgu + t * 2 * F + F + j, du[0], du[1], du[2], du[3]);
  }
}

// ------------------------------------------------------------------ cross-entropy
// One block per token row of f32 logits: loss_row = lse - logit[label];
// dlogits = bf16((softmax - onehot) * inv_n); rows with label < 0 give zeros.
// inv_n = 1 / (labeled tokens of the batch) is read from device memory: it is
// written with each batch's H2D, so a captured CUDA graph replays the current
// batch's scale, not the capture-time one.
__global__ void __launch_bounds__(256) ce_kernel(const float* __restrict__ logits,
                                                 const int* __restrict__ labels,
                                                 __nv_bfloat16* __restrict__ dlogits,
                                                 float* __restrict__ loss_rows, int V,
                                                 const float* __restrict__ inv_n_dev) {
  const int row = blockIdx.x;
  const float inv_n = *inv_n_dev;
  const float* lr = logits + static_cast<long long>(row) * V;
  __nv_bfloat16* dr = dlogits + static_cast<long long>(row) * V;
  const int label = labels[row];
  __shared__ float sh[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (label < 0) {
    for (int j = threadIdx.x * 4; j < V; j += 1024) store_bf16x4(dr + j, 0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) loss_rows[row] = 0.f;
    return;
  }
  float mx = -INFINITY;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    mx = fmaxf(mx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
  }
  mx = warp_max(mx);
  if (lane == 0) sh[warp] = mx;
  __syncthreads();
  mx = sh[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, sh[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    sum += __expf(t.x - mx) + __expf(t.y - mx) + __expf(t.z - mx) + __expf(t.w - mx);
  }
  sum = warp_sum(sum);
  if (lane == 0) sh[warp] = sum;
  __syncthreads();
  sum = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) sum += sh[w];
  const float inv_sum = 1.f / sum;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    float p[4] = {__expf(t.x - mx) * inv_sum, __expf(t.y - mx) * inv_sum,
                  __expf(t.z - mx) * inv_sum, __expf(t.w - mx) * inv_sum};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (j + k == label) p[k] -= 1.f;
    store_bf16x4(dr + j, p[0] * inv_n, p[1] * inv_n, p[2] * inv_n, p[3] * inv_n);
  }
  if (threadIdx.x == 0) loss_rows[row] = (mx + logf(sum)) - lr[label];
}

// Deterministic single-block sum of n floats into out[0], times `scale`.
__global__ void sum_kernel(const float* __restrict__ v, long long n,
                           const float* __restrict__ scale, float* __restrict__ out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = static_cast<float>(sh[0] * *scale);
}

// ------------------------------------------------------------------ optimizer
// t += 1; bias corrections of step t (double, rounded once)
__global__ void adam_step_kernel(int* step, float2* c12, float b1, float b2) {
  const int t = ++*step;
  *c12 = make_float2(static_cast<float>(1.0 / (1.0 - pow(static_cast<double>(b1), t))),
                     static_cast<float>(1.0 / (1.0 - pow(static_cast<double>(b2), t))));
}

// Fused AdamW over the flat parameter buffer: f32 master/m/v, bf16 working copy.
__global__ void adamw_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w,
                             const float* __restrict__ grad, float* __restrict__ m,
                             float* __restrict__ v, long long n, float lr, float b1, float b2,
                             float eps, float wd, const float2* __restrict__ c12) {
  const float c1 = c12->x, c2 = c12->y;
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 p = reinterpret_cast<float4*>(master)[i];
    const float4 g = reinterpret_cast<const float4*>(grad)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* pp = &p.x;
    const float* gg = &g.x;
    float* mp = &mm.x;
    float* vp = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mp[k] = b1 * mp[k] + (1.f - b1) * gg[k];
      vp[k] = b2 * vp[k] + (1.f - b2) * gg[k] * gg[k];
      const float mh = mp[k] * c1, vh = vp[k] * c2;
      pp[k] -= lr * (mh / (sqrtf(vh) + eps) + wd * pp[k]);
    }
    reinterpret_cast<float4*>(master)[i] = p;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    store_bf16x4(w + i * 4, p.x, p.y, p.z, p.w);
  }
}


// ------------------------------------------------------------------ tensor-parallel helpers
// Counter-hash init of a shard: local [R_l, C_l] whose rows map to global rows
// through up to three contiguous segments; identical values to the full init.
struct RowSegs {
  long long local0[3], count[3], global0[3];
  int n;
};
__global__ void init_sliced_kernel(__nv_bfloat16* __restrict__ w, float* __restrict__ master,
                                   long long R, long long C, RowSegs segs, long long C_glob,
                                   long long c_off, uint64_t seed, uint64_t tid, int is_norm) {
  const long long n = R * C;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / C, c = i - r * C;
    long long gr = r;
    for (int k = 0; k < segs.n; ++k)
      if (r >= segs.local0[k] && r < segs.local0[k] + segs.count[k]) gr = segs.global0[k] + (r - segs.local0[k]);
    const uint64_t gi = static_cast<uint64_t>(gr * C_glob + c_off + c);
    const uint64_t h = splitmix64(seed * 0x9E3779B97F4A7C15ULL + tid * 0xD1B54A32D192ED03ULL + gi);
    const float u = __fmul_rn(static_cast<float>(h >> 40), 1.0f / 16777216.0f);
    const float x = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
    const float v = is_norm ? __fadd_rn(1.0f, __fmul_rn(x, 0.1f)) : __fmul_rn(x, 0.0346410161513775f);
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    w[i] = b;
    if (master) master[i] = __bfloat162float(b);
  }
}

// out = x + bf16(a) ; a_bf16 = bf16(a) (optional).  The reduce-scattered
// projection output becomes the bf16 skeletal tensor the residual adds.
__global__ void resid_round_kernel(const float* __restrict__ x, const float* __restrict__ a,
                                   __nv_bfloat16* __restrict__ a_bf16, float* __restrict__ out,
                                   long long n4) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 xv = reinterpret_cast<const float4*>(x)[i];
    const float4 av = reinterpret_cast<const float4*>(a)[i];
    const float r0 = dev::bf16_round(av.x), r1 = dev::bf16_round(av.y), r2 = dev::bf16_round(av.z),
                r3 = dev::bf16_round(av.w);
    if (a_bf16) store_bf16x4(a_bf16 + i * 4, r0, r1, r2, r3);
    reinterpret_cast<float4*>(out)[i] = make_float4(xv.x + r0, xv.y + r1, xv.z + r2, xv.w + r3);
  }
}

// Vocab-parallel cross-entropy on a shard of V_l logits per row (columns
// v0..v0+V_l of the full vocabulary): three passes around two all-reduces.
__global__ void __launch_bounds__(256) ce_vp_max_kernel(const float* __restrict__ logits,
                                                        float* __restrict__ rmax, int V) {
  const float* lr = logits + static_cast<long long>(blockIdx.x) * V;
  __shared__ float sh[8];
  float mx = -INFINITY;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    mx = fmaxf(mx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = sh[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, sh[w]);
    rmax[blockIdx.x] = m;
  }
}
// stats[row] = sum exp(x - max) over the shard; stats[T + row] = target logit if owned, else 0
__global__ void __launch_bounds__(256) ce_vp_sum_kernel(const float* __restrict__ logits,
                                                        const float* __restrict__ gmax,
                                                        const int* __restrict__ labels, int v0,
                                                        float* __restrict__ stats, int T, int V) {
  const int row = blockIdx.x;
  const float* lr = logits + static_cast<long long>(row) * V;
  const float m = gmax[row];
  __shared__ float sh[8];
  float sum = 0.f;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    sum += __expf(t.x - m) + __expf(t.y - m) + __expf(t.z - m) + __expf(t.w - m);
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += sh[w];
    stats[row] = s;
    const int lab = labels[row] - v0;
    stats[T + row] = (labels[row] >= 0 && lab >= 0 && lab < V) ? lr[lab] : 0.f;
  }
}
__global__ void __launch_bounds__(256) ce_vp_grad_kernel(const float* __restrict__ logits,
                                                         const float* __restrict__ gmax,
                                                         const float* __restrict__ gstats,
                                                         const int* __restrict__ labels, int v0,
                                                         __nv_bfloat16* __restrict__ dlogits,
                                                         float* __restrict__ loss_rows, int T, int V,
                                                         const float* __restrict__ inv_n_dev) {
  const int row = blockIdx.x;
  const float inv_n = *inv_n_dev;
  const float* lr = logits + static_cast<long long>(row) * V;
  __nv_bfloat16* dr = dlogits + static_cast<long long>(row) * V;
  const int label = labels[row];
  if (label < 0) {
    for (int j = threadIdx.x * 4; j < V; j += 1024) store_bf16x4(dr + j, 0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) loss_rows[row] = 0.f;
    return;
  }
  const float m = gmax[row], inv_sum = 1.f / gstats[row];
  const int lab = label - v0;
  for (int j = threadIdx.x * 4; j < V; j += 1024) {
    const float4 t = *reinterpret_cast<const float4*>(lr + j);
    float p[4] = {__expf(t.x - m) * inv_sum, __expf(t.y - m) * inv_sum, __expf(t.z - m) * inv_sum,
                  __expf(t.w - m) * inv_sum};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (j + k == lab) p[k] -= 1.f;
    store_bf16x4(dr + j, p[0] * inv_n, p[1] * inv_n, p[2] * inv_n, p[3] * inv_n);
  }
  if (threadIdx.x == 0) loss_rows[row] = (m + logf(gstats[row])) - gstats[T + row];
}

int stride_grid(long long n, int per_thread, int threads) {
  const long long want = (n / per_thread + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms()) * 16;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

cudaError_t init_sliced(__nv_bfloat16* w, float* master, long long R, long long C,
                        const long long* local0, const long long* count, const long long* global0,
                        int nseg, long long C_glob, long long c_off, uint64_t seed, uint64_t tid,
                        bool is_norm, cudaStream_t st) {
  RowSegs segs{};
  segs.n = nseg;
  for (int k = 0; k < nseg && k < 3; ++k) {
    segs.local0[k] = local0[k];
    segs.count[k] = count[k];
    segs.global0[k] = global0[k];
  }
  init_sliced_kernel<<<stride_grid(R * C, 1, 256), 256, 0, st>>>(w, master, R, C, segs, C_glob, c_off,
                                                                 seed, tid, is_norm);
  return cudaGetLastError();
}

cudaError_t resid_round(const float* x, const float* a, __nv_bfloat16* a_bf16, float* out,
                        long long n, cudaStream_t st) {
  if (n % 4) return cudaErrorInvalidValue;
  resid_round_kernel<<<stride_grid(n, 4, 256), 256, 0, st>>>(x, a, a_bf16, out, n / 4);
  return cudaGetLastError();
}

cudaError_t ce_vp_max(const float* logits, float* rmax, int T, int V, cudaStream_t st) {
  ce_vp_max_kernel<<<T, 256, 0, st>>>(logits, rmax, V);
  return cudaGetLastError();
}
cudaError_t ce_vp_sum(const float* logits, const float* gmax, const int* labels, int v0,
                      float* stats, int T, int V, cudaStream_t st) {
  ce_vp_sum_kernel<<<T, 256, 0, st>>>(logits, gmax, labels, v0, stats, T, V);
  return cudaGetLastError();
}
cudaError_t ce_vp_grad(const float* logits, const float* gmax, const float* gstats,
                       const int* labels, int v0, __nv_bfloat16* dlogits, float* loss_rows, int T,
                       int V, const float* inv_n, cudaStream_t st) {
  ce_vp_grad_kernel<<<T, 256, 0, st>>>(logits, gmax, gstats, labels, v0, dlogits, loss_rows, T, V, inv_n);
  return cudaGetLastError();
}

cudaError_t init_uniform(__nv_bfloat16* w, float* master, long long n, uint64_t seed,
                         uint64_t tid, bool is_norm, cudaStream_t st) {
  init_uniform_kernel<<<stride_grid(n, 1, 256), 256, 0, st>>>(w, master, n, seed, tid, is_norm);
  return cudaGetLastError();
}

cudaError_t embed_fwd(const int* tok, const __nv_bfloat16* E, float* x, int S, int h,
                      cudaStream_t st) {
  if (h % 128) return cudaErrorInvalidValue;
  embed_fwd_kernel<<<grid_for_rows(S, 8), 256, 0, st>>>(tok, E, x, S, h);
  return cudaGetLastError();
}

cudaError_t embed_bwd(const int* offsets, const int* pos, const float* dx, float* dE, int V,
                      int h, cudaStream_t st) {
  embed_bwd_kernel<<<V, 128, 0, st>>>(offsets, pos, dx, dE, V, h);
  return cudaGetLastError();
}

cudaError_t rmsnorm_fwd(const float* x, const __nv_bfloat16* a, const __nv_bfloat16* g,
                        __nv_bfloat16* y, int S, int h, float eps, cudaStream_t st) {
  if (h % 128) return cudaErrorInvalidValue;
  const int grid = grid_for_rows(S, 8);
  switch (h / 128) {
    case 2: rmsnorm_fwd_kernel<2><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    case 4: rmsnorm_fwd_kernel<4><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    case 8: rmsnorm_fwd_kernel<8><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    case 16: rmsnorm_fwd_kernel<16><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    case 32: rmsnorm_fwd_kernel<32><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    case 40: rmsnorm_fwd_kernel<40><<<grid, 256, 0, st>>>(x, a, g, y, S, h, eps); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int rmsnorm_bwd_partials(int S) { return (S + NORM_BWD_ROWS - 1) / NORM_BWD_ROWS; }

cudaError_t rmsnorm_bwd(const float* x, const __nv_bfloat16* a, const __nv_bfloat16* g,
                        const float* dy, const float* dres, float* dx, __nv_bfloat16* dx_bf16,
                        float* partial, float* dg, int S, int h, float eps, bool accumulate_dg,
                        cudaStream_t st) {
  if (h % 128) return cudaErrorInvalidValue;
  const int P = rmsnorm_bwd_partials(S);
  const int smem = 8 * h * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rmsnorm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  switch (h) {  // register-resident single-pass variant for the model widths
    case 4096:
      rmsnorm_bwd_reg_kernel<4><<<P, 256, 0, st>>>(x, a, g, dy, dres, dx, dx_bf16, partial, S, eps);
      break;
    case 5120:
      rmsnorm_bwd_reg_kernel<5><<<P, 256, 0, st>>>(x, a, g, dy, dres, dx, dx_bf16, partial, S, eps);
      break;
    case 8192:
      rmsnorm_bwd_reg_kernel<8><<<P, 256, 0, st>>>(x, a, g, dy, dres, dx, dx_bf16, partial, S, eps);
      break;
    default:
      rmsnorm_bwd_kernel<<<P, 256, smem, st>>>(x, a, g, dy, dres, dx, dx_bf16, partial, S, h, eps);
  }
  dg_reduce_kernel<<<(h + 255) / 256, 256, 0, st>>>(partial, dg, P, h, accumulate_dg);
  return cudaGetLastError();
}

cudaError_t swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* act, long long S, int F,
                       cudaStream_t st) {
  if (F % 4) return cudaErrorInvalidValue;
  if (F % 8 == 0) {
    const long long g = S < 148LL * 8 ? S : 148LL * 8;
    swiglu_fwd_rows_kernel<<<static_cast<int>(g > 0 ? g : 1), 256, 0, st>>>(gu, act, S, F);
    return cudaGetLastError();
  }
  swiglu_fwd_kernel<<<stride_grid(S * F, 4, 256), 256, 0, st>>>(gu, act, S, F);
  return cudaGetLastError();
}

cudaError_t swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* dact, __nv_bfloat16* dgu,
                       long long S, int F, cudaStream_t st) {
  if (F % 4) return cudaErrorInvalidValue;
  if (F % 8 == 0) {
    const long long g = S < 148LL * 8 ? S : 148LL * 8;
    swiglu_bwd_rows_kernel<<<static_cast<int>(g > 0 ? g : 1), 256, 0, st>>>(gu, dact, dgu, S, F);
    return cudaGetLastError();
  }
  swiglu_bwd_kernel<<<stride_grid(S * F, 4, 256), 256, 0, st>>>(gu, dact, dgu, S, F);
  return cudaGetLastError();
}

cudaError_t cross_entropy(const float* logits, const int* labels, __nv_bfloat16* dlogits,
                          float* loss_rows, int T, int V, const float* inv_n, cudaStream_t st) {
  if (V % 4) return cudaErrorInvalidValue;
  ce_kernel<<<T, 256, 0, st>>>(logits, labels, dlogits, loss_rows, V, inv_n);
  return cudaGetLastError();
}

cudaError_t sum_scaled(const float* v, long long n, const float* scale, float* out, cudaStream_t st) {
  sum_kernel<<<1, 1024, 0, st>>>(v, n, scale, out);
  return cudaGetLastError();
}

cudaError_t adamw(float* master, __nv_bfloat16* w, const float* grad, float* m, float* v,
                  long long n, float lr, float b1, float b2, float eps, float wd, int* step,
                  float2* c12, cudaStream_t st) {
  if (n % 4) return cudaErrorInvalidValue;
  adam_step_kernel<<<1, 1, 0, st>>>(step, c12, b1, b2);
  adamw_kernel<<<stride_grid(n, 4, 256), 256, 0, st>>>(master, w, grad, m, v, n, lr, b1, b2, eps,
                                                       wd, c12);
  return cudaGetLastError();
}

}  // namespace memo
