// tcgen05.mma throughput by shape on this B200: one CTA per SM, one converged
// warp issuing REPS back-to-back MMAs (TS: A from TMEM, B from shared memory;
// SS: both from shared memory), one commit, one wait.  Prints cycles per MMA
// against the ideal M*N*K*2 / 8192 FLOP per SM-cycle, for the small-N shapes
// the attention backward uses (dK/dV: M128 N32 K16 TS; dQ: N64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2407_12117_b200/csrc \
//        -o tools/_build/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include <cstdint>

#include "kernels/sm100.cuh"
namespace dev = memo::dev;

constexpr int REPS = 4096;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) kern(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t warp = dev::warp_id();
  if (threadIdx.x == 0) {
    dev::mbar_init(&bar, 1);
    dev::fence_barrier_init();
  }
  if (warp == 0) dev::tmem_alloc(&slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t idesc = dev::idesc_bf16_f32(128, N, false, false);
    const uint64_t bd = dev::umma_desc_sw128(dev::smem_u32(smem), 16, 1024);
    const uint64_t ad = dev::umma_desc_sw128(dev::smem_u32(smem + 65536), 16, 1024);
    // warm-up
    for (int i = 0; i < 64; ++i) {
      if (TS) dev::mma_bf16_ts_w(tmem, tmem + 256, bd, idesc, i > 0);
      else dev::mma_bf16_ss_w(tmem, ad, bd, idesc, i > 0);
    }
    dev::mma_commit_w(&bar);
    dev::mbar_wait_w(&bar, 0);
    const long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < REPS; ++i) {
      if (TS) dev::mma_bf16_ts_w(tmem, tmem + 256, bd + (i & 3) * 2, idesc, 1);
      else dev::mma_bf16_ss_w(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
    }
    dev::mma_commit_w(&bar);
    dev::mbar_wait_w(&bar, 1);
    const long long t1 = clock64();
    if (dev::lane_id() == 0) out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) dev::tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run(long long* d, int n_sm) {
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(kern<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<N, TS><<<n_sm, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[1024];
  cudaMemcpy(h, d, n_sm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < n_sm; ++i) avg += h[i];
  avg /= n_sm;
  const double ideal = 128.0 * N * 16 * 2 / 8192;
  printf("{\"shape\": \"M128 N%d K16 %s\", \"cycles_per_mma\": %.2f, \"ideal\": %.1f, \"efficiency\": %.3f}\n", N,
         TS ? "TS" : "SS", avg / REPS, ideal, ideal / (avg / REPS));
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, n_sm * sizeof(long long));
  run<16, true>(d, n_sm);
  run<32, true>(d, n_sm);
  run<64, true>(d, n_sm);
  run<128, true>(d, n_sm);
  run<256, true>(d, n_sm);
  run<32, false>(d, n_sm);
  run<64, false>(d, n_sm);
  run<128, false>(d, n_sm);
  run<256, false>(d, n_sm);
  return 0;
}
