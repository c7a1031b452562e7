// Throughput of the instructions the attention softmax is made of, per SMSP,
// on this B200: MUFU.EX2, FFMA2 (fma.rn.f32x2), FADD2, FMNMX3, F2FP (bf16x2
// pack), and the mixes the kernels issue.  One CTA per SM, W warps per SMSP,
// each warp runs 8 independent chains of the op; cycles per warp-instruction
// per SMSP = elapsed clock64 / (instructions issued per SMSP).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/ubench_sfu tools/ubench_sfu.cu
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;

template <int OP>
__global__ void kern(float* out, long long* cyc) {
  float a[8];
  uint64_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = -1.f - 0.001f * (threadIdx.x + i);
    v[i] = (static_cast<uint64_t>(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i] * 0.5f);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // MUFU.EX2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (OP == 1) {  // FFMA2
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v[i]));
      } else if (OP == 2) {  // FADD2
        asm volatile("add.f32x2 %0, %0, %0;" : "+l"(v[i]));
      } else if (OP == 3) {  // FMNMX3
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      } else if (OP == 4) {  // F2FP pack
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 3) & 7]));
        a[i] = __uint_as_float(r);
      } else if (OP == 5) {  // FFMA (scalar)
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      } else if (OP == 6) {  // MUFU + FFMA2 interleaved (1:1)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v[i]));
      } else if (OP == 8) {  // MUFU.EX2 on f16x2 (two exponentials per lane)
        uint32_t r = __float_as_uint(a[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r));
        a[i] = __uint_as_float(r);
      } else if (OP == 9) {  // MUFU.EX2 on bf16x2
        uint32_t r = __float_as_uint(a[i]);
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r));
        a[i] = __uint_as_float(r);
      } else if (OP == 7) {  // MUFU + FMNMX3 + F2FP (1:1:1)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(i + 1) & 7]), "f"(a[(i + 3) & 7]));
        float b = __uint_as_float(r);
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(b) : "f"(a[(i + 5) & 7]), "f"(a[(i + 6) & 7]));
        a[(i + 4) & 7] += b * 0.f;
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(static_cast<uint32_t>(v[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int wps, float* out, long long* cyc, int n_sm) {
  const int threads = 32 * 4 * wps;
  kern<OP><<<n_sm, threads>>>(out, cyc);
  kern<OP><<<n_sm, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, n_sm * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < n_sm; ++i) avg += h[i];
  avg /= n_sm;
  const double instr_per_smsp = static_cast<double>(ITERS) * 8 * wps * (OP == 6 ? 2 : OP == 7 ? 3 : 1);
  printf("{\"op\": \"%s\", \"warps_per_smsp\": %d, \"cycles_per_warp_instr\": %.3f}\n", name, wps,
         avg / instr_per_smsp);
}

int main() {
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, n_sm * 1024 * sizeof(float));
  cudaMalloc(&cyc, n_sm * sizeof(long long));
  for (int w : {1, 2, 4}) {
    run<0>("MUFU.EX2", w, out, cyc, n_sm);
    run<1>("FFMA2", w, out, cyc, n_sm);
    run<2>("FADD2", w, out, cyc, n_sm);
    run<3>("FMNMX3", w, out, cyc, n_sm);
    run<4>("F2FP.BF16", w, out, cyc, n_sm);
    run<5>("FFMA", w, out, cyc, n_sm);
    run<6>("EX2+FFMA2", w, out, cyc, n_sm);
    run<7>("EX2+F2FP+FMNMX3+FFMA", w, out, cyc, n_sm);
    run<8>("EX2.F16x2", w, out, cyc, n_sm);
    run<9>("EX2.BF16x2", w, out, cyc, n_sm);
  }
  return 0;
}
