// MUFU throughput probe: tanh.approx vs ex2.approx vs rcp.approx vs an
// FMA-only sigmoid, 148 x 1024 threads, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_bench.cu -o /tmp/mufu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void probe(float *out, int iters) {
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = 0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float y;
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[j]));
      if (OP == 3) {  // ex2 + FMA Newton reciprocal: 1 / (1 + e)
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(v[j]));
        const float d = 1.f + e;
        float r = __int_as_float(0x7EF311C3 - __float_as_int(d));
        r = r * (2.f - d * r);
        r = r * (2.f - d * r);
        y = r;
      }
      v[j] = y * 0.5f + 0.25f;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
float run(float *out, int iters) {
  probe<OP><<<148 * 2, 512>>>(out, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<OP><<<148 * 2, 512>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  float *out;
  cudaMalloc(&out, 148 * 2 * 512 * sizeof(float));
  const int iters = 4096;
  const double ops = 148.0 * 2 * 512 * 8 * iters;
  const char *names[] = {"tanh.approx", "ex2.approx", "rcp.approx", "ex2+fma-rcp"};
  float t[4] = {run<0>(out, iters), run<1>(out, iters), run<2>(out, iters), run<3>(out, iters)};
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int i = 0; i < 4; ++i)
    printf("%-12s %8.3f ms  %7.1f Gop/s  %5.2f op/clk/SM (at %d MHz max)\n", names[i], t[i],
           ops / t[i] / 1e6, ops / (t[i] * 1e-3) / (clk * 1e3) / 148, clk / 1000);
  return 0;
}
