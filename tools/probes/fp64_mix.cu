// FP64 pipe probe: DFMA alone, DMMA alone (4 and 8 accumulators), and both
// interleaved in the same warps -- do DMMA and DFMA share one pipe on B200?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int ND>
__global__ void __launch_bounds__(256) mix_kernel(double* sink, int iters) {
  double a[NF > 0 ? NF : 1];
#pragma unroll
  for (int k = 0; k < NF; ++k) a[k] = 1.0 + 1e-7 * (threadIdx.x + 37 * k);
  const double b = 0.9999999999, c = 1e-12;
  double x = 1.0 + 1e-9 * threadIdx.x, y = 0.5 - 1e-9 * threadIdx.x;
  double acc[ND > 0 ? ND : 1][2];
#pragma unroll
  for (int u = 0; u < ND; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < ND; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(x), "d"(y));
#pragma unroll
    for (int k = 0; k < NF; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NF; ++k) s += a[k];
#pragma unroll
  for (int u = 0; u < ND; ++u) s += acc[u][0] + acc[u][1];
  if (s == 123.456) sink[0] = s;
}

template <int NF, int ND>
void run(const char* name, double* sink, int nsm) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0, bf = 0, bd = 0;
  for (int blocks : {nsm * 2, nsm * 4, nsm * 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      mix_kernel<NF, ND><<<blocks, 256>>>(sink, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = blocks * 8.0;
      const double ff = warps * 32 * NF * 2.0 * iters;   // DFMA flops
      const double fd = warps * ND * 512.0 * iters;      // DMMA flops
      const double t = (ff + fd) / (ms * 1e-3) / 1e12;
      if (t > best) { best = t; bf = ff / (ms * 1e-3) / 1e12; bd = fd / (ms * 1e-3) / 1e12; }
    }
  }
  printf("{\"probe\": \"%s\", \"dfma_chains\": %d, \"dmma_chains\": %d, \"total_tflops\": %.2f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f}\n",
         name, NF, ND, best, bf, bd);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  run<8, 0>("dfma", sink, nsm);
  run<16, 0>("dfma16", sink, nsm);
  run<0, 4>("dmma4", sink, nsm);
  run<0, 8>("dmma8", sink, nsm);
  run<8, 4>("mix_8f_4d", sink, nsm);
  run<16, 4>("mix_16f_4d", sink, nsm);
  run<8, 8>("mix_8f_8d", sink, nsm);
  run<4, 8>("mix_4f_8d", sink, nsm);
  return 0;
}
