// Shared-memory wavefronts per warp-wide LDS.64 / LDS.128 for lane->address
// patterns (read the counts with ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared.sum).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_wf lds_wf.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int chunk(int pat, int lane) {
  switch (pat) {
    case 0: return lane / 6;            // contiguous broadcast groups of 6 (axis-1 pencil)
    case 1: return lane % 6;            // strided groups (axis-0 column)
    case 2: return lane % 8;
    case 3: return lane / 4;
    case 4: return lane;                // all distinct
    case 5: return lane % 2;
    case 6: return lane % 4;
    case 7: return lane / 8;
    case 8: return lane / 16;
    case 9: return (lane % 6) * 3;      // strided, spread banks
    case 10: return lane / 2;
    case 11: return (lane % 4) + 8 * (lane / 16);   // 2x4 tiles
    case 12: return 0;
    case 13: return (lane / 6) * 6;     // groups of 6, chunk stride 6 (48 B per row of 6 doubles... )
    default: return lane;
  }
}

template <int W>   // W = 8 (LDS.64) or 16 (LDS.128)
__global__ void lds_kernel(double* out, int pat, int iters) {
  __shared__ __align__(16) double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int c = chunk(pat, lane);
  double acc = 0;
  if (W == 8) {
    const volatile double* p = buf + c;
    for (int i = 0; i < iters; ++i) acc += p[(i & 7) * 64];
  } else {
    const volatile double2* p = reinterpret_cast<const double2*>(buf) + c;
    for (int i = 0; i < iters; ++i) { double2 v = const_cast<const double2&>(p[(i & 7) * 64]); acc += v.x + v.y; }
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  for (int pat = 0; pat <= 13; ++pat) {
    lds_kernel<8><<<1, 32>>>(out, pat, 1000);
    lds_kernel<16><<<1, 32>>>(out, pat, 1000);
  }
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
