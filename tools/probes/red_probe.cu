// Micro-benchmark: throughput of global vector reds into 32-byte cell records.
//   mode 0: each lane reds its own record with two red.v4 (the walk's flush)
//   mode 1: lane pairs: per instruction, lanes 2j and 2j+1 red the two halves of ONE
//           record (the pair's records A then B), after exchanging halves by shuffles
//   mode 2: each lane reds its own record with one red.v4 (half the bytes: a bound)
//   mode 3: lanes of a warp red records of consecutive cells (coalesced pattern)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__global__ void k(float* buf, unsigned ncell, int iters, int mode) {
  const unsigned lane = threadIdx.x & 31;
  unsigned h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = 1e-6f * (j + 1);
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    unsigned cell = mode == 3 ? ((h >> 5) + lane) % ncell : (h >> 3) % ncell;
    float* q = buf + 8ull * cell;
    if (mode == 0 || mode == 3) {
      red4(q, v[0], v[1], v[2], v[3]);
      red4(q + 4, v[4], v[5], v[6], v[7]);
    } else if (mode == 2) {
      red4(q, v[0], v[1], v[2], v[3]);
    } else {
      // pair (even, odd): even lane sends its hi half, odd lane its lo half
      const bool odd = lane & 1;
      float s0 = __shfl_xor_sync(~0u, odd ? v[0] : v[4], 1);
      float s1 = __shfl_xor_sync(~0u, odd ? v[1] : v[5], 1);
      float s2 = __shfl_xor_sync(~0u, odd ? v[2] : v[6], 1);
      float s3 = __shfl_xor_sync(~0u, odd ? v[3] : v[7], 1);
      unsigned long long qa = (unsigned long long)q;
      unsigned long long qo = __shfl_xor_sync(~0u, qa, 1);
      // instruction 1: record of the even lane, halves lo (even) / hi (odd)
      float* p1 = odd ? (float*)qo + 4 : q;
      red4(p1, odd ? s0 : v[0], odd ? s1 : v[1], odd ? s2 : v[2], odd ? s3 : v[3]);
      // instruction 2: record of the odd lane
      float* p2 = odd ? q + 4 : (float*)qo;
      red4(p2, odd ? v[4] : s0, odd ? v[5] : s1, odd ? v[6] : s2, odd ? v[7] : s3);
    }
  }
}
int main(int argc, char** argv) {
  // records in the working set: 17 M (544 MB, C4's cell workspace) by default
  const unsigned ncell = argc > 1 ? (unsigned)atoi(argv[1]) : 17u << 20;
  float* buf;
  cudaMalloc(&buf, 32ull * ncell);
  cudaMemset(buf, 0, 32ull * ncell);
  const int blocks = 148 * 8, threads = 256, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    k<<<blocks, threads>>>(buf, ncell, 10, mode);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(buf, ncell, iters, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flushes = (double)blocks * threads * iters;
    printf("ncell %u mode %d: %.3f ms, %.1f G record-flushes/s\n", ncell, mode, ms, flushes / ms / 1e6);
  }
  return 0;
}
