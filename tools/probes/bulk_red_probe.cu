// Micro-benchmark: cost of flushing 32-byte cell records (8 fp32 moments) into a
// record array, per mechanism (is the per-lane LSU cost of red.v4 avoidable?).
//   mode 0: each lane: two red.global.add.v4.f32 (the walk's flush), random cells
//   mode 1: same, lanes of a warp on consecutive cells (coalesced pattern)
//   mode 2: each lane: record -> its own shared slot (2 STS.128), then ONE
//           cp.reduce.async.bulk .add.f32 of 32 bytes (TMA engine), random cells
//   mode 3: mode 2 with lanes on consecutive cells
//   mode 4: warp-cooperative: the warp's 32 records (consecutive cells) staged in
//           shared, one lane issues one 1 KB bulk reduce (a bound for large ops)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void bulk_red(float* g, const void* s, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
               :: "l"(g), "r"((unsigned)__cvta_generic_to_shared(s)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kSlots = 4;   // ring of staging slots per lane
__global__ void k(float* buf, unsigned ncell, int iters, int mode) {
  __shared__ __align__(128) float4 stage[kSlots][256][2];
  const unsigned lane = threadIdx.x & 31;
  unsigned h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = 1e-6f * (j + 1);
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    const bool coal = mode == 1 || mode == 3 || mode == 4;
    unsigned hw = __shfl_sync(~0u, h, 0);
    unsigned cell = coal ? ((hw >> 5) + lane) % ncell : (h >> 3) % ncell;
    float* q = buf + 8ull * cell;
    if (mode <= 1) {
      red4(q, v[0], v[1], v[2], v[3]);
      red4(q + 4, v[4], v[5], v[6], v[7]);
    } else if (mode <= 3) {
      const int s = it % kSlots;
      bulk_wait_read<kSlots - 1>();   // the slot's previous op has read its source
      stage[s][threadIdx.x][0] = make_float4(v[0], v[1], v[2], v[3]);
      stage[s][threadIdx.x][1] = make_float4(v[4], v[5], v[6], v[7]);
      fence_async();
      bulk_red(q, &stage[s][threadIdx.x][0], 32);
      bulk_commit();
    } else {
      const int s = it % kSlots;
      if (lane == 0) bulk_wait_read<kSlots - 1>();
      __syncwarp();
      stage[s][threadIdx.x][0] = make_float4(v[0], v[1], v[2], v[3]);
      stage[s][threadIdx.x][1] = make_float4(v[4], v[5], v[6], v[7]);
      fence_async();
      __syncwarp();
      if (lane == 0 && (hw >> 5) % ncell + 32 <= ncell) {
        bulk_red(buf + 8ull * ((hw >> 5) % ncell), &stage[s][threadIdx.x & ~31][0], 1024);
        bulk_commit();
      }
    }
  }
  bulk_wait_read<0>();
}
int main(int argc, char** argv) {
  const unsigned ncell = argc > 1 ? (unsigned)atoi(argv[1]) : 2u << 20;   // 64 MB default
  float* buf;
  cudaMalloc(&buf, 32ull * ncell);
  cudaMemset(buf, 0, 32ull * ncell);
  const int blocks = 148 * 4, threads = 256, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 5; ++mode) {
    k<<<blocks, threads>>>(buf, ncell, 10, mode);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(buf, ncell, iters, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flushes = (double)blocks * threads * iters;
    printf("ncell %u (%u MB) mode %d: %.3f ms, %.1f G record-flushes/s %s\n", ncell, (unsigned)(32ull * ncell >> 20), mode, ms,
           flushes / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
