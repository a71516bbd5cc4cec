// Micro-benchmark: host->device bandwidth of 4 MiB of points, DMA copy vs zero-copy kernel
// reads of mapped pinned memory at 4 / 16 bytes per thread (the e2e path's transfer).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void sum4(const unsigned* __restrict__ p, size_t n, unsigned* out) {
  unsigned s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += p[i];
  if (s == 0x12345678u) *out = s;
}
__global__ void sum16(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i]; s += v.x + v.y + v.z + v.w;
  }
  if (s == 0x12345678u) *out = s;
}
int main() {
  const size_t bytes = 4u << 20;
  unsigned *h, *d, *out, *hm;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes); cudaMalloc(&out, 4);
  cudaHostGetDevicePointer(&hm, h, 0);
  for (size_t i = 0; i < bytes / 4; ++i) h[i] = (unsigned)i;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    for (size_t sz : {bytes, bytes * 3 / 4, bytes * 4}) {
      if (sz > bytes) continue;
      cudaEventRecord(a); cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("DMA %zu B: %.1f us %.1f GB/s\n", sz, ms * 1e3, sz / ms / 1e6);
    }
    for (int grid : {148, 444, 1184}) {
      cudaEventRecord(a); sum4<<<grid, 256>>>(hm, bytes / 4, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("zero-copy 4B/thread grid %d: %.1f us %.1f GB/s\n", grid, ms * 1e3, bytes / ms / 1e6);
      cudaEventRecord(a); sum16<<<grid, 256>>>((const uint4*)hm, bytes / 16, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("zero-copy 16B/thread grid %d: %.1f us %.1f GB/s\n", grid, ms * 1e3, bytes / ms / 1e6);
    }
  }
  return 0;
}
