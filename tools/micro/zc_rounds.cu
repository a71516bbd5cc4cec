// Micro-benchmark: zero-copy point streaming with compute between rounds (the e2e kernel's
// pattern): 444 blocks x 256 threads, each warp reads its round's 96 bytes (3-byte points,
// 24 words) D rounds ahead of use and spins ~C ns per round.  Prints time and GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int D>
__global__ void rounds_kernel(const unsigned* __restrict__ p, int rounds_per_warp, long long spin, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned buf[D + 1];
  unsigned acc = 0;
  for (int d = 0; d < D; ++d) buf[d] = lane < 24 ? __ldg(p + ((long long)d * nwarps + warp) * 24 + lane) : 0;
  for (int r = 0; r < rounds_per_warp; ++r) {
    if (r + D < rounds_per_warp) buf[D] = lane < 24 ? __ldg(p + ((long long)(r + D) * nwarps + warp) * 24 + lane) : 0;
    acc += buf[0];
    long long t0 = clock64();
    while (clock64() - t0 < spin) acc = acc * 3 + 1;
    for (int d = 0; d < D; ++d) buf[d] = buf[d + 1];
  }
  if (acc == 0x12345u) *out = acc;
}
int main() {
  const int grid = 444, tpb = 256;
  const long long nwarps = grid * tpb / 32;
  const int rpw = 9;  // 2^20 points / (444 * 256) ~ 9.2 rounds
  const size_t bytes = (size_t)nwarps * rpw * 96;
  unsigned *h, *hm, *out;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hm, h, 0);
  cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (long long spin : {0LL, 5000LL, 11000LL}) {
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      cudaEventRecord(a); rounds_kernel<1><<<grid, tpb>>>(hm, rpw, spin, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("spin %lld depth 1: %.1f us %.1f GB/s\n", spin, ms * 1e3, bytes / ms / 1e6);
      cudaEventRecord(a); rounds_kernel<2><<<grid, tpb>>>(hm, rpw, spin, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("spin %lld depth 2: %.1f us %.1f GB/s\n", spin, ms * 1e3, bytes / ms / 1e6);
      cudaEventRecord(a); rounds_kernel<4><<<grid, tpb>>>(hm, rpw, spin, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); printf("spin %lld depth 4: %.1f us %.1f GB/s\n", spin, ms * 1e3, bytes / ms / 1e6);
    }
  }
  return 0;
}
