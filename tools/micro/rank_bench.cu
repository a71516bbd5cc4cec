// Micro-benchmark: one block ranks c distinct 16-byte keys held in shared memory
// (the last block's final step of the bound merge).  Prints cycles per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
struct Key { unsigned long long s; long long i; };
__device__ __forceinline__ bool kless(const Key& a, const Key& b) { return a.s < b.s || (a.s == b.s && a.i < b.i); }
__global__ void rank_kernel(const Key* in, int c, int k, int variant, double* out_s, long long* out_i, long long* cyc) {
  extern __shared__ Key B[];
  for (int j = threadIdx.x; j < c; j += blockDim.x) B[j] = in[j];
  __syncthreads();
  long long t0 = clock64();
  if (variant == 0) {  // warp per key, lanes split comparisons
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int q = threadIdx.x >> 5; q < c; q += nw) {
      const Key x = B[q];
      int r = 0;
      for (int j = lane; j < c; j += 32) r += kless(B[j], x) ? 1 : 0;
      r = __reduce_add_sync(0xffffffffu, r);
      if (lane == 0 && r < k) { out_s[r] = (double)x.s; out_i[r] = x.i; }
    }
  } else if (variant == 1) {  // thread per key
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
      const Key x = B[q];
      int r = 0;
      for (int j = 0; j < c; ++j) r += kless(B[j], x) ? 1 : 0;
      if (r < k) { out_s[r] = (double)x.s; out_i[r] = x.i; }
    }
  } else if (variant == 3) {  // bitonic sort of the next power of two, +inf padded
    int size0 = 2;
    while (size0 < c) size0 <<= 1;
    for (int i = c + threadIdx.x; i < size0; i += blockDim.x) { B[i].s = ~0ull; B[i].i = 0x7fffffffffffffffll; }
    __syncthreads();
    for (int size = 2; size <= size0; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < size0 / 2; t += blockDim.x) {
          const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const Key a = B[lo], b = B[hi];
          if (kless(b, a) == up) { B[lo] = b; B[hi] = a; }
        }
        __syncthreads();
      }
    for (int j = threadIdx.x; j < k && j < c; j += blockDim.x) { out_s[j] = (double)B[j].s; out_i[j] = B[j].i; }
  } else if (variant == 4) {  // warp per key, lanes split, branch-free
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int q = threadIdx.x >> 5; q < c; q += nw) {
      const Key x = B[q];
      int r = 0;
      for (int j = lane; j < c; j += 32) { const Key y = B[j]; r += (int)((y.s < x.s) | ((y.s == x.s) & (y.i < x.i))); }
      r = __reduce_add_sync(0xffffffffu, r);
      if (lane == 0 && r < k) { out_s[r] = (double)x.s; out_i[r] = x.i; }
    }
  } else {  // thread per key, branch-free compare
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
      const Key x = B[q];
      int r = 0;
#pragma unroll 8
      for (int j = 0; j < c; ++j) {
        const Key y = B[j];
        r += (int)((y.s < x.s) | ((y.s == x.s) & (y.i < x.i)));
      }
      if (r < k) { out_s[r] = (double)x.s; out_i[r] = x.i; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *cyc = clock64() - t0;
}
int main() {
  const int c = 306, k = 64;
  Key h[1024];
  for (int j = 0; j < c; ++j) { h[j].s = (unsigned long long)((j * 2654435761u) % 100003) << 20; h[j].i = j; }
  Key* d; double* os; long long *oi, *cyc;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&os, 8 * k); cudaMalloc(&oi, 8 * k); cudaMalloc(&cyc, 8);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int v = 0; v < 5; ++v) for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    rank_kernel<<<1, 256, 16 * 1024>>>(d, c, k, v, os, oi, cyc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long hc; cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %lld cycles (%.2f us at 1.965 GHz), kernel %.1f us\n", v, hc, hc / 1965.0, ms * 1e3);
  }
  return 0;
}
