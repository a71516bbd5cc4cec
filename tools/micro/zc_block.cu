// Micro-benchmark: zero-copy streaming of 3-byte points in block rounds (768 B per 256-thread
// round) with compute between rounds: (a) 48 threads LDG.128 (aligned lines) into registers,
// staged to smem; (b) one TMA bulk copy (cp.async.bulk) per round into smem, mbarrier completion.
// Depth = rounds in flight.  Prints time and GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
template <int D>
__global__ void tma_kernel(const unsigned char* __restrict__ p, int rounds, long long spin, unsigned* out) {
  __shared__ __align__(128) unsigned char buf[D][768];
  __shared__ __align__(8) uint64_t bar[D];
  if (threadIdx.x == 0) for (int d = 0; d < D; ++d) mbar_init(&bar[d], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  unsigned acc = 0;
  auto src = [&](int r) { return p + ((long long)r * gridDim.x + blockIdx.x) * 768; };
  if (threadIdx.x == 0) for (int d = 0; d < D && d < rounds; ++d) { mbar_expect_tx(&bar[d], 768); bulk_g2s(buf[d], src(d), 768, &bar[d]); }
  for (int r = 0; r < rounds; ++r) {
    const int b = r % D;
    mbar_wait(&bar[b], (r / D) & 1);
    const unsigned char* q = buf[b] + 3 * threadIdx.x;
    acc += q[0] | q[1] << 8 | q[2] << 16;
    __syncthreads();
    if (threadIdx.x == 0 && r + D < rounds) { mbar_expect_tx(&bar[b], 768); bulk_g2s(buf[b], src(r + D), 768, &bar[b]); }
    long long t0 = clock64();
    while (clock64() - t0 < spin) acc = acc * 3 + 1;
  }
  if (acc == 0x12345u) *out = acc;
}
template <int D>
__global__ void ldg_kernel(const unsigned char* __restrict__ p, int rounds, long long spin, unsigned* out) {
  __shared__ __align__(16) unsigned char buf[2][768];
  unsigned acc = 0;
  auto src = [&](int r) { return reinterpret_cast<const uint4*>(p + ((long long)r * gridDim.x + blockIdx.x) * 768); };
  uint4 v[D];
  for (int d = 0; d < D; ++d) if (threadIdx.x < 48 && d < rounds) v[d] = __ldg(src(d) + threadIdx.x);
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x < 48) reinterpret_cast<uint4*>(buf[r & 1])[threadIdx.x] = v[0];
    for (int d = 0; d + 1 < D; ++d) v[d] = v[d + 1];
    if (threadIdx.x < 48 && r + D < rounds) v[D - 1] = __ldg(src(r + D) + threadIdx.x);
    __syncthreads();
    const unsigned char* q = buf[r & 1] + 3 * threadIdx.x;
    acc += q[0] | q[1] << 8 | q[2] << 16;
    long long t0 = clock64();
    while (clock64() - t0 < spin) acc = acc * 3 + 1;
  }
  if (acc == 0x12345u) *out = acc;
}
int main() {
  const int grid = 444, tpb = 256, rounds = 9;
  const size_t bytes = (size_t)grid * rounds * 768;
  unsigned char *h, *hm; unsigned* out;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hm, h, 0);
  cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (long long spin : {0LL, 11000LL}) for (int rep = 0; rep < 2; ++rep) {
    float ms;
#define RUN(K, NAME) cudaEventRecord(a); K<<<grid, tpb>>>(hm, rounds, spin, out); cudaEventRecord(b); cudaEventSynchronize(b); \
    cudaEventElapsedTime(&ms, a, b); printf("spin %lld %s: %.1f us %.1f GB/s %s\n", spin, NAME, ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    RUN(tma_kernel<2>, "tma depth 2")
    RUN(tma_kernel<4>, "tma depth 4")
    RUN(ldg_kernel<1>, "ldg depth 1")
    RUN(ldg_kernel<2>, "ldg depth 2")
  }
  return 0;
}
