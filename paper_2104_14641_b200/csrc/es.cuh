// Evolution-strategies search on device (throughput mode).
//
// Included by engine.cu (same translation unit: the scoring kernels' task
// table, evaluators and point decoding are reused).  One generation of the
// reference's optimize loop (ls/es.py:130-204) is four launches with no host
// round trip, captured once into a CUDA graph and replayed `iterations` times:
//
//   es_gen_kernel     member i: Gaussian noise from Philox4x32-10 keyed by
//                     (seed, generation) with counter (i, pair), Box-Muller;
//                     theta + sigma*eps; ThetaEncoding.decode = clip(rint(.),
//                     0, n_d - 1) per axis (ls/es.py:57-62); the flat space
//                     point; the memo of distinct schedules (ls/es.py:139-160)
//                     as an open-addressing table keyed by the point; a new
//                     point is scored by the task's points kernel code; the
//                     sort key of F = -score (ls/es.py:176)
//   cub radix sort    (F bits, member index): stable ranks, _shape_fitness's
//                     argsort(argsort(., stable), stable) (ls/es.py:65-71)
//   es_partial_kernel fixed 1024-position chunks of sum_i w_i eps_i (noise
//                     regenerated, not stored), fixed-order reductions
//   es_update_kernel  theta += alpha / (population * sigma) * sum (ls/es.py:91-92),
//                     incumbent trace (ls/es.py:189-190), generation counter
//
// The noise stream is not numpy's PCG64 (the device cannot reproduce it), so
// trajectories differ from the reference's optimize; es.optimize keeps the
// reference's exact trajectory with host noise (parity mode).  Everything
// downstream of the noise follows the reference's arithmetic.
//
// Sharded over G ranks: rank r evaluates members [r P/G,
// (r+1) P/G) (their noise depends on the global member index only), the F keys
// are all-gathered in place (every rank then holds the whole population's keys
// and sorts them: global stable ranks, ls/es.py:65-71), rank r sums its share
// of the fixed 1024-position chunks, the chunk partials are all-gathered in
// place and every rank adds all of them in chunk order.  Chunk boundaries and
// the order of every float64 addition are independent of G, so theta, the
// trace and the evaluated set are bit-identical for G = 1, 2, 4, 8.  The memo
// is per rank; the distinct count is the size of the union of the ranks'
// evaluated lists and the trace the per-generation minimum over ranks (both
// computed by the caller after the run).

#include <cub/device/device_radix_sort.cuh>

constexpr int ES_CHUNK = 1024;  // sorted positions per partial sum (independent of the grid)
constexpr int ES_MAXDIM = LS_MAX_AXES;

struct EsDev {
  double theta[ES_MAXDIM];
  double alpha, sigma, coef;           // coef = alpha / (population * sigma)
  uint64_t seed;
  int32_t pop, iters, dim, rank_normalize;
  int32_t gen, pad;
  int32_t lo, hi;                      // this rank's members [lo, hi)
  int32_t c0, c1;                      // this rank's chunks [c0, c1) of sum_i w_i eps_i
  int32_t chunks, pad2;                // all chunks
  uint32_t n_ax[ES_MAXDIM];            // choices per axis
  unsigned long long best;             // order bits of the best score so far
  unsigned long long evaluations;      // distinct schedules scored
  unsigned long long err;              // first failure (atomicMin; ~0 none): (generation+1 | 0 start) << 40 | member << 8 | status
  unsigned long long* keys;            // memo: flat point + 1 (0 = empty)
  unsigned long long* vals;            // memo: order bits of the score (0 = being scored)
  unsigned long long cap_mask;
  unsigned long long* list_p;          // evaluated points in discovery order
  double* list_s;                      // their scores
  unsigned long long list_cap;
  unsigned long long full;             // memo probes exhausted (table full): reported as a failure
  unsigned long long* sort_in;         // per member: order bits of F = -score
  unsigned long long* sort_out;
  uint32_t* idx_in;
  uint32_t* idx_out;
  double* partial;                     // [chunks][dim]
  double* theta_hist;                  // [iters + 1][dim]
  double* trace;                       // [iters]
};

// ---- Philox4x32-10 (Salmon et al., SC'11) ---------------------------------------
__host__ __device__ inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
  }
}

// Standard normals eps[2q], eps[2q+1] of member i in generation g: one Philox
// block per pair, Box-Muller on two 53-bit uniforms (u1 in (0, 1], u2 in [0, 1)).
__device__ __forceinline__ void es_normal_pair(uint64_t seed, int g, uint32_t i, int q, double& z0, double& z1) {
  uint32_t c[4] = {i, (uint32_t)q, (uint32_t)g, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)c[1] << 32 | c[0]) >> 11, b = ((uint64_t)c[3] << 32 | c[2]) >> 11;
  const double u1 = (double)(a + 1) * 0x1.0p-53, u2 = (double)b * 0x1.0p-53;
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586 * u2;
  z0 = rad * cos(ang);
  z1 = rad * sin(ang);
}

__device__ __forceinline__ double es_eps(const EsDev& E, int g, uint32_t i, int d) {
  double z0, z1;
  es_normal_pair(E.seed, g, i, d >> 1, z0, z1);
  return (d & 1) ? z1 : z0;
}

// Score of space point x through the task's points kernel code (status != 0: failure).
template <int TM, int RM, int MODE>
__device__ __forceinline__ int score_point(const DTask& T, const int32_t* tab, Evaluator<TM, RM, MODE>& ev,
                                           uint64_t x, double* s) {
  double f[LS_NFEAT_GPU];
  if constexpr (MODE == 4 || MODE == 5) {
    return eval_space<TM, MODE == 5>(T, tab, x, ev.fc, f, s);
  } else {
    ls_record r;
    uint32_t kt[4];
    uint32_t pch = 0;
    int st = point_record<MODE == 3>(T, x, r, kt, pch);
    if (st == LS_OK) st = ev(T, r, kt, pch, f, s);
    return st;
  }
}

// Memoised score of point x (ls/es.py:139-160): the first thread to claim the
// key scores it and counts a distinct evaluation; others reuse the value (or
// rescore it themselves while it is being written: scores are pure).
template <int TM, int RM, int MODE>
__device__ int es_memo_score(const DTask& T, const int32_t* tab, Evaluator<TM, RM, MODE>& ev, EsDev& E, uint64_t x,
                             double* s) {
  const unsigned long long key = x + 1;
  unsigned long long h = (key * 0x9E3779B97F4A7C15ull) >> 17;
  for (unsigned long long probe = 0; probe <= E.cap_mask; ++probe, ++h) {
    h &= E.cap_mask;
    const unsigned long long k = atomicCAS(&E.keys[h], 0ull, key);
    if (k == 0ull) {  // claimed: a new distinct schedule
      const int st = score_point<TM, RM, MODE>(T, tab, ev, x, s);
      if (st) return st;
      const unsigned long long pos = atomicAdd(&E.evaluations, 1ull);
      if (pos < E.list_cap) {
        E.list_p[pos] = x;
        E.list_s[pos] = *s;
      }
      atomicMin(&E.best, order_bits(*s));
      atomicExch(&E.vals[h], order_bits(*s));
      return LS_OK;
    }
    if (k == key) {
      const unsigned long long v = __ldcg(&E.vals[h]);
      if (v) {
        *s = from_order_bits(v);
        return LS_OK;
      }
      return score_point<TM, RM, MODE>(T, tab, ev, x, s);
    }
  }
  atomicExch(&E.full, 1ull);  // cannot happen within the sizing of ls_es_create
  return LS_ST_OVERFLOW;
}

// One generation (start = true: the decode of theta alone, ls/es.py:183-186).
template <int TM, int RM, int MODE>
__global__ void __launch_bounds__(TPB, 2) es_gen_kernel(const DTask* __restrict__ gtask, EsDev* __restrict__ ges,
                                                       int start) {
  extern __shared__ __align__(16) unsigned char dyn[];
  DTask& T = *reinterpret_cast<DTask*>(dyn);
  stage_task(T, gtask);
  unsigned char* p = dyn + T.task_bytes;
  const int32_t* tab = stage_tab<MODE>(p, T);
  p += tab_smem_bytes(MODE, T);
  Evaluator<TM, RM, MODE> ev(T, p, tab);
  EsDev& E = *ges;
  const int g = E.gen;
  const int lo = start ? 0 : E.lo, hi = start ? 1 : E.hi;
  for (int i = lo + blockIdx.x * TPB + threadIdx.x; i < hi; i += gridDim.x * TPB) {
    uint64_t x = 0;
    for (int d = 0; d < E.dim; d += 2) {
      double z0 = 0.0, z1 = 0.0;
      if (!start) es_normal_pair(E.seed, g, (uint32_t)i, d >> 1, z0, z1);
      for (int q = d; q < d + 2 && q < E.dim; ++q) {
        const double pt = __dadd_rn(E.theta[q], __dmul_rn(E.sigma, q == d ? z0 : z1));
        const double m = (double)(E.n_ax[q] - 1);
        const double c = fmin(fmax(rint(pt), 0.0), m);  // np.clip(round(x), 0, n - 1)
        x = x * E.n_ax[q] + (uint64_t)c;
      }
    }
    double s = 0.0;
    const int st = es_memo_score<TM, RM, MODE>(T, tab, ev, E, x, &s);
    if (st) {  // generation field 0: the start point
      atomicMin(&E.err, ((unsigned long long)(start ? 0 : g + 1) << 40) | ((unsigned long long)i << 8) |
                            (unsigned long long)st);
      s = 0.0;
    }
    if (!start) {
      E.sort_in[i] = order_bits(-s);  // F = -score, maximised (ls/es.py:176); idx_in is the identity
    }
  }
}

// sum over fixed chunks of sorted positions of w_j * eps[member_j]; w_j = the
// centred rank j/(n-1) - 0.5 (rank_normalize) or F itself (ls/es.py:65-71, 90).
__global__ void __launch_bounds__(TPB) es_partial_kernel(EsDev* __restrict__ ges) {
  __shared__ double red[TPB];
  EsDev& E = *ges;
  const int n = E.pop, dim = E.dim, g = E.gen;
  const bool flat = E.rank_normalize && E.sort_out[0] == E.sort_out[n - 1];  // np.ptp(values) == 0
  const int chunk = E.c0 + blockIdx.x;
  const int j0 = chunk * ES_CHUNK;
  double acc[ES_MAXDIM];
  for (int d = 0; d < dim; ++d) acc[d] = 0.0;
  for (int j = j0 + threadIdx.x; j < min(n, j0 + ES_CHUNK); j += TPB) {
    double w;
    if (E.rank_normalize)
      w = flat ? 0.0 : __dadd_rn(__ddiv_rn((double)j, (double)(n - 1)), -0.5);
    else
      w = from_order_bits(E.sort_out[j]);
    const uint32_t i = E.idx_out[j];
    for (int d = 0; d < dim; d += 2) {
      double z0, z1;
      es_normal_pair(E.seed, g, i, d >> 1, z0, z1);
      acc[d] = __dadd_rn(acc[d], __dmul_rn(w, z0));
      if (d + 1 < dim) acc[d + 1] = __dadd_rn(acc[d + 1], __dmul_rn(w, z1));
    }
  }
  for (int d = 0; d < dim; ++d) {
    red[threadIdx.x] = acc[d];
    __syncthreads();
    for (int w = TPB / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) E.partial[(size_t)chunk * dim + d] = red[0];
    __syncthreads();
  }
}

__global__ void es_update_kernel(EsDev* __restrict__ ges) {
  EsDev& E = *ges;
  const int chunks = E.chunks;
  const int d = threadIdx.x;
  const int g = E.gen;
  if (d < E.dim) {
    double sum = 0.0;
    for (int b = 0; b < chunks; ++b) sum = __dadd_rn(sum, E.partial[(size_t)b * E.dim + d]);
    E.theta[d] = __dadd_rn(E.theta[d], __dmul_rn(E.coef, sum));
    E.theta_hist[(size_t)(g + 1) * E.dim + d] = E.theta[d];
  }
  __syncthreads();
  if (d == 0) {
    E.trace[g] = from_order_bits(E.best);
    E.gen = g + 1;
  }
}

// Diagnostic: the Gaussian noise of generation g, [pop][dim].
__global__ void es_noise_kernel(const EsDev* __restrict__ ges, int g, double* __restrict__ out) {
  const EsDev& E = *ges;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E.pop) return;
  for (int d = 0; d < E.dim; ++d) out[(size_t)i * E.dim + d] = es_eps(E, g, (uint32_t)i, d);
}

struct ls_es {
  ls_task* task;
  EsDev host;
  EsDev* dev;
  void* sort_tmp;
  size_t sort_tmp_bytes;
  int chunks, mode;
  int rank, world, cpr;  // shard: rank of world, chunks per rank (the partials' gather slice)
  cudaGraphExec_t graph;
  std::vector<void*> owned;
};

namespace {

using EsGenFn = void (*)(const DTask*, EsDev*, int);

EsGenFn es_gen_fn(const DTask& T, int mode) {
  if (mode == 4) {
    switch (T.n_tensors) {
      case 1: return es_gen_kernel<1, 4, 4>;
      case 2: return es_gen_kernel<2, 4, 4>;
      case 3: return es_gen_kernel<3, 4, 4>;
      default: return es_gen_kernel<4, 4, 4>;
    }
  }
  if (mode == 5) {
    switch (T.n_tensors) {
      case 1: return es_gen_kernel<1, 4, 5>;
      case 2: return es_gen_kernel<2, 4, 5>;
      case 3: return es_gen_kernel<3, 4, 5>;
      default: return es_gen_kernel<4, 4, 5>;
    }
  }
  if (mode == 6) return es_gen_kernel<4, 4, 6>;
  if (mode == 3) return es_gen_kernel<4, 4, 3>;
  if (mode == 2) return es_gen_kernel<4, 4, 2>;
  if (mode == 1) return es_gen_kernel<4, 4, 1>;
  return T.layout_rm == 4 ? es_gen_kernel<4, 4, 0> : es_gen_kernel<MAXT, MAXRANK, 0>;
}

int es_launch_gen(ls_es* es, int start, cudaStream_t s) {
  const ls_task* t = es->task;
  const EsGenFn fn = es_gen_fn(t->host, es->mode);
  const size_t sm = smem_score(t->host, es->mode);
  const int64_t n = start ? 1 : es->host.hi - es->host.lo;
  BPS_TRY(bps, fn, sm);
  fn<<<grid_for(t, n, bps), TPB, sm, s>>>(t->d_task, es->dev, start);
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

// after the F keys of the whole population are present: global stable ranks and this
// rank's chunk partials
int es_launch_rank(ls_es* es, cudaStream_t s) {
  size_t bytes = es->sort_tmp_bytes;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(es->sort_tmp, bytes, es->host.sort_in, es->host.sort_out, es->host.idx_in,
                                           es->host.idx_out, es->host.pop, 0, 64, s));
  if (es->host.c1 > es->host.c0) {
    es_partial_kernel<<<es->host.c1 - es->host.c0, TPB, 0, s>>>(es->dev);
    CUDA_TRY(cudaGetLastError());
  }
  return LS_E_OK;
}

int es_launch_update(ls_es* es, cudaStream_t s) {
  es_update_kernel<<<1, 32, 0, s>>>(es->dev);
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

int es_enqueue_generation(ls_es* es, cudaStream_t s) {
  if (int rc = es_launch_gen(es, 0, s)) return rc;
  if (int rc = es_launch_rank(es, s)) return rc;
  return es_launch_update(es, s);
}

}  // namespace

extern "C" {

int ls_es_create_shard(ls_task* t, const ls_es_params* p, const double* h_theta0, int32_t rank, int32_t world,
                       ls_es** out) {
  if (!t || !p || !out) return fail(LS_E_ARG, "null argument");
  *out = nullptr;
  if (t->host.sp_n < 1) return fail(LS_E_ARG, "no schedule space attached (ls_task_set_space)");
  if (!(p->alpha > 0) || !(p->sigma > 0)) return fail(LS_E_ARG, "alpha and sigma must be positive");
  if (p->population < 2 || p->iterations < 1) return fail(LS_E_ARG, "population >= 2 and iterations >= 1");
  if (world < 1 || rank < 0 || rank >= world) return fail(LS_E_ARG, "bad rank / world");
  if (p->population % world) return fail(LS_E_ARG, "population must be a multiple of the number of ranks");
  CUDA_TRY(cudaSetDevice(t->device));
  ls_es* es = new ls_es();
  es->task = t;
  es->graph = nullptr;
  es->sort_tmp = nullptr;
  es->rank = rank;
  es->world = world;
  EsDev& H = es->host;
  memset(&H, 0, sizeof(H));
  H.dim = t->host.sp_n;
  double space = 1.0;
  for (int a = 0; a < H.dim; ++a) {
    H.n_ax[a] = t->host.sp_ax[a].n;
    space *= H.n_ax[a];
    H.theta[a] = h_theta0 ? h_theta0[a] : (H.n_ax[a] - 1) / 2.0;  // ThetaEncoding.initial (ls/es.py:54-55)
  }
  if (space >= 1.8e19) {
    delete es;
    return fail(LS_E_UNSUPPORTED, "space has more than 2^64 points");
  }
  H.alpha = p->alpha;
  H.sigma = p->sigma;
  H.coef = p->alpha / ((double)p->population * p->sigma);
  H.seed = p->seed;
  H.pop = p->population;
  H.iters = p->iterations;
  H.rank_normalize = p->rank_normalize ? 1 : 0;
  H.best = ~0ull;
  H.err = ~0ull;
  const int per = p->population / world;
  H.lo = rank * per;
  H.hi = H.lo + per;
  es->chunks = (H.pop + ES_CHUNK - 1) / ES_CHUNK;
  es->cpr = (es->chunks + world - 1) / world;
  H.chunks = es->chunks;
  H.c0 = std::min(es->chunks, rank * es->cpr);
  H.c1 = std::min(es->chunks, (rank + 1) * es->cpr);
  // memo sized for this rank's distinct schedules at load <= 1/2; the probe is bounded
  const double distinct = std::min(space, (double)per * p->iterations + 1.0);
  constexpr double ES_MAX_DISTINCT = (double)(1ull << 28);
  if (distinct > ES_MAX_DISTINCT) {
    delete es;
    return fail(LS_E_UNSUPPORTED, "more than 2^28 distinct schedules per rank (population x iterations); "
                                  "shard the population over more ranks or run fewer iterations per call");
  }
  unsigned long long cap = 1024;
  while ((double)cap < 2.0 * distinct) cap <<= 1;
  H.cap_mask = cap - 1;
  H.list_cap = (unsigned long long)distinct;
  es->mode = mode_of(t, true);
  auto alloc = [&](void** ptr, size_t bytes) -> int {
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) return fail(LS_E_NOMEM, "ES buffer allocation");
    es->owned.push_back(*ptr);
    return LS_E_OK;
  };
  int rc = LS_E_OK;
  rc = rc ? rc : alloc((void**)&H.keys, sizeof(unsigned long long) * cap);
  rc = rc ? rc : alloc((void**)&H.vals, sizeof(unsigned long long) * cap);
  rc = rc ? rc : alloc((void**)&H.list_p, sizeof(unsigned long long) * H.list_cap);
  rc = rc ? rc : alloc((void**)&H.list_s, sizeof(double) * H.list_cap);
  rc = rc ? rc : alloc((void**)&H.sort_in, sizeof(unsigned long long) * H.pop);
  rc = rc ? rc : alloc((void**)&H.sort_out, sizeof(unsigned long long) * H.pop);
  rc = rc ? rc : alloc((void**)&H.idx_in, sizeof(uint32_t) * H.pop);
  rc = rc ? rc : alloc((void**)&H.idx_out, sizeof(uint32_t) * H.pop);
  rc = rc ? rc : alloc((void**)&H.partial, sizeof(double) * (size_t)es->cpr * world * H.dim);
  rc = rc ? rc : alloc((void**)&H.theta_hist, sizeof(double) * (H.iters + 1) * H.dim);
  rc = rc ? rc : alloc((void**)&H.trace, sizeof(double) * H.iters);
  rc = rc ? rc : alloc((void**)&es->dev, sizeof(EsDev));
  if (rc == LS_E_OK) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, H.sort_in, H.sort_out, H.idx_in, H.idx_out, H.pop, 0, 64);
    es->sort_tmp_bytes = bytes;
    rc = alloc(&es->sort_tmp, bytes);
  }
  if (rc == LS_E_OK) {  // member indices of the gathered keys: the identity (rank slices in rank order)
    std::vector<uint32_t> iota((size_t)H.pop);
    for (int i = 0; i < H.pop; ++i) iota[i] = (uint32_t)i;
    if (cudaMemcpy(H.idx_in, iota.data(), sizeof(uint32_t) * H.pop, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail(LS_E_CUDA, "ES index upload");
  }
  if (rc) {
    ls_es_destroy(es);
    return rc;
  }
  *out = es;
  return LS_E_OK;
}

int ls_es_create(ls_task* t, const ls_es_params* p, const double* h_theta0, ls_es** out) {
  return ls_es_create_shard(t, p, h_theta0, 0, 1, out);
}

int ls_es_begin(ls_es* es, void* stream) {
  if (!es) return fail(LS_E_ARG, "null argument");
  ls_task* t = es->task;
  CUDA_TRY(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  EsDev& H = es->host;
  // fresh state: memo, counters, theta0 and its history row
  CUDA_TRY(cudaMemsetAsync(H.keys, 0, sizeof(unsigned long long) * (H.cap_mask + 1), s));
  CUDA_TRY(cudaMemsetAsync(H.vals, 0, sizeof(unsigned long long) * (H.cap_mask + 1), s));
  CUDA_TRY(cudaMemcpyAsync(es->dev, &H, sizeof(EsDev), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(H.theta_hist, H.theta, sizeof(double) * H.dim, cudaMemcpyHostToDevice, s));
  return es_launch_gen(es, 1, s);  // the start point (ls/es.py:183-186), on every rank
}

int ls_es_step(ls_es* es, int32_t stage, void* stream) {
  if (!es || stage < 0 || stage > 2) return fail(LS_E_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(es->task->device));
  cudaStream_t s = (cudaStream_t)stream;
  return stage == 0 ? es_launch_gen(es, 0, s) : stage == 1 ? es_launch_rank(es, s) : es_launch_update(es, s);
}

int ls_es_shard_buffers(ls_es* es, void** d_keys, int64_t* keys_per_rank, void** d_partials,
                        int64_t* partials_per_rank) {
  if (!es) return fail(LS_E_ARG, "null argument");
  if (d_keys) *d_keys = es->host.sort_in;
  if (keys_per_rank) *keys_per_rank = es->host.hi - es->host.lo;
  if (d_partials) *d_partials = es->host.partial;
  if (partials_per_rank) *partials_per_rank = (int64_t)es->cpr * es->host.dim;
  return LS_E_OK;
}

int ls_es_run(ls_es* es, void* stream) {
  if (!es) return fail(LS_E_ARG, "null argument");
  if (es->world != 1) return fail(LS_E_ARG, "a sharded run is driven generation by generation (ls_es_step)");
  if (int rc = ls_es_begin(es, stream)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  EsDev& H = es->host;
  bool single = true;
  for (int a = 0; a < H.dim; ++a) single &= H.n_ax[a] == 1;
  if (single) return LS_E_OK;  // a 1-schedule space needs no generation (ls/es.py:187-188)
  if (!es->graph) {  // one generation, captured once, replayed per iteration
    cudaStream_t cs;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    const int rc = es_enqueue_generation(es, cs);
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(LS_E_CUDA, std::string("ES graph capture: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&es->graph, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      es->graph = nullptr;
      return fail(LS_E_CUDA, std::string("ES graph instantiate: ") + cudaGetErrorString(ie));
    }
  }
  for (int it = 0; it < H.iters; ++it) CUDA_TRY(cudaGraphLaunch(es->graph, s));
  return LS_E_OK;
}

int ls_es_result(ls_es* es, double* h_theta_hist, double* h_trace, int64_t* h_evaluations, int64_t* h_error,
                 double* h_best_score, void* stream) {
  if (!es) return fail(LS_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(es->task->device));
  cudaStream_t s = (cudaStream_t)stream;
  EsDev D;
  CUDA_TRY(cudaMemcpyAsync(&D, es->dev, sizeof(EsDev), cudaMemcpyDeviceToHost, s));
  const EsDev& H = es->host;
  if (h_theta_hist)
    CUDA_TRY(cudaMemcpyAsync(h_theta_hist, H.theta_hist, sizeof(double) * (H.iters + 1) * H.dim,
                             cudaMemcpyDeviceToHost, s));
  if (h_trace) CUDA_TRY(cudaMemcpyAsync(h_trace, H.trace, sizeof(double) * H.iters, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (h_evaluations) *h_evaluations = (int64_t)D.evaluations;
  if (h_error) *h_error = D.err == ~0ull ? 0 : (int64_t)D.err;
  if (h_best_score) *h_best_score = D.best == ~0ull ? 0.0 : [](unsigned long long o) {
    unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double x;
    memcpy(&x, &b, 8);
    return x;
  }(D.best);
  return LS_E_OK;
}

int ls_es_evaluated(ls_es* es, uint64_t* h_points, double* h_scores, int64_t cap, int64_t* h_count, void* stream) {
  if (!es || !h_count || cap < 0) return fail(LS_E_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(es->task->device));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long ev = 0;
  CUDA_TRY(cudaMemcpyAsync(&ev, &es->dev->evaluations, sizeof(ev), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t m = std::min<int64_t>({(int64_t)ev, (int64_t)es->host.list_cap, cap});
  if (m > 0 && h_points)
    CUDA_TRY(cudaMemcpyAsync(h_points, es->host.list_p, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost, s));
  if (m > 0 && h_scores)
    CUDA_TRY(cudaMemcpyAsync(h_scores, es->host.list_s, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *h_count = (int64_t)ev;
  return LS_E_OK;
}

int ls_es_noise(ls_es* es, int32_t generation, double* d_out, void* stream) {
  if (!es || !d_out || generation < 0) return fail(LS_E_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(es->task->device));
  es_noise_kernel<<<(es->host.pop + 255) / 256, 256, 0, (cudaStream_t)stream>>>(es->dev, generation, d_out);
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

int ls_es_destroy(ls_es* es) {
  if (!es) return LS_E_OK;
  cudaSetDevice(es->task->device);
  cudaDeviceSynchronize();
  if (es->graph) cudaGraphExecDestroy(es->graph);
  for (void* q : es->owned) cudaFree(q);
  delete es;
  return LS_E_OK;
}

}  // extern "C"
