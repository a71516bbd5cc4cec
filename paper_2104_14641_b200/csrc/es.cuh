// Evolution-strategies search on device (throughput mode).
//
// Included by engine.cu (same translation unit: the scoring kernels' task
// table, evaluators and point decoding are reused).  One generation of the
// reference's optimize loop (ls/es.py:130-204) is one memset and 13 launches with no host
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
//   rs_* kernels      stable onesweep radix sort of (F bits, member index): stable ranks,
//                     _shape_fitness's argsort(argsort(., stable), stable) (ls/es.py:65-71)
//   es_partial_kernel fixed 1024-member chunks of sum_i w_i eps_i in member order (w_i from
//                     the member's sorted position, written by the sort's last pass; noise
//                     kept by es_gen for this rank's members), fixed-shape reductions
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
// of the fixed 1024-member chunks, the chunk partials are all-gathered in
// place and every rank adds all of them in one fixed tree (es_update_kernel).  Chunk
// boundaries and the order of every float64 addition are independent of G, so theta, the
// trace and the evaluated set are bit-identical for G = 1, 2, 4, 8.  The memo
// is per rank; the distinct count is the size of the union of the ranks'
// evaluated lists and the trace the per-generation minimum over ranks (both
// computed by the caller after the run).

// EsDev, the Philox noise, the rank sort and the kernels: es_dev.cuh (included by every TU)

struct ls_es {
  ls_task* task;
  EsDev host;
  EsDev* dev;
  RsBufs rs;  // the rank sort's buffers (es_dev.cuh)
  int chunks, mode;
  int rank, world, cpr;  // shard: rank of world, chunks per rank (the partials' gather slice)
  cudaGraphExec_t graph;
  std::vector<void*> owned;
};

namespace {

EsGenFn es_gen_fn(const DTask& T, int mode) { return k_es_gen_fn(T, mode); }

#ifndef LS_ES_PDL
#define LS_ES_PDL 1
#endif
// Programmatic dependent launch: the kernel's blocks are scheduled behind the previous kernel's
// tail instead of after a full kernel boundary; every ES kernel starts with griddepcontrol.wait
// (es_pdl_wait), so nothing upstream is read before the previous grid is complete and visible.
template <typename... P, typename... A>
int launch_pdl(void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, A&&... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = LS_ES_PDL;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k, std::forward<A>(a)...));
  return LS_E_OK;
}

int es_launch_gen(ls_es* es, int start, cudaStream_t s) {
  const ls_task* t = es->task;
  const EsGenFn fn = es_gen_fn(t->host, es->mode);
  const size_t sm = smem_score(t->host, es->mode);
  const int64_t n = start ? 1 : es->host.hi - es->host.lo;
  BPS_TRY(bps, fn, sm);
  return launch_pdl(fn, (unsigned)grid_for(t, n, bps), TPB, sm, s, (const DTask*)t->d_task, es->dev, start);
}

// after the F keys of the whole population are present: global stable ranks and this
// rank's chunk partials
int es_launch_rank(ls_es* es, cudaStream_t s) {
  const RsBufs& R = es->rs;
  CUDA_TRY(cudaMemsetAsync(R.ctl, 0, RS_CTL_RESET, s));  // status words are epoch-tagged: never cleared
  rs_upsweep_kernel<<<std::min(R.nblk, 2 * es->task->num_sms), TPB, 0, s>>>(R);  // behind a memset
  CUDA_TRY(cudaGetLastError());
  if (int rc = launch_pdl(rs_plan_kernel, 1, 256, 0, s, R)) return rc;
  for (int d = 0; d < 8; ++d)
    if (int rc = launch_pdl(rs_pass_kernel, (unsigned)R.nblk, RS_TPB, 0, s, R, d)) return rc;
  if (es->host.c1 > es->host.c0)
    if (int rc = launch_pdl(es_partial_kernel, (unsigned)(es->host.c1 - es->host.c0), TPB, 0, s, es->dev)) return rc;
  return LS_E_OK;
}

int es_launch_update(ls_es* es, cudaStream_t s) {
  return launch_pdl(es_update_kernel, 1, ES_UPD_TPB, 0, s, es->dev);
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
  memset(&es->rs, 0, sizeof(es->rs));
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
  {  // es_gen keeps this rank's members' noise for es_partial (a partial over other ranks'
     // members regenerates theirs: the values are the same function either way)
    const size_t nb = sizeof(double) * 2 * (size_t)((H.dim + 1) / 2) * (size_t)(H.hi - H.lo);
    H.noise = nullptr;
    if (nb <= ((size_t)1 << 31)) rc = rc ? rc : alloc((void**)&H.noise, nb);
  }
  rc = rc ? rc : alloc((void**)&H.rank_of, sizeof(uint32_t) * H.pop);
  rc = rc ? rc : alloc((void**)&es->dev, sizeof(EsDev));
  if (rc == LS_E_OK) {  // the rank sort: ping-pong buffers, tile histograms, plan, AND / OR
    RsBufs& R = es->rs;
    R.n = H.pop;
    R.nblk = (H.pop + RS_TILE - 1) / RS_TILE;
    R.key[0] = H.sort_in;
    R.key[1] = H.sort_out;
    R.idx[0] = H.idx_in;
    R.idx[1] = H.idx_out;
    R.rank = H.rank_of;
    rc = rc ? rc : alloc((void**)&R.key[2], sizeof(unsigned long long) * H.pop);
    rc = rc ? rc : alloc((void**)&R.idx[2], sizeof(uint32_t) * H.pop);
    const size_t st_bytes = sizeof(unsigned long long) * 8 * 256 * (size_t)R.nblk;
    rc = rc ? rc : alloc((void**)&R.ctl, sizeof(RsCtl));
    rc = rc ? rc : alloc((void**)&R.status, st_bytes);
    rc = rc ? rc : alloc((void**)&R.plan, sizeof(int32_t) * 32);
    if (rc == LS_E_OK && (cudaMemset(R.ctl, 0, sizeof(RsCtl)) != cudaSuccess || cudaMemset(R.status, 0, st_bytes) != cudaSuccess))
      rc = fail(LS_E_CUDA, "ES sort buffer initialisation");
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
  LS_NVTX("ls_es_begin");
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
  LS_NVTX("ls_es_step");
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
  LS_NVTX("ls_es_run");
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

int ls_es_sort_state(ls_es* es, uint64_t* d_keys_in, uint64_t* d_keys_out, uint32_t* d_members, uint32_t* d_ranks,
                     void* stream) {
  if (!es || !d_keys_in || !d_keys_out || !d_members) return fail(LS_E_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(es->task->device));
  const cudaStream_t s = (cudaStream_t)stream;
  const size_t n = (size_t)es->host.pop;
  CUDA_TRY(cudaMemcpyAsync(d_keys_in, es->host.sort_in, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_keys_out, es->host.sort_out, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_members, es->host.idx_out, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  if (d_ranks)
    CUDA_TRY(cudaMemcpyAsync(d_ranks, es->host.rank_of, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
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
