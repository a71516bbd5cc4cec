// Device part of the ES search (see es.cuh for the design notes): the device
// state, Philox noise, the memoised scoring step and the generation kernels.
#pragma once

constexpr int ES_CHUNK = 1024;  // members per partial sum (independent of the grid; 512 and 4096 measured slower)
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
  double* noise;                       // [hi - lo][dim rounded up to pairs]: this rank's members' noise kept
                                       // by es_gen for es_partial, or null (regenerated)
  uint32_t* rank_of;                   // [pop] member -> position in the stable sort (the last pass)
};

// griddepcontrol.wait: a no-op unless the kernel was launched as a programmatic dependent
// (launch_pdl, es.cuh); then it returns once the previous grid is complete and visible.
__device__ __forceinline__ void es_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
  double sn, cs;
  sincos(ang, &sn, &cs);  // one shared argument reduction
  z0 = rad * cs;
  z1 = rad * sn;
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
    return eval_space_mode<TM, MODE>(T, tab, x, ev.fc, f, s);
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
  stage_task(T, gtask);  // the task's tables are constant over the run: staged before the wait
  unsigned char* p = dyn + T.task_bytes;
  const int32_t* tab = stage_tab<MODE>(p, T);
  p += tab_smem_bytes(MODE, T);
  Evaluator<TM, RM, MODE> ev(T, p, tab);
  es_pdl_wait();
  EsDev& E = *ges;
  const int g = E.gen;
  const int lo = start ? 0 : E.lo, hi = start ? 1 : E.hi;
  for (int i = lo + blockIdx.x * TPB + threadIdx.x; i < hi; i += gridDim.x * TPB) {
    uint64_t x = 0;
    for (int d = 0; d < E.dim; d += 2) {
      double z0 = 0.0, z1 = 0.0;
      if (!start) {
        es_normal_pair(E.seed, g, (uint32_t)i, d >> 1, z0, z1);
        if (E.noise) reinterpret_cast<double2*>(E.noise)[(size_t)(i - lo) * ((E.dim + 1) >> 1) + (d >> 1)] = make_double2(z0, z1);
      }
      for (int q = d; q < d + 2 && q < E.dim; ++q) {
        const double pt = __dadd_rn(E.theta[q], __dmul_rn(E.sigma, q == d ? z0 : z1));
        // np.clip(round(x), 0, n - 1): round-half-even conversion, then an integer clamp (NaN
        // converts to INT64_MIN and clamps to 0, +-inf saturate: the same as fmin/fmax on rint)
        const long long r = __double2ll_rn(pt);
        const long long c = r < 0 ? 0 : (r > (long long)E.n_ax[q] - 1 ? (long long)E.n_ax[q] - 1 : r);
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

#ifdef LS_MAIN_TU
// ---- stable LSD radix sort of (F order bits, member) pairs: the ranks of _shape_fitness
// (argsort(argsort(F, stable), stable), ls/es.py:65-71).  Single-pass-per-digit ("onesweep")
// form, 8-bit digits:
//   rs_upsweep_kernel  the global counts of all eight digits in one read (order-independent),
//                      AND / OR of the keys;
//   rs_plan_kernel     the digits some keys differ in (the others are skipped), their global
//                      digit bases, the in -> {tmp, out} chain so the last pass writes `out`;
//   rs_pass_kernel     per active digit: tiles of RS_TILE keys taken in launch order (ticket),
//                      stable in-tile ranks (each warp ranks its contiguous run of the tile
//                      by __match_any_sync with warp-private digit counters, then one
//                      exclusive scan over the warps per digit), the tile's exclusive prefix per
//                      digit by decoupled look-back over its predecessors' published counts
//                      (RS_WIN words per round trip), scatter.  A predecessor tile always
//                      belongs to a block already running, so the look-back never waits on an
//                      unscheduled block.
// Every launch is fixed (inactive passes exit at once): a generation stays one CUDA graph.
#ifndef LS_RS_TILE
#define LS_RS_TILE 8192
#endif
#ifndef LS_RS_WIN
#define LS_RS_WIN 8
#endif
constexpr int RS_TILE = LS_RS_TILE;    // keys per tile
constexpr int RS_WIN = LS_RS_WIN;      // look-back window: predecessor words read per round trip
#ifndef LS_RS_TPB
#define LS_RS_TPB 512
#endif
constexpr int RS_TPB = LS_RS_TPB;      // pass-kernel threads
constexpr int RS_SUB = RS_TILE / RS_TPB;  // keys per thread
constexpr uint32_t RS_AGG = 1u << 30, RS_INC = 2u << 30, RS_MASK = (1u << 30) - 1u;
// Per-sort control words, one allocation: everything before `epoch` is zeroed by ONE memset
// per sort; the look-back status words carry the sort's epoch in their high half, so the
// status array is never cleared (a word from an earlier sort reads as "not yet published").
struct RsCtl {
  unsigned long long nand, bor;  // OR of ~key (= ~AND of the keys), OR of the keys
  uint32_t ticket[8];            // tile tickets per pass
  uint32_t count[8 * 256];       // global digit counts, then (plan) digit bases
  uint32_t epoch, pad[3];        // sort counter (plan kernel), never cleared
};
constexpr size_t RS_CTL_RESET = offsetof(RsCtl, epoch);
struct RsBufs {
  unsigned long long* key[3];  // in, out, tmp
  uint32_t* idx[3];
  RsCtl* ctl;
  unsigned long long* status;  // [8][nblk][256] look-back words (epoch << 32 | flag << 30 | count)
  int32_t* plan;               // [8][4]: active (2: the last active pass), shift, src, dst
  uint32_t* rank;              // [n] member -> sorted position, written by the last pass
  int32_t n, nblk;
};

__global__ void __launch_bounds__(TPB) rs_upsweep_kernel(RsBufs R) {
  __shared__ uint32_t h[8][256];
  for (int c = threadIdx.x; c < 8 * 256; c += TPB) (&h[0][0])[c] = 0;
  __syncthreads();
  unsigned long long a = ~0ull, o = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < R.n; i += (int64_t)gridDim.x * TPB) {
    const unsigned long long k = R.key[0][i];
    a &= k;
    o |= k;
#pragma unroll
    for (int d = 0; d < 8; ++d) atomicAdd(&h[d][(k >> (8 * d)) & 0xFFu], 1u);
  }
  for (int off = 16; off > 0; off >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, off);
    o |= __shfl_xor_sync(0xffffffffu, o, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&R.ctl->nand, ~a);
    atomicOr(&R.ctl->bor, o);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 8 * 256; c += TPB)
    if ((&h[0][0])[c]) atomicAdd(&R.ctl->count[c], (&h[0][0])[c]);
}

__global__ void __launch_bounds__(256) rs_plan_kernel(RsBufs R) {
  es_pdl_wait();
  const int t = threadIdx.x;
  if (t == 0) {
    const unsigned long long x = ~R.ctl->nand ^ R.ctl->bor;  // AND ^ OR: the bits that vary
    int act[8], m = 0;
    for (int d = 0; d < 8; ++d) m += act[d] = ((x >> (8 * d)) & 0xFFull) != 0;
    if (!m) act[0] = 1, m = 1;  // every key equal: one stable copy in -> out
    int left = m, src = 0;
    for (int d = 0; d < 8; ++d) {
      int32_t* p = R.plan + 4 * d;
      p[0] = act[d];
      p[1] = 8 * d;
      if (!act[d]) continue;
      const int dst = (--left) % 2 == 0 ? 1 : 2;  // the last active pass writes `out`
      p[0] = left == 0 ? 2 : 1;                     // 2: the last pass also writes the ranks
      p[2] = src;
      p[3] = dst;
      src = dst;
    }
    R.ctl->epoch += 1u;
  }
  // digit bases: warp d scans digit d's 256 global counts (8 per lane)
  const int d = t >> 5, lane = t & 31;
  uint4* row = reinterpret_cast<uint4*>(R.ctl->count + d * 256 + lane * 8);
  uint4 c0 = row[0], c1 = row[1];
  const uint32_t v[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  uint32_t tot = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) tot += v[q];
  uint32_t inc = tot;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += u;
  }
  uint32_t e[8], run = inc - tot;
#pragma unroll
  for (int q = 0; q < 8; ++q) e[q] = run, run += v[q];
  row[0] = make_uint4(e[0], e[1], e[2], e[3]);
  row[1] = make_uint4(e[4], e[5], e[6], e[7]);
}

__global__ void __launch_bounds__(RS_TPB) rs_pass_kernel(RsBufs R, int d) {
  es_pdl_wait();
  const int32_t* p = R.plan + 4 * d;
  if (!p[0]) return;
  const bool last = p[0] == 2;
  __shared__ uint32_t lcount[256];       // the tile's keys per digit
  __shared__ uint32_t wcnt[RS_TPB / 32][256];  // per warp: running digit counts, then the warp's digit offsets
  __shared__ uint32_t gbase[256];        // global position of the tile's first key of each digit
  __shared__ int s_tile;
  const int sh = p[1];
  const int src = p[2], dst = p[3];  // selects, not a dynamically indexed parameter array (no stack copy)
  const unsigned long long* ks = src == 0 ? R.key[0] : src == 1 ? R.key[1] : R.key[2];
  const uint32_t* is = src == 0 ? R.idx[0] : src == 1 ? R.idx[1] : R.idx[2];
  unsigned long long* kd = dst == 1 ? R.key[1] : R.key[2];
  uint32_t* id = dst == 1 ? R.idx[1] : R.idx[2];
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&R.ctl->ticket[d], 1u);
  for (int c = threadIdx.x; c < (RS_TPB / 32) * 256; c += RS_TPB) (&wcnt[0][0])[c] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // warp w owns the tile's positions [w * 32 * RS_SUB, (w + 1) * 32 * RS_SUB): key q of a lane is
  // position w * 32 * RS_SUB + 32 q + lane (coalesced loads; tile order = warp, then q, then lane)
  const int64_t t0 = (int64_t)tile * RS_TILE + (int64_t)w * 32 * RS_SUB + lane;
  unsigned long long key[RS_SUB];
  uint32_t val[RS_SUB], pos[RS_SUB];  // pos: rank among the tile's keys of the same digit
#pragma unroll
  for (int q = 0; q < RS_SUB; ++q) {  // every load of the tile in flight before the ranking
    const int64_t i = t0 + 32 * q;
    key[q] = 0;
    val[q] = 0;
    if (i < R.n) {
      key[q] = ks[i];
      val[q] = is[i];
    }
  }
  // warp-local stable ranks: no block barrier until the warps' digit counts are complete
  uint32_t* wc = wcnt[w];
#pragma unroll
  for (int q = 0; q < RS_SUB; ++q) {
    const bool has = t0 + 32 * q < R.n;
    const uint32_t dig = has ? (uint32_t)(key[q] >> sh) & 0xFFu : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (has) pos[q] = wc[dig] + rank;
    __syncwarp();
    if (has && rank == 0) wc[dig] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < 256) {  // per digit: exclusive scan over the warps, the tile's count
    uint32_t run = 0;
#pragma unroll
    for (int u = 0; u < RS_TPB / 32; ++u) {
      const uint32_t c = wcnt[u][threadIdx.x];
      wcnt[u][threadIdx.x] = run;
      run += c;
    }
    lcount[threadIdx.x] = run;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RS_SUB; ++q)
    if (t0 + 32 * q < R.n) pos[q] += wc[(uint32_t)(key[q] >> sh) & 0xFFu];
  // decoupled look-back: thread t owns digit t and reads RS_WIN predecessor words per round trip
  if (threadIdx.x < 256) {
    const int t = threadIdx.x;
    unsigned long long* st = R.status + (size_t)d * R.nblk * 256;
    const unsigned long long ep = (unsigned long long)R.ctl->epoch << 32;
    const uint32_t mine = lcount[t];
    volatile unsigned long long* me = st + (size_t)tile * 256 + t;
    if (tile == 0) {
      *me = ep | RS_INC | mine;
      gbase[t] = R.ctl->count[d * 256 + t];
    } else {
      *me = ep | RS_AGG | mine;
      uint32_t excl = 0;
      int pt = tile - 1;  // tile 0 always publishes an inclusive prefix: the walk ends there at the latest
      for (;;) {
        unsigned long long v[RS_WIN];
#pragma unroll
        for (int q = 0; q < RS_WIN; ++q)
          v[q] = pt - q >= 0 ? *(const volatile unsigned long long*)(st + (size_t)(pt - q) * 256 + t) : 0ull;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int q = 0; q < RS_WIN; ++q) {
          if (done || used < q) continue;  // stopped at an inclusive prefix or an unpublished word
          if ((v[q] & ~(unsigned long long)RS_MASK) < (ep | RS_AGG)) continue;
          excl += (uint32_t)v[q] & RS_MASK;
          used = q + 1;
          done = ((uint32_t)v[q] >> 30) == 2u;
        }
        if (done) break;
        pt -= used;
        if (used < RS_WIN) __nanosleep(32);
      }
      __threadfence();
      *me = ep | RS_INC | (excl + mine);
      gbase[t] = R.ctl->count[d * 256 + t] + excl;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RS_SUB; ++q) {
    if (t0 + 32 * q >= R.n) continue;
    const uint32_t dig = (uint32_t)(key[q] >> sh) & 0xFFu;
    const uint32_t o = gbase[dig] + pos[q];
    kd[o] = key[q];
    id[o] = val[q];
    if (last) R.rank[val[q]] = o;
  }
}

// sum over fixed chunks of members of w_i * eps_i; w_i = the member's centred rank
// rank_i/(n-1) - 0.5 (rank_normalize; rank_i from the sort's last pass) or F_i itself
// (ls/es.py:65-71, 90).  Members in index order: the kept noise rows are read sequentially.
__global__ void __launch_bounds__(TPB) es_partial_kernel(EsDev* __restrict__ ges) {
  es_pdl_wait();
  __shared__ double wred[TPB / 32][ES_MAXDIM];
  EsDev& E = *ges;
  const int n = E.pop, dim = E.dim, g = E.gen;
  const bool flat = E.rank_normalize && E.sort_out[0] == E.sort_out[n - 1];  // np.ptp(values) == 0
  const int chunk = E.c0 + blockIdx.x;
  const int i0 = chunk * ES_CHUNK;
  const int pairs = (dim + 1) >> 1;
  double acc[ES_MAXDIM];  // unrolled over ES_MAXDIM with dim guards: registers, not a stack array
#pragma unroll
  for (int d = 0; d < ES_MAXDIM; ++d) acc[d] = 0.0;
  for (int i = i0 + threadIdx.x; i < min(n, i0 + ES_CHUNK); i += TPB) {  // members in index order
    double w;
    if (E.rank_normalize)  // the member's centred rank: its position in the stable sort
      w = flat ? 0.0 : __dadd_rn(__ddiv_rn((double)E.rank_of[i], (double)(n - 1)), -0.5);
    else
      w = from_order_bits(E.sort_in[i]);  // F itself, in member order
    const double2* kept = E.noise && i >= E.lo && i < E.hi
                              ? reinterpret_cast<const double2*>(E.noise) + (size_t)(i - E.lo) * pairs
                              : nullptr;
#pragma unroll
    for (int d = 0; d < ES_MAXDIM; d += 2) {
      if (d >= dim) break;
      double z0, z1;
      if (kept) {
        const double2 z = kept[d >> 1];
        z0 = z.x;
        z1 = z.y;
      } else {
        es_normal_pair(E.seed, g, (uint32_t)i, d >> 1, z0, z1);
      }
      acc[d] = __dadd_rn(acc[d], __dmul_rn(w, z0));
      if (d + 1 < dim) acc[d + 1] = __dadd_rn(acc[d + 1], __dmul_rn(w, z1));
    }
  }
  // fixed-shape reduction: butterfly within each warp, then the warps in order
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < ES_MAXDIM; ++d) {
    if (d >= dim) break;
    double v = acc[d];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wred[wp][d] = v;
  }
  __syncthreads();
  if (threadIdx.x < dim) {
    double v = wred[0][threadIdx.x];
#pragma unroll
    for (int u = 1; u < TPB / 32; ++u) v = __dadd_rn(v, wred[u][threadIdx.x]);
    E.partial[(size_t)chunk * dim + threadIdx.x] = v;
  }
}

// One block: the chunk partials summed in a fixed-shape tree (thread t adds chunks t, t + TPB,
// ... in order, a butterfly in each warp, then the warps in order) -- the same shape for every
// rank count G, so theta stays bit-identical across G; every row load of a thread in flight.
constexpr int ES_UPD_TPB = 256;
__global__ void __launch_bounds__(ES_UPD_TPB) es_update_kernel(EsDev* __restrict__ ges) {
  es_pdl_wait();
  __shared__ double wred[ES_UPD_TPB / 32][ES_MAXDIM];
  EsDev& E = *ges;
  const int chunks = E.chunks, dim = E.dim;
  const int g = E.gen;
  const double* __restrict__ part = E.partial;
  double acc[ES_MAXDIM];
#pragma unroll
  for (int d = 0; d < ES_MAXDIM; ++d) acc[d] = 0.0;
  for (int b = threadIdx.x; b < chunks; b += ES_UPD_TPB) {
    const double* row = part + (size_t)b * dim;
#pragma unroll
    for (int d = 0; d < ES_MAXDIM; ++d)
      if (d < dim) acc[d] = __dadd_rn(acc[d], row[d]);
  }
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < ES_MAXDIM; ++d) {
    if (d >= dim) break;
    double v = acc[d];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wred[wp][d] = v;
  }
  __syncthreads();
  const int d = threadIdx.x;
  if (d < dim) {
    double sum = wred[0][d];
#pragma unroll
    for (int u = 1; u < ES_UPD_TPB / 32; ++u) sum = __dadd_rn(sum, wred[u][d]);
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
#endif  // LS_MAIN_TU
