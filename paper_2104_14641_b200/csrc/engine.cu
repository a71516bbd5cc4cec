// loopscout_b200 engine: batched static cost evaluation of candidate loop-nest
// schedules on sm_100a, behind the C-ABI of include/loopscout_b200.h.
//
// One thread evaluates one candidate end to end (record decode -> transform
// application -> footprint/movement model -> instruction counts -> block
// cycles -> linear score); a block-level streaming top-k is fused into the
// same pass.  The reference pipeline this replaces, per candidate
// (ls/ = /root/reference/pkg/src/loopscout):
//   apply_schedule ls/ir.py:454-474, emit_mock_asm ls/ir.py:557-659,
//   parse_asm/loop_map/count_simd ls/asm.py:110-337, CacheModel ls/cache.py:133-259,
//   schedule_block/ilp_feature ls/ilp.py:158-271, PTX features ls/ptx.py:90-327,
//   extract_features/score ls/cost.py:132-161, rank ls/cost.py:164-168.
// The text pipeline is replaced by its structure: for a perfect loop chain the
// emitted blocks, their trip weights and their schedules are closed-form in
// the transformed chain (DESIGN.md §3 derives each term).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/loopscout_b200.h"

namespace lsb {
void fixed_block_cycles(const ls_task_desc& d, int64_t* c_init, int64_t* c_latch, int64_t* c_ret);
int64_t group_block_cycles(const ls_task_desc& d, const std::vector<int>& load_t, const std::vector<int>& store_t,
                           bool with_latch);
int64_t body_block_cycles(const ls_task_desc& d, const std::vector<int>& load_t,
                          const std::vector<int>& store_t, int64_t U, bool with_latch);
}  // namespace lsb

// ---------------------------------------------------------------------------
// error reporting
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(LS_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// device task table (staged into shared memory by every block)
// ---------------------------------------------------------------------------
constexpr int TPB = 256;          // threads per block of the scoring kernels
constexpr int NSLOT = 16;         // loop-variable slots that can exist (a chain has <= 16 loops)
constexpr int MAXACC = 16;
constexpr int MAXRANK = LS_MAX_RANK;
constexpr int MAXT = LS_MAX_TENSORS;
constexpr int MAXD = MAXT * MAXRANK;  // dimension slots of the generic layout
constexpr int MAXDV = 8;              // distinct loop variables per tensor dimension
constexpr int MAXTERM = 384;
constexpr int MAXCH = LS_MAX_CHAIN;
constexpr int MAXSTAGE = 64;
constexpr uint8_t NOSLOT = 0xFF;

struct DTerm {
  int32_t coef;
  uint32_t req;  // enable bits that must be set for the term to exist
  int32_t slot;
};

struct DExpr {
  int32_t konst;
  int16_t t0;  // first term in DTask::term (terms sorted by variable name)
  int16_t nt;
};

struct DXform {
  int8_t kind;
  uint8_t slot, new_slot;  // NOSLOT: the name never exists
  int8_t param;
  int8_t enable_bit, n_order, perm_shift, pad;
  int32_t value;
  uint8_t order[LS_MAX_ORDER];
};

struct DUnroll {
  int64_t u, c_inner, c_all;
};

// loop flags in the per-candidate state
constexpr uint8_t F_PAR = 1, F_UNR = 2, F_VEC = 4;

// one axis of an attached schedule space (points API)
struct DAxis {
  int8_t kind, param, bit, pad;
  uint32_t n, voff, pad2;
  uint64_t magic;  // floor(2^64 / n) + 1: q = umulhi(x, magic) == x / n for x < 2^32, n >= 2
};

struct __align__(16) DTask {
  int32_t n_base, n_xf, n_acc, n_tensors;
  int32_t L, S;  // loads / stores of the innermost body
  int32_t family, costs_integral, tid_slot, n_u;
  int32_t banks, warp_size, layout_rm, n_stage;
  int32_t has_shared, n_slots, n_chain, task_bytes;
  int32_t has_optional, pad1;
  uint32_t t_vmask[MAXT];  // slots used by each tensor's terms (valid when !has_optional)
  int64_t cap;
  int64_t c_init, c_latch, c_ret;
  double coef[LS_NFEAT_GPU];
  double ptx_cost[LS_I_COUNT];
  int64_t ptx_icost[LS_I_COUNT];
  double sm_underuse, warp_slack;
  const DUnroll* u_tab;
  int32_t base_ext[MAXCH], base_step[MAXCH];
  uint8_t base_slot[MAXCH], base_flags[MAXCH];
  DXform xf[LS_MAX_XFORMS];
  // accesses of the innermost body, program order
  uint8_t acc_tensor[MAXACC], acc_store[MAXACC];
  DExpr expr[MAXACC][MAXRANK];
  // tensors in first-appearance order among the accesses (CacheModel merge order)
  uint8_t t_rank[MAXT], t_nu[MAXT], t_uacc[MAXT][MAXACC], t_eb[MAXT], t_shared[MAXT];
  int32_t t_nacc[MAXT];
  int64_t t_stride[MAXT][MAXRANK];
  // dimension slots D = t * layout_rm + r
  uint8_t dim_nv[MAXD], dim_base[MAXD];
  uint8_t dim_var[MAXD][MAXDV];
  int32_t dim_count0[MAXD];
  uint64_t slot_dnib[NSLOT][3];  // nibble D of slot s: 1 + index of s in dim D's variable list
  // ---- tabulated path: every dimension count is a table lookup
  int32_t fast;      // 1: the task is eligible (4x4 layout, every dimension tabulated)
  int32_t tab_smem;  // the table is staged into shared memory
  int32_t tab_len;   // int32 entries
  int32_t pad3;
  const int32_t* tab;                  // device table: [dimension][key][expanded-variable mask]
  uint64_t chain0;                     // base chain, one slot per nibble
  uint32_t base_exist, base_unr, base_vec, base_par;  // slot masks of the base chain
  uint64_t vbits[NSLOT];               // bit dim_base[D] + x for every (D, x) with dim_var[D][x] == slot
  int32_t ftab_off[16], ftab_len[16];  // per dimension slot of the 4x4 layout
  uint32_t fsel[16];                   // (dim_base[D]) | (((1 << dim_nv[D]) - 1) << 8)
  int8_t fk_n[16], fk_src[16][3];      // key digits: 0..7 record param, 8 + b enable bit b
  int32_t fk_rad[16][3];
  int32_t fk_bound[LS_MAX_PARAMS];     // largest valid value of each record param
  int32_t tab_one, pad4;               // entry holding 1 (dimension slots the layout leaves unused)
  // ---- attached schedule space (points API)
  int32_t sp_n, pad5;
  const uint64_t* sp_vals;
  DAxis sp_ax[LS_MAX_AXES];
  // ---- tensor tables (points path): a tensor's whole footprint per (axis choices, stage mask)
  int32_t tt_ok, tt_len;
  const uint64_t* tt;
  uint32_t tt_off[4], tt_len_t[4], tt_nb[4];
  uint32_t tt_sh[4], tt_mk[4];            // byte offset of the row entry: (mall >> tt_sh) & tt_mk
  uint32_t tt_stride[4][LS_MAX_AXES];     // key stride of each axis (0: the axis does not affect the tensor)
  // ---- space-specialised points path: tile + reorder spaces whose transformed
  //      chain order is a function of the reorder choice alone
  int32_t sp_ok, sp_nchain;     // eligible + tables built; chain length after the tiles
  const uint64_t* sp_chain;     // per reorder choice: final chain, one slot per nibble
  const int32_t* sp_pstat;      // per reorder choice: status of apply_schedule with valid tiles
  int64_t c_inner1;             // innermost-block cycles with no unrolling (CPU family)
  // group tables of the space path: a tensor's dimensions are split into <= 2
  // groups; a group's table holds the product of its dimension counts, rows of 2^nb entries (stage
  // mask of nb <= 6 variables) keyed by the tile-axis choices, staged into shared memory.  Group slot
  // g = 2t + j owns bits 8g..8g+7 of the stage word, holding 4 * its stage mask (a byte offset).
  int32_t sd_len, sd_pad;             // uint32 entries (entries 0..3: the ones row)
  const int32_t* sd_tab;
  uint32_t sd_off[8];                 // byte offset of each group slot's table
  uint32_t sd_S[LS_MAX_AXES][8];      // byte stride of one choice of each axis in each group table
  uint64_t vb8[NSLOT];                // per loop slot: its stage bits in every group slot
  int8_t sd_gd[8][4];                 // dimension slots of each group (-1: none)
  int8_t sd_gx[8][4];                 // bit offset of each of them within the group's stage mask
  int8_t sd_nb[8];                    // stage bits of each group (rows of 2^nb entries)
  // static tiles: every tile is driven by one tile axis and splits a base loop not split before,
  // so a choice fixes both extents; sp_ext per choice = F | ceil(E/F) << 16 | out-of-range << 63
  int32_t sp_static, sp_narrow;         // static tiles; walk values proven to fit 32 bits (MODE 5)
  const uint64_t* sp_ext;
  uint8_t sp_tslot[LS_MAX_AXES], sp_tnew[LS_MAX_AXES];
  int32_t sp_n_untiled, pad8;            // static tiles: base loops no tile splits
  uint8_t sp_untiled[MAXCH], sp_untiled_pos[MAXCH];
  // ---- general trees: unified node ids, accesses 0..tr_na-1 (preorder), loops
  //      tr_na + j for base loop j (preorder; header j = base_slot/ext/step/flags[j]), tile loops after
  int32_t tree, tr_nl, tr_na, tr_root_first;
  int32_t tr_inline, tr_target, tr_dialect, tr_issue;  // inlined (unrolled / vector) loops possible: emulated emission
  int32_t tr_lat[LS_I_COUNT], tr_klass[LS_I_COUNT], tr_ucap[LS_I_COUNT];  // schedule_block tables (ls/ilp.py:18-35)
  uint8_t acc_decl[MAXACC];  // declaration index of each access's tensor (base register)
  int8_t tr_parent[32], tr_first[32], tr_next[32];
  uint8_t tr_nld[MAXCH], tr_nst[MAXCH];  // per base loop: its direct loads / stores (one access group)
  int64_t tr_c_hi[MAXCH], tr_c_hl[MAXCH];  // cycles of [group body + counter init] / [group body + latch]
  int32_t n_terms;
  DTerm term[MAXTERM];
};

struct ls_task {
  ls_task_desc desc;
  int device;
  DTask host;     // host copy (u_tab points to the current device table)
  DTask* d_task;  // current device copy
  std::vector<DUnroll> utab;
  std::vector<void*> retired;  // previous device copies / tables, freed on destroy
  std::vector<int> load_t, store_t;
  std::mutex mu;
  int num_sms;
  int path;            // LS_PATH_AUTO / LS_PATH_GENERIC / LS_PATH_TABULATED
  int32_t* d_tab;      // tabulated path's dimension-count table (owned)
  unsigned char* stage = nullptr;  // pinned staging of the host-buffer calls' results
  size_t stage_bytes = 0;
  bool stage_busy = false;
  unsigned char* ws = nullptr;     // cached top-k workspace (counters self-reset), tied to one stream
  size_t ws_bytes = 0;
  cudaStream_t ws_stream = nullptr;
  bool ws_busy = false;
  bool ws_dirty = false;           // a call failed after its first launch: re-initialise before reuse
};

// ---------------------------------------------------------------------------
// per-thread candidate state, kept in shared memory ([slot][thread] layout:
// bank-conflict free, no local-memory round trips)
// ---------------------------------------------------------------------------
struct Cand {
  int32_t* ext;    // [NSLOT][TPB]
  int32_t* step;   // [NSLOT][TPB]
  int32_t* stage;  // [n_stage][TPB]
  uint8_t* pos;    // [NSLOT][TPB], NOSLOT when the variable does not exist
  uint8_t* flg;    // [NSLOT][TPB]
  uint8_t* chain;  // [MAXCH][TPB]
  int n;
  uint32_t flags;
  __device__ __forceinline__ int32_t& E(int v) { return ext[v * TPB + threadIdx.x]; }
  __device__ __forceinline__ int32_t& St(int v) { return step[v * TPB + threadIdx.x]; }
  __device__ __forceinline__ int32_t& G(int i) { return stage[i * TPB + threadIdx.x]; }
  __device__ __forceinline__ uint8_t& P(int v) { return pos[v * TPB + threadIdx.x]; }
  __device__ __forceinline__ uint8_t& Fl(int v) { return flg[v * TPB + threadIdx.x]; }
  __device__ __forceinline__ uint8_t& C(int p) { return chain[p * TPB + threadIdx.x]; }
};

// Candidate state of the tabulated path: the chain is a register (one slot
// per nibble), loop flags are slot masks, only the extents stay in shared
// memory (they are indexed by a data-dependent slot).
struct FastCand {
  int32_t* ext;  // this thread's column of [NSLOT][TPB] (base + threadIdx.x)
  uint64_t chain;
  uint32_t unr, vec, par, exist;
  int n;
  uint32_t flags;
  __device__ __forceinline__ int32_t& E(int v) { return ext[v * TPB]; }
  __device__ __forceinline__ int C(int p) const { return (int)((chain >> (4 * p)) & 15u); }
  __device__ __forceinline__ uint8_t Fl(int v) const {
    return (uint8_t)((((par >> v) & 1u) ? 1 : 0) | (((unr >> v) & 1u) ? 2 : 0) | (((vec >> v) & 1u) ? 4 : 0));
  }
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ constexpr size_t cand_bytes(int n_slots, int n_chain, int n_stage) {
  return align16(sizeof(int32_t) * (size_t)n_slots * TPB) * 2 + align16(sizeof(int32_t) * (size_t)n_stage * TPB) +
         align16((size_t)n_slots * TPB) * 2 + align16((size_t)n_chain * TPB);
}

// Per-thread arrays sized to the task (slots, chain length, stages) so that
// more blocks fit per SM.
__device__ __forceinline__ Cand carve(unsigned char* p, const DTask& T) {
  Cand c;
  c.ext = reinterpret_cast<int32_t*>(p);
  p += align16(sizeof(int32_t) * (size_t)T.n_slots * TPB);
  c.step = reinterpret_cast<int32_t*>(p);
  p += align16(sizeof(int32_t) * (size_t)T.n_slots * TPB);
  c.stage = reinterpret_cast<int32_t*>(p);
  p += align16(sizeof(int32_t) * (size_t)T.n_stage * TPB);
  c.pos = p;
  p += align16((size_t)T.n_slots * TPB);
  c.flg = p;
  p += align16((size_t)T.n_slots * TPB);
  c.chain = p;
  return c;
}

// ---------------------------------------------------------------------------
// strided-interval algebra (ls/cache.py:28-77)
// ---------------------------------------------------------------------------
struct SI {
  int32_t lo, hi, stride, count;
  int32_t exact;
};

__device__ __forceinline__ uint32_t gcd_u32(uint32_t a, uint32_t b) {
  if (a == 0) return b;
  if (b == 0) return a;
  int sh = __ffs(a | b) - 1;
  a >>= __ffs(a) - 1;
  do {
    b >>= __ffs(b) - 1;
    uint32_t mn = min(a, b), mx = max(a, b);
    a = mn;
    b = mx - mn;
  } while (b);
  return a << sh;
}

// _si_sum (ls/cache.py:46-62)
__device__ __forceinline__ SI si_sum(SI a, SI b) {
  if (a.count == 1) {
    b.lo += a.lo;
    b.hi += a.lo;
    return b;
  }
  if (b.count == 1) {
    a.lo += b.lo;
    a.hi += b.lo;
    return a;
  }
  SI r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi;
  const bool af = a.stride <= b.stride;
  const int32_t gf = af ? a.stride : b.stride, gc = af ? b.stride : a.stride;
  const int32_t cf = af ? a.count : b.count;
  if (a.exact && b.exact && gc % gf == 0 && (int64_t)gc <= (int64_t)gf * cf) {
    r.stride = gf;
    r.count = (r.hi - r.lo) / gf + 1;
    r.exact = 1;
    return r;
  }
  const int32_t g = (int32_t)gcd_u32((uint32_t)a.stride, (uint32_t)b.stride);
  const int64_t est = g ? (r.hi - r.lo) / g + 1 : 1;
  const int64_t prod = (int64_t)a.count * b.count;
  r.stride = g;
  r.count = (int32_t)(est < prod ? est : prod);
  r.exact = 0;
  return r;
}

// _si_union (ls/cache.py:65-77)
__device__ __forceinline__ SI si_union(SI a, SI b) {
  if (a.lo == b.lo && a.hi == b.hi && a.stride == b.stride && a.count == b.count && a.exact == b.exact)
    return a;
  SI r;
  r.lo = min(a.lo, b.lo);
  r.hi = max(a.hi, b.hi);
  if (a.exact && b.exact && a.stride == b.stride && a.stride > 0 && (a.lo - b.lo) % a.stride == 0 &&
      a.lo <= b.hi + a.stride && b.lo <= a.hi + a.stride) {
    r.stride = a.stride;
    r.count = (r.hi - r.lo) / a.stride + 1;
    r.exact = 1;
    return r;
  }
  const uint32_t dl = (uint32_t)abs(a.lo - b.lo);
  const int32_t g = (int32_t)gcd_u32(gcd_u32((uint32_t)a.stride, (uint32_t)b.stride), dl);
  const int64_t est = g ? (r.hi - r.lo) / g + 1 : 1;
  const int64_t sum = (int64_t)a.count + b.count;
  r.stride = g;
  r.count = (int32_t)(est < sum ? est : sum);
  r.exact = 0;
  return r;
}

__device__ __forceinline__ bool present(const DTerm& t, uint32_t flags) { return (t.req & ~flags) == 0; }

// expr_range (ls/cache.py:80-96): terms in name order; variables at chain
// positions >= thr expanded, all others held at 0
__device__ __forceinline__ SI expr_range(const DTask& T, const DExpr& e, Cand& c, int thr) {
  SI acc;
  acc.lo = acc.hi = e.konst;
  acc.stride = 0;
  acc.count = 1;
  acc.exact = 1;
  for (int k = 0; k < e.nt; ++k) {
    const DTerm& t = T.term[e.t0 + k];
    const int u = t.slot;
    const int pu = c.P(u);
    if (!present(t, c.flags) || pu == NOSLOT || pu < thr) continue;
    const int32_t E = c.E(u);
    if (E == 1) continue;
    const int32_t d = t.coef * c.St(u);
    SI s;
    s.lo = d > 0 ? 0 : d * (E - 1);
    s.hi = d > 0 ? d * (E - 1) : 0;
    s.stride = abs(d);
    s.count = E;
    s.exact = 1;
    acc = si_sum(acc, s);
  }
  return acc;
}

__device__ __forceinline__ int64_t unroll_lookup(const DTask& T, int64_t U, bool inner, bool* ok) {
  int lo = 0, hi = T.n_u - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int64_t u = __ldg(&T.u_tab[mid].u);
    if (u == U) {
      *ok = true;
      return inner ? __ldg(&T.u_tab[mid].c_inner) : __ldg(&T.u_tab[mid].c_all);
    }
    if (u < U)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  *ok = false;
  return 0;
}

// Apply the record's transforms to the base chain (ls/ir.py:361-474).
__device__ int apply_transforms(const DTask& T, const ls_record& r, Cand& c) {
  c.n = T.n_base;
  c.flags = r.flags;
  for (int v = 0; v < T.n_slots; ++v) c.P(v) = NOSLOT;
  for (int p = 0; p < T.n_base; ++p) {
    const int v = T.base_slot[p];
    c.C(p) = (uint8_t)v;
    c.P(v) = (uint8_t)p;
    c.E(v) = T.base_ext[p];
    c.St(v) = T.base_step[p];
    c.Fl(v) = T.base_flags[p];
  }
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.enable_bit >= 0 && !((r.flags >> xf.enable_bit) & 1u)) continue;
    const int v = xf.slot;
    const bool exists = v != NOSLOT && c.P(v) != NOSLOT;
    switch (xf.kind) {
      case LS_XF_TILE:
      case LS_XF_VECTORIZE: {
        if (!exists || xf.new_slot == NOSLOT) return LS_ST_NO_LOOP;
        const int32_t F = xf.param >= 0 ? (int32_t)r.param[xf.param] : xf.value;
        const int32_t Ev = c.E(v);
        if (xf.kind == LS_XF_VECTORIZE) {
          if (F == 0) return LS_ST_VEC_ZERO;
          if (Ev % F != 0) return LS_ST_VEC_DIVIDE;
        }
        if (F < 1 || F > Ev) return LS_ST_TILE_RANGE;
        if (c.n >= MAXCH) return LS_ST_OVERFLOW;
        const int u = xf.new_slot;
        const int p = c.P(v);
        for (int q = c.n; q > p + 1; --q) {
          const int w = c.C(q - 1);
          c.C(q) = (uint8_t)w;
          c.P(w) = (uint8_t)q;
        }
        c.C(p + 1) = (uint8_t)u;
        c.P(u) = (uint8_t)(p + 1);
        c.n++;
        c.E(u) = F;
        c.St(u) = c.St(v);
        c.Fl(u) = xf.kind == LS_XF_VECTORIZE ? F_VEC : 0;
        c.E(v) = (Ev + F - 1) / F;
        c.St(v) *= F;
        c.Fl(v) &= (uint8_t)~F_VEC;  // the outer loop is rebuilt without vector_width
        break;
      }
      case LS_XF_REORDER: {
        const int m = xf.n_order;
        if (m < 2) break;
        uint8_t vars[LS_MAX_ORDER];
        for (int j = 0; j < m; ++j) {
          const int nib = (int)((r.perm >> (4 * (xf.perm_shift + j))) & 0xF);
          const int w = nib < m ? xf.order[nib] : NOSLOT;
          if (w == NOSLOT || c.P(w) == NOSLOT) return LS_ST_NO_LOOP;
          vars[j] = (uint8_t)w;
        }
        uint32_t seen = 0;
        int pmin = MAXCH, pmax = -1;
        for (int j = 0; j < m; ++j) {
          const uint32_t bit = 1u << vars[j];
          if (seen & bit) return LS_ST_REORDER_MISSING;
          seen |= bit;
          const int pv = c.P(vars[j]);
          pmin = min(pmin, pv);
          pmax = max(pmax, pv);
        }
        if (pmax - pmin != m - 1) return LS_ST_REORDER_CHAIN;
        for (int j = 0; j < m; ++j) {
          c.C(pmin + j) = vars[j];
          c.P(vars[j]) = (uint8_t)(pmin + j);
        }
        break;
      }
      case LS_XF_UNROLL:
      case LS_XF_PARALLEL:
        if (!exists) return LS_ST_NO_LOOP;
        c.Fl(v) |= xf.kind == LS_XF_UNROLL ? F_UNR : F_PAR;
        break;
      default:
        return LS_ST_UNSUPPORTED;
    }
  }
  return LS_OK;
}

// record parameter p without a dynamically indexed (local-memory) array
__device__ __forceinline__ uint32_t rparam(const ls_record& r, int p) {
  uint64_t lo, hi;
  memcpy(&lo, &r.param[0], 8);
  memcpy(&hi, &r.param[4], 8);
  return (uint32_t)(((p < 4 ? lo : hi) >> (16 * (p & 3))) & 0xFFFFu);
}

// position of slot v in a nibble-packed chain (v must be on the chain): the
// lowest zero nibble of chain ^ v is exact (borrows only flag higher nibbles)
__device__ __forceinline__ int chain_find(uint64_t chain, int v) {
  const uint64_t x = chain ^ (0x1111111111111111ull * (uint64_t)v);
  const uint64_t z = (x - 0x1111111111111111ull) & ~x & 0x8888888888888888ull;
  return (__ffsll((long long)z) - 1) >> 2;
}

// apply_transforms on the register chain (tabulated path).  Same checks in
// the same order as apply_transforms, hence the same status codes.
__device__ int apply_fast(const DTask& T, const ls_record& r, FastCand& c) {
  c.n = T.n_base;
  c.flags = r.flags;
  c.chain = T.chain0;
  c.exist = T.base_exist;
  c.unr = T.base_unr;
  c.vec = T.base_vec;
  c.par = T.base_par;
  for (int p = 0; p < T.n_base; ++p) c.E(T.base_slot[p]) = T.base_ext[p];
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.enable_bit >= 0 && !((r.flags >> xf.enable_bit) & 1u)) continue;
    const int v = xf.slot;
    const bool exists = v != NOSLOT && ((c.exist >> v) & 1u);
    switch (xf.kind) {
      case LS_XF_TILE:
      case LS_XF_VECTORIZE: {
        if (!exists || xf.new_slot == NOSLOT) return LS_ST_NO_LOOP;
        const int32_t F = xf.param >= 0 ? (int32_t)rparam(r, xf.param) : xf.value;
        const int32_t Ev = c.E(v);
        if (xf.kind == LS_XF_VECTORIZE) {
          if (F == 0) return LS_ST_VEC_ZERO;
          if (Ev % F != 0) return LS_ST_VEC_DIVIDE;
        }
        if (F < 1 || F > Ev) return LS_ST_TILE_RANGE;
        if (c.n >= MAXCH) return LS_ST_OVERFLOW;
        const int u = xf.new_slot;
        const int q = chain_find(c.chain, v) + 1;  // q <= 15
        const uint64_t low = (1ull << (4 * q)) - 1;
        c.chain = (c.chain & low) | ((uint64_t)u << (4 * q)) | ((c.chain & ~low) << 4);
        c.n++;
        c.exist |= 1u << u;
        c.E(u) = F;
        c.E(v) = (Ev + F - 1) / F;
        c.unr &= ~(1u << u);
        c.par &= ~(1u << u);
        c.vec = (c.vec & ~((1u << u) | (1u << v))) | (xf.kind == LS_XF_VECTORIZE ? (1u << u) : 0u);
        break;
      }
      case LS_XF_REORDER: {
        const int m = xf.n_order;
        if (m < 2) break;
        uint64_t seg = 0;
        for (int j = 0; j < m; ++j) {
          const int nib = (int)((r.perm >> (4 * (xf.perm_shift + j))) & 0xF);
          const int w = nib < m ? xf.order[nib] : NOSLOT;
          if (w == NOSLOT || !((c.exist >> w) & 1u)) return LS_ST_NO_LOOP;
          seg |= (uint64_t)w << (4 * j);
        }
        uint32_t seen = 0;
        for (int j = 0; j < m; ++j) {
          const uint32_t bit = 1u << ((seg >> (4 * j)) & 15u);
          if (seen & bit) return LS_ST_REORDER_MISSING;
          seen |= bit;
        }
        int pmin = 0;
        if (m != c.n) {  // m distinct loops of an n-chain: contiguous iff their positions span m - 1
          int pmax = -1;
          pmin = MAXCH;
          for (int j = 0; j < m; ++j) {
            const int pv = chain_find(c.chain, (int)((seg >> (4 * j)) & 15u));
            pmin = min(pmin, pv);
            pmax = max(pmax, pv);
          }
          if (pmax - pmin != m - 1) return LS_ST_REORDER_CHAIN;
        }
        const uint64_t mk = m >= 16 ? ~0ull : ((1ull << (4 * m)) - 1);
        c.chain = (c.chain & ~(mk << (4 * pmin))) | (seg << (4 * pmin));
        break;
      }
      case LS_XF_UNROLL:
      case LS_XF_PARALLEL:
        if (!exists) return LS_ST_NO_LOOP;
        if (xf.kind == LS_XF_UNROLL)
          c.unr |= 1u << v;
        else
          c.par |= 1u << v;
        break;
      default:
        return LS_ST_UNSUPPORTED;
    }
  }
  return LS_OK;
}

__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }

// bank_conflict_factor (ls/ptx.py:264-307) of innermost access a
template <class CT>
__device__ int64_t bank_factor(const DTask& T, CT& c, int a) {
  const int t = T.acc_tensor[a];
  const int rank = T.t_rank[t];
  uint32_t used = 0;
  for (int d = 0; d < rank; ++d) {
    const DExpr& e = T.expr[a][d];
    for (int k = 0; k < e.nt; ++k)
      if (present(T.term[e.t0 + k], c.flags)) used |= 1u << T.term[e.t0 + k].slot;
  }
  int tid = -1;
  if (T.tid_slot >= 0 && ((used >> T.tid_slot) & 1u)) {
    tid = T.tid_slot;
  } else {
    for (int p = 0; p < c.n; ++p) {
      const int v = c.C(p);
      if ((c.Fl(v) & F_PAR) && ((used >> v) & 1u)) tid = v;
    }
  }
  if (tid < 0) return 1;  // every lane hits one word
  const int lanes = min(T.warp_size, c.E(tid));
  int64_t A = 0, B = 0;
  for (int d = 0; d < rank; ++d) {
    const DExpr& e = T.expr[a][d];
    int64_t ct = 0;
    for (int k = 0; k < e.nt; ++k) {
      const DTerm& tm = T.term[e.t0 + k];
      if (present(tm, c.flags) && tm.slot == tid) ct += tm.coef;
    }
    A += (int64_t)e.konst * T.t_stride[t][d];
    B += ct * T.t_stride[t][d];
  }
  // words are monotone in the lane id, so equal words are adjacent
  uint8_t cnt[64];
  for (int b = 0; b < T.banks; ++b) cnt[b] = 0;
  int64_t prev = 0, best = 0;
  for (int l = 0; l < lanes; ++l) {
    const int64_t num = (A + B * l) * T.t_eb[t];
    const int64_t w = num >= 0 ? num / 4 : -((-num + 3) / 4);
    if (l == 0 || w != prev) {
      int64_t b = w % T.banks;
      if (b < 0) b += T.banks;
      best = max(best, (int64_t)++cnt[b]);
    }
    prev = w;
  }
  return best;
}

// thread_cycles in line order (ls/ptx.py:225-235), for non-integral cost tables
template <class CT>
__device__ double ptx_work_ordered(const DTask& T, CT& c, int k, double wi) {
  const double* pc = T.ptx_cost;
  double wpre[MAXCH], wpost[MAXCH];
  int32_t rem[MAXCH];
  {
    double w = 1.0;
    int j = 0;
    for (int p = 0; p < c.n; ++p) {
      const int v = c.C(p);
      if (c.Fl(v) & (F_VEC | F_UNR)) continue;
      wpre[p] = w;
      if (!(j + 8 <= k - 1)) w *= (double)c.E(v);
      wpost[p] = w;
      ++j;
    }
  }
  double work = 0.0;
  int p = 0;
  bool down = true;
  while (true) {
    if (down) {
      if (p == c.n) {
        for (int a = 0; a < T.L; ++a) work = rn_add(work, rn_mul(pc[LS_I_LOAD], wi));
        for (int a = 0; a < T.S; ++a) {
          work = rn_add(work, rn_mul(pc[LS_I_FMA], wi));
          work = rn_add(work, rn_mul(pc[LS_I_STORE], wi));
        }
        down = false;
        p = c.n - 1;
        continue;
      }
      const int v = c.C(p);
      const uint8_t fl = c.Fl(v);
      if (fl & (F_VEC | F_UNR)) {
        rem[p] = (fl & F_VEC) ? 1 : c.E(v);
      } else {
        work = rn_add(work, rn_mul(pc[LS_I_INIT], wpre[p]));
      }
      ++p;
    } else {
      if (p < 0) break;
      const int v = c.C(p);
      const uint8_t fl = c.Fl(v);
      if (fl & (F_VEC | F_UNR)) {
        if (--rem[p] > 0) {
          ++p;
          down = true;
        } else {
          --p;
        }
      } else {
        work = rn_add(work, rn_mul(pc[LS_I_ADD], wpost[p]));
        work = rn_add(work, rn_mul(pc[LS_I_CMP], wpost[p]));
        work = rn_add(work, rn_mul(pc[LS_I_BRANCH], wpost[p]));
        --p;
      }
    }
  }
  return rn_add(work, pc[LS_I_RET]);
}

template <class CT>
__device__ int features_score(const DTask& T, CT& c, int64_t dmov, double* f, double* score);

// extract_features + score of one candidate (ls/cost.py:132-161).  TM x RM is
// the compile-time tensor x dimension layout of the register-resident walk.
template <int TM, int RM>
__device__ int eval_candidate(const DTask& T, const ls_record& r, Cand& c, double* f, double* score) {
  int st = apply_transforms(T, r, c);
  if (st) return st;
  const int nT = T.n_tensors;

  // ---- movement model (CacheModel._visit_loop, ls/cache.py:167-236) ----------
  // (a) for every tensor dimension and every variable of it, the dimension's
  //     count once the chain walk has passed that variable (all its variables
  //     at positions >= that variable's position expanded)
  for (int t = 0; t < nT; ++t) {
    for (int rr = 0; rr < T.t_rank[t]; ++rr) {
      const int D = t * RM + rr;
      for (int j = 0; j < T.dim_nv[D]; ++j) {
        const int thr = c.P(T.dim_var[D][j]);
        if (thr == NOSLOT) continue;
        SI u = expr_range(T, T.expr[T.t_uacc[t][0]][rr], c, thr);
        for (int a = 1; a < T.t_nu[t]; ++a) u = si_union(u, expr_range(T, T.expr[T.t_uacc[t][a]][rr], c, thr));
        c.G(T.dim_base[D] + j) = u.count;
      }
    }
  }
  // (b) walk the chain innermost-first with counts, footprints and movement in registers
  int32_t cur[TM * RM];
  uint32_t tmask[TM];
  int64_t Fb[TM], dm[TM];
  uint32_t reuse = 0;
#pragma unroll
  for (int D = 0; D < TM * RM; ++D) cur[D] = T.dim_count0[D];
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    tmask[t] = 0;
    dm[t] = 0;
    Fb[t] = 0;
    if (t < nT) {
      int64_t F = 1;
#pragma unroll
      for (int rr = 0; rr < RM; ++rr) F *= cur[t * RM + rr];
      Fb[t] = F;
      dm[t] = T.t_nacc[t];
      reuse |= 1u << t;
      tmask[t] = T.t_vmask[t];
      if (T.has_optional) {
        tmask[t] = 0;
        for (int a = 0; a < T.t_nu[t]; ++a)
        for (int rr = 0; rr < T.t_rank[t]; ++rr) {
          const DExpr& e = T.expr[T.t_uacc[t][a]][rr];
          for (int q = 0; q < e.nt; ++q)
            if (present(T.term[e.t0 + q], c.flags)) tmask[t] |= 1u << T.term[e.t0 + q].slot;
        }
      }
    }
  }
  const int64_t cap = T.cap;
  for (int p = c.n - 1; p >= 0; --p) {
    const int v = c.C(p);
    const int64_t E = c.E(v);
#pragma unroll
    for (int w = 0; w < (TM * RM + 15) / 16; ++w) {
      const uint64_t nib = T.slot_dnib[v][w];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int D = 16 * w + q;
        if (D < TM * RM) {
          const int x = (int)((nib >> (4 * q)) & 15u);
          if (x) cur[D] = c.G(T.dim_base[D] + x - 1);
        }
      }
    }
    int64_t single = 0;
#pragma unroll
    for (int t = 0; t < TM; ++t) single += Fb[t];
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      if (t < nT) {
        int64_t Ff = 1;
#pragma unroll
        for (int rr = 0; rr < RM; ++rr) Ff *= cur[t * RM + rr];
        const bool uses = (tmask[t] >> v) & 1u;
        bool ru = (reuse >> t) & 1u;
        if (single > cap && !uses) ru = false;
        const int64_t per = (single <= cap || ru) ? Ff : dm[t] * E;
        if (Ff > cap) ru = false;
        dm[t] = per;
        reuse = ru ? (reuse | (1u << t)) : (reuse & ~(1u << t));
        Fb[t] = Ff;
      }
    }
  }
  int64_t dmov = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) dmov += dm[t];
  return features_score(T, c, dmov, f, score);
}

// Emitted-code features + linear score of a transformed candidate (shared by
// both paths): ls/asm.py:250-337, ls/ilp.py:262-271, ls/ptx.py:90-327,
// ls/cost.py:132-161.
template <class CT>
__device__ int features_score(const DTask& T, CT& c, int64_t dmov, double* f, double* score) {
  // ---- emitted-block structure of the transformed chain -----------------------
  // branching loops j = 0..k-1 (not unrolled/vectorized); R_j = copies of loop j
  // emitted because unrolled loops above it inline their bodies R_j times
  // (ls/ir.py:619-626); U = body copies in the innermost block.
  int k = 0;
  for (int p = 0; p < c.n; ++p) k += (c.Fl(c.C(p)) & (F_VEC | F_UNR)) ? 0 : 1;
  int64_t W = 1, Wp = 1, R = 1, Uin = 1;
  int64_t sumR = 0, sumW = 0, sumRl = 0, Wlast = 1, Rlast = 1;
  int64_t ptx_loops = 0;  // sum_j R_j * (c_mov W'_{j-1} + (c_add+c_setp+c_bra) W'_j), integral costs
  const int64_t* ic = T.ptx_icost;
  {
    int j = 0;
    for (int p = 0; p < c.n; ++p) {
      const int v = c.C(p);
      const uint8_t fl = c.Fl(v);
      const int64_t e = c.E(v);
      if (fl & F_VEC) continue;
      if (fl & F_UNR) {
        R *= e;
        Uin *= e;
        continue;
      }
      const int64_t Wprev = Wp;
      W *= e;
      if (!(j + 8 <= k - 1)) Wp *= e;  // PTX counter registers repeat every 8 depths (ls/ir.py:627, ls/ptx.py:163-169)
      sumR += R;
      if (j < k - 1) {
        sumW += W;
        sumRl += R;
      }
      if (T.family == LS_FAMILY_GPU)
        ptx_loops += R * (ic[LS_I_INIT] * Wprev + (ic[LS_I_ADD] + ic[LS_I_CMP] + ic[LS_I_BRANCH]) * Wp);
      Wlast = W;
      Rlast = R;
      Uin = 1;
      ++j;
    }
  }
  const int64_t L = T.L, S = T.S;
  int nf;
  if (T.family == LS_FAMILY_CPU) {
    // only the first emitted copy of each loop block is matched by the greedy
    // loop_map (ls/asm.py:250-294); every block is scheduled (ls/ilp.py:262-271)
    int64_t ilp, nld = 0, nst = 0;
    bool ok;
    if (k == 0) {
      ilp = unroll_lookup(T, R, false, &ok);
      if (!ok) return LS_ST_UNROLL_TABLE;
    } else {
      const int64_t ci = unroll_lookup(T, Uin, true, &ok);
      if (!ok) return LS_ST_UNROLL_TABLE;
      ilp = T.c_init * (sumR - (k - 1) + sumW) + ci * (Wlast + Rlast - 1) + T.c_latch * sumRl + T.c_ret;
      nld = L * Uin * Wlast;
      nst = S * Uin * Wlast;
    }
    f[0] = (double)nst;  // n_fma == n_vstore: one fma per store
    f[1] = (double)nld;
    f[2] = (double)nst;
    f[3] = (double)dmov;
    f[4] = (double)ilp;
    nf = LS_NFEAT_CPU;
  } else {
    // loop_map_ptx counts every emitted copy (ls/ptx.py:90-108, 196-235)
    const int64_t Ubody = R;  // R_{k-1} * U_inner == all unrolled extents
    double work;
    if (T.costs_integral) {
      work = (double)(ptx_loops + Ubody * Wp * (L * ic[LS_I_LOAD] + S * (ic[LS_I_FMA] + ic[LS_I_STORE])) +
                      ic[LS_I_RET]);
    } else {
      work = ptx_work_ordered(T, c, k, (double)Wp);
    }
    double smem = 0.0;
    if (T.has_shared) {  // shared-memory ops (ls/ptx.py:310-327): vector loops count once
      int64_t vol = 1;
      for (int p = 0; p < c.n; ++p) {
        const int v = c.C(p);
        vol *= (c.Fl(v) & F_VEC) ? 1 : c.E(v);
      }
      for (int a = 0; a < T.n_acc; ++a)
        if (T.t_shared[T.acc_tensor[a]]) smem = rn_add(smem, (double)(vol * bank_factor(T, c, a)));
    }
    f[0] = work;
    f[1] = T.sm_underuse;
    f[2] = T.warp_slack;
    f[3] = smem;
    f[4] = (double)(S * Ubody * Wp);
    f[5] = (double)(L * Ubody * Wp);
    f[6] = (double)(S * Ubody * Wp);
    nf = LS_NFEAT_GPU;
  }
  double total = 0.0;
  for (int q = 0; q < nf; ++q) {
    if (!(f[q] >= 0.0) || isinf(f[q])) return LS_ST_BAD_FEATURE;
    total = rn_add(total, rn_mul(T.coef[q], f[q]));
  }
  *score = total;
  return LS_OK;
}

// Tabulated path: the cache model's dimension counts are
// lookups.  For dimension D, the count after the walk has passed a set of D's
// variables is a function of (the record fields that determine those
// variables' extents/steps and term presence = the key, the set = a bit mask);
// ls_task_create tabulates it once per task with the generic fold
// (build_tab_kernel), so per candidate the walk only ORs a per-slot bit mask
// and multiplies looked-up counts.
// Decode a space point (mixed radix, axis 0 most significant) into the record
// the host packer would have produced for the same choices (pack.SpaceTemplate).
template <bool KEYS>
__device__ __forceinline__ int point_record(const DTask& T, uint64_t x, ls_record& r, uint32_t* kt, uint32_t& pch) {
  uint64_t lo = 0, hi = 0, perm = 0;
  uint32_t flags = 0;
  if constexpr (KEYS) {
#pragma unroll
    for (int t = 0; t < 4; ++t) kt[t] = 0;
  }
  for (int a = T.sp_n - 1; a >= 0; --a) {
    const DAxis& ax = T.sp_ax[a];
    uint32_t c;
    if (a == 0) {
      if (x >= ax.n) return LS_ST_POINT_RANGE;
      c = (uint32_t)x;
    } else if (ax.n == 1) {
      c = 0;
    } else {
      const uint64_t q = (x >> 32) ? x / ax.n : __umul64hi(x, ax.magic);
      c = (uint32_t)(x - q * ax.n);
      x = q;
    }
    if constexpr (KEYS) {
#pragma unroll
      for (int t = 0; t < 4; ++t) kt[t] += c * T.tt_stride[t][a];
    }
    if (ax.kind == LS_AX_BIT) {
      flags |= c << ax.bit;
      continue;
    }
    const uint64_t v = __ldg(reinterpret_cast<const unsigned long long*>(T.sp_vals) + ax.voff + c);
    if (ax.kind == LS_AX_PERM) {
      perm |= v;
      pch = c;
      continue;
    }
    if (ax.param < 4)
      lo |= v << (16 * ax.param);
    else
      hi |= v << (16 * (ax.param - 4));
    if (ax.kind == LS_AX_VEC && v != 0) flags |= 1u << ax.bit;
  }
  memcpy(&r.param[0], &lo, 8);
  memcpy(&r.param[4], &hi, 8);
  r.perm = perm;
  r.flags = flags;
  r.tag = 0;
  if constexpr (KEYS) {
#pragma unroll
    for (int t = 0; t < 4; ++t) kt[t] = 8u * (T.tt_off[t] + (kt[t] << T.tt_nb[t]));
  }
  return LS_OK;
}

// Candidate source of the scoring kernels: SRC 0 = ls_record array, 1 = points.
template <int SRC, bool KEYS>
__device__ __forceinline__ int load_cand(const DTask& T, const void* __restrict__ src, int pbytes, int64_t i,
                                         ls_record& r, uint32_t* kt, uint32_t& pch);

template <int TM, int RM, bool SMT>
__device__ __forceinline__ int32_t tab_at(const int32_t* __restrict__ tab, int32_t i) {
  if constexpr (SMT)
    return tab[i];
  else
    return __ldg(&tab[i]);
}

// The movement walk of the tabulated paths (CacheModel._visit_loop,
// ls/cache.py:167-236, chain form): fp(t) is tensor t's footprint for the
// stage bits in `mall` (every variable at positions >= p expanded).
template <int TM, class FP>
__device__ __forceinline__ int walk_score(const DTask& T, FastCand& c, uint64_t& mall, FP fp, double* f,
                                          double* score) {
  const int nT = T.n_tensors;
  uint32_t tmask[TM];
  int64_t Fb[TM], dm[TM];
  uint32_t reuse = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    tmask[t] = 0;
    dm[t] = 0;
    Fb[t] = 0;
    if (t < nT) {
      Fb[t] = fp(t);
      dm[t] = T.t_nacc[t];
      reuse |= 1u << t;
      tmask[t] = T.t_vmask[t];
      if (T.has_optional) {
        tmask[t] = 0;
        for (int a = 0; a < T.t_nu[t]; ++a)
          for (int rr = 0; rr < T.t_rank[t]; ++rr) {
            const DExpr& e = T.expr[T.t_uacc[t][a]][rr];
            for (int q = 0; q < e.nt; ++q)
              if (present(T.term[e.t0 + q], c.flags)) tmask[t] |= 1u << T.term[e.t0 + q].slot;
          }
      }
    }
  }
  const int64_t cap = T.cap;
  for (int p = c.n - 1; p >= 0; --p) {
    const int v = c.C(p);
    const int64_t E = c.E(v);
    mall |= T.vbits[v];
    int64_t single = 0;
#pragma unroll
    for (int t = 0; t < TM; ++t) single += Fb[t];
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      if (t < nT) {
        const int64_t Ff = fp(t);
        const bool uses = (tmask[t] >> v) & 1u;
        bool ru = (reuse >> t) & 1u;
        if (single > cap && !uses) ru = false;
        const int64_t per = (single <= cap || ru) ? Ff : dm[t] * E;
        if (Ff > cap) ru = false;
        dm[t] = per;
        reuse = ru ? (reuse | (1u << t)) : (reuse & ~(1u << t));
        Fb[t] = Ff;
      }
    }
  }
  int64_t dmov = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) dmov += dm[t];
  return features_score(T, c, dmov, f, score);
}

template <int TM, int RM, bool SMT>
__device__ int eval_fast(const DTask& T, const int32_t* __restrict__ tab, const ls_record& r, FastCand& c,
                         double* f, double* score) {
  const int st = apply_fast(T, r, c);
  if (st) return st;
  // byte offset of each dimension's row for this candidate's key
  uint32_t kb[TM * RM];
#pragma unroll
  for (int D = 0; D < TM * RM; ++D) {
    int32_t k = 0;
    const int nd = T.fk_n[D];
    for (int q = 0; q < nd; ++q) {
      const int src = T.fk_src[D][q];
      int32_t val;
      if (src < LS_MAX_PARAMS) {
        val = (int32_t)rparam(r, src);
        if (val > T.fk_bound[src]) val = 0;  // only possible when no applied transform reads it
      } else {
        val = (int32_t)((r.flags >> (src - LS_MAX_PARAMS)) & 1u);
      }
      k = k * T.fk_rad[D][q] + val;
    }
    kb[D] = 4u * (uint32_t)(T.ftab_off[D] + (k << T.dim_nv[D]));
  }
  uint64_t mall = 0;
  const char* tb = reinterpret_cast<const char*>(tab);
  auto cnt = [&](int D) -> uint32_t {
    const uint32_t sel = T.fsel[D];
    const uint32_t off = kb[D] + ((uint32_t)(mall >> (sel & 0xFFu)) & (sel >> 8));
    return (uint32_t)tab_at<TM, RM, SMT>(reinterpret_cast<const int32_t*>(tb + off), 0);
  };
  static_assert(RM == 4, "tabulated path uses the 4x4 layout");
  auto prod = [&](int t) -> int64_t {
    const uint64_t a = (uint64_t)cnt(t * 4 + 0) * cnt(t * 4 + 1);
    const uint64_t b = (uint64_t)cnt(t * 4 + 2) * cnt(t * 4 + 3);
    return (int64_t)(a * b);
  };
  return walk_score<TM>(T, c, mall, prod, f, score);
}

// Extents/steps of every slot for given record params/flags: apply_schedule's
// Tile/Vectorize arithmetic (ls/ir.py:361-382) without the chain.  Transforms
// that would make a candidate fail are skipped (such candidates never look
// their counts up).
__device__ void sim_slots(const DTask& T, const int32_t* prm, uint32_t flags, int32_t* E, int32_t* St,
                          uint32_t& exist) {
  exist = T.base_exist;
  for (int p = 0; p < T.n_base; ++p) {
    E[T.base_slot[p]] = T.base_ext[p];
    St[T.base_slot[p]] = T.base_step[p];
  }
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.kind != LS_XF_TILE && xf.kind != LS_XF_VECTORIZE) continue;
    if (xf.enable_bit >= 0 && !((flags >> xf.enable_bit) & 1u)) continue;
    const int v = xf.slot, u = xf.new_slot;
    if (v == NOSLOT || u == NOSLOT || !((exist >> v) & 1u)) continue;
    const int32_t F = xf.param >= 0 ? prm[xf.param] : xf.value;
    if (F < 1 || F > E[v]) continue;
    E[u] = F;
    St[u] = St[v];
    E[v] = (E[v] + F - 1) / F;
    St[v] *= F;
    exist |= 1u << u;
  }
}

// Count of dimension D (4x4 layout) with the variables of `mask` (bit x =
// dim_var[D][x]) expanded: the generic fold, expr_range + _si_union
// (ls/cache.py:80-130) in the same order.
__device__ int32_t dim_count(const DTask& T, int D, uint32_t mask, uint32_t flags, const int32_t* E, const int32_t* St,
                             uint32_t exist) {
  uint32_t expanded = 0;
  for (int x = 0; x < T.dim_nv[D]; ++x)
    if ((mask >> x) & 1u) expanded |= 1u << T.dim_var[D][x];
  const int t = D / 4, rr = D % 4;
  SI u;
  for (int a = 0; a < T.t_nu[t]; ++a) {
    const DExpr& ex = T.expr[T.t_uacc[t][a]][rr];
    SI acc;
    acc.lo = acc.hi = ex.konst;
    acc.stride = 0;
    acc.count = 1;
    acc.exact = 1;
    for (int k = 0; k < ex.nt; ++k) {
      const DTerm& tm = T.term[ex.t0 + k];
      const int w = tm.slot;
      if (!present(tm, flags) || !((expanded >> w) & 1u) || !((exist >> w) & 1u)) continue;
      const int32_t Ew = E[w];
      if (Ew == 1) continue;
      const int32_t d = tm.coef * St[w];
      SI s;
      s.lo = d > 0 ? 0 : d * (Ew - 1);
      s.hi = d > 0 ? d * (Ew - 1) : 0;
      s.stride = abs(d);
      s.count = Ew;
      s.exact = 1;
      acc = si_sum(acc, s);
    }
    u = a == 0 ? acc : si_union(u, acc);
  }
  return u.count;
}

// Tensor-table path (points only): one 8-byte lookup gives a tensor footprint.
template <int TM>
__device__ int eval_tensor(const DTask& T, const ls_record& r, const uint32_t* kt, FastCand& c, double* f,
                           double* score) {
  const int st = apply_fast(T, r, c);
  if (st) return st;
  uint64_t mall = 0;
  const char* tb = reinterpret_cast<const char*>(T.tt);
  auto fp = [&](int t) -> int64_t {
    const uint32_t off = kt[t] + ((uint32_t)(mall >> T.tt_sh[t]) & T.tt_mk[t]);
    return (int64_t)__ldg(reinterpret_cast<const unsigned long long*>(tb + off));
  };
  return walk_score<TM>(T, c, mall, fp, f, score);
}

// Space-specialised points path.  Eligible spaces only hold
// tile-factor and reorder axes over unconditional Tile transforms followed by
// one Reorder, with no unroll/vector/parallel marks: every loop of the
// transformed chain branches, its order is a function of the reorder choice
// alone (tabulated per choice by ls_task_set_space) and only the extents
// depend on the tile choices.  The movement walk, the emitted-block terms and
// the score then fuse into one innermost-first pass over the chain:
//   CPU  sum_{j<n-1} W_j      = E_0(1 + E_1(1 + ... E_{n-2}))       (Horner, exact integers)
//        ilp = c_init (1 + sum W) + c_inner(1) W_{n-1} + c_latch (n-1) + c_ret
//   PTX  W'_j uses extent 1 for loops 8+ above the innermost (counter-register wrap),
//        sum_j W'_{j-1} = 1 + A, sum_j W'_j = A + W'_{n-1}, A = sum_{j<n-1} W'_j
// which are the general closed forms of features_score with every R_j = 1.
__device__ __forceinline__ uint64_t load_point(const void* __restrict__ src, int pbytes, int64_t i) {
  return pbytes == 4 ? (uint64_t)__ldg(reinterpret_cast<const unsigned int*>(src) + i)
                     : (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(src) + i);
}

template <int TM, bool NARROW>
__device__ int eval_space(const DTask& T, const int32_t* __restrict__ sdt, uint64_t x, FastCand& c, double* f,
                          double* score) {
  // ---- decode the space point (mixed radix, axis 0 most significant): tile factors into the
  //      record's parameter slots (or, static tiles, both extents straight from the choice), the
  //      reorder choice, the group-table row offsets
  const bool stat = T.sp_static;
  if (stat)  // base loops no tile splits (the tiles write both extents of theirs)
    for (int q = 0; q < T.sp_n_untiled; ++q) c.E(T.sp_untiled[q]) = T.base_ext[T.sp_untiled_pos[q]];
  uint32_t kd[TM * 2];
#pragma unroll
  for (int g = 0; g < TM * 2; ++g) kd[g] = T.sd_off[g];
  uint64_t lo = 0, hi = 0;
  uint32_t pch = 0;
  for (int a = T.sp_n - 1; a >= 0; --a) {
    const DAxis& ax = T.sp_ax[a];
    uint32_t ch;
    if (a == 0) {
      if (x >= ax.n) return LS_ST_POINT_RANGE;
      ch = (uint32_t)x;
    } else if (ax.n == 1) {
      ch = 0;
    } else if (x >> 32) {
      const uint64_t q = x / ax.n;
      ch = (uint32_t)(x - q * ax.n);
      x = q;
    } else {  // umulhi(x, magic) for x < 2^32: x * magic_hi + umulhi(x, magic_lo), top word
      const uint32_t x32 = (uint32_t)x;
      const uint32_t q = (uint32_t)(((uint64_t)x32 * (uint32_t)(ax.magic >> 32) + __umulhi(x32, (uint32_t)ax.magic)) >> 32);
      ch = x32 - q * (uint32_t)ax.n;
      x = q;
    }
    if (ax.kind == LS_AX_PERM) {
      pch = ch;
      continue;
    }
#pragma unroll
    for (int g = 0; g < TM * 2; ++g) kd[g] += ch * T.sd_S[a][g];
    if (stat) {  // Tile (ls/ir.py:361-382) of a base loop: F and ceil(E/F) per choice
      const uint64_t e = __ldg(reinterpret_cast<const unsigned long long*>(T.sp_ext) + ax.voff + ch);
      if (e >> 63) return LS_ST_TILE_RANGE;
      c.E(T.sp_tnew[a]) = (int32_t)(e & 0xFFFFu);
      c.E(T.sp_tslot[a]) = (int32_t)((e >> 16) & 0x7FFFFFFFu);
      continue;
    }
    const uint64_t v = __ldg(reinterpret_cast<const unsigned long long*>(T.sp_vals) + ax.voff + ch);
    if (ax.param < 4)
      lo |= v << (16 * ax.param);
    else
      hi |= v << (16 * (ax.param - 4));
  }
  if (!stat) {
    ls_record r;
    memcpy(&r.param[0], &lo, 8);
    memcpy(&r.param[4], &hi, 8);
    // ---- extents: Tile arithmetic in template order (ls/ir.py:361-382), with the
    //      checks of apply_fast that a tile factor can fail
    for (int p = 0; p < T.n_base; ++p) c.E(T.base_slot[p]) = T.base_ext[p];
    for (int q = 0; q < T.n_xf; ++q) {
      const DXform& xf = T.xf[q];
      if (xf.kind != LS_XF_TILE) continue;
      const int32_t F = xf.param >= 0 ? (int32_t)rparam(r, xf.param) : xf.value;
      const int32_t Ev = c.E(xf.slot);
      if (F < 1 || F > Ev) return LS_ST_TILE_RANGE;
      c.E(xf.new_slot) = F;
      c.E(xf.slot) = (Ev + F - 1) / F;
    }
  }
  const int pst = __ldg(T.sp_pstat + pch);
  if (pst) return pst;
  const uint64_t chain = __ldg(reinterpret_cast<const unsigned long long*>(T.sp_chain) + pch);
  const int n = T.sp_nchain;
  // ---- movement walk (ls/cache.py:167-236, chain form): a tensor footprint is
  //      the product of its dimension counts (ls/cache.py:117-130) = the product
  //      of its two group entries, shared-memory lookups at (row of this
  //      candidate, stage mask so far)
  const char* tb = reinterpret_cast<const char*>(sdt);
  uint64_t mall = 0;
  auto grp = [&](int g) -> uint32_t {
    return *reinterpret_cast<const uint32_t*>(tb + kd[g] + ((uint32_t)(mall >> (8 * g)) & 0xFFu));
  };
  // NARROW: the host proved every footprint, their sum and every movement fit 32 bits
  using W = typename std::conditional<NARROW, uint32_t, int64_t>::type;
  auto fp = [&](int t) -> W {
    if constexpr (NARROW)
      return grp(2 * t) * grp(2 * t + 1);
    else
      return (int64_t)((uint64_t)grp(2 * t) * grp(2 * t + 1));
  };
  uint32_t vm[TM];
  W Fb[TM], dm[TM];
  bool ru[TM];
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    vm[t] = T.t_vmask[t];
    Fb[t] = fp(t);
    dm[t] = (W)T.t_nacc[t];
    ru[t] = true;
  }
  const W cap = (W)T.cap;
  const bool cpu = T.family == LS_FAMILY_CPU;
  const int wrap = cpu ? -1 : n - 9;  // PTX: no trip for loops 8+ levels above the innermost
  W P = 1, H = 0;  // product of all extents; Horner sum of the outer prefix products (NARROW: < 2^32 proven)
  for (int p = n - 1; p >= 0; --p) {
    const int v = (int)((chain >> (4 * p)) & 15u);
    const int32_t E = c.E(v);
    mall |= T.vb8[v];
    W single = 0;
#pragma unroll
    for (int t = 0; t < TM; ++t) single += Fb[t];
    const bool over = single > cap;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const bool uses = (vm[t] >> v) & 1u;
      const W Ff = fp(t);
      const bool r0 = ru[t] && !(over && !uses);
      if constexpr (NARROW)
        dm[t] = (!over || r0) ? Ff : dm[t] * (uint32_t)E;
      else
        dm[t] = (!over || r0) ? Ff : (int64_t)((uint64_t)dm[t] * (uint32_t)E);
      ru[t] = r0 && !(Ff > cap);
      Fb[t] = Ff;
    }
    const W Ee = p > wrap ? (W)E : (W)1;
    if (p < n - 1) H = Ee * (1 + H);
    P *= Ee;
  }
  int64_t dmov = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) dmov += (int64_t)dm[t];
  const int64_t L = T.L, S = T.S;
  double total = 0.0;
  if (cpu) {
    const int64_t ilp = T.c_init * (1 + H) + T.c_inner1 * P + T.c_latch * (n - 1) + T.c_ret;
    f[0] = (double)(S * P);
    f[1] = (double)(L * P);
    f[2] = (double)(S * P);
    f[3] = (double)dmov;
    f[4] = (double)ilp;
#pragma unroll
    for (int q = 0; q < LS_NFEAT_CPU; ++q) {
      if (!(f[q] >= 0.0) || isinf(f[q])) return LS_ST_BAD_FEATURE;
      total = rn_add(total, rn_mul(T.coef[q], f[q]));
    }
  } else {
    const int64_t* ic = T.ptx_icost;
    const int64_t loops = ic[LS_I_INIT] * (1 + H) + (ic[LS_I_ADD] + ic[LS_I_CMP] + ic[LS_I_BRANCH]) * (H + P);
    f[0] = (double)(loops + P * (L * ic[LS_I_LOAD] + S * (ic[LS_I_FMA] + ic[LS_I_STORE])) + ic[LS_I_RET]);
    f[1] = T.sm_underuse;
    f[2] = T.warp_slack;
    f[3] = 0.0;
    f[4] = (double)(S * P);
    f[5] = (double)(L * P);
    f[6] = (double)(S * P);
#pragma unroll
    for (int q = 0; q < LS_NFEAT_GPU; ++q) {
      if (!(f[q] >= 0.0) || isinf(f[q])) return LS_ST_BAD_FEATURE;
      total = rn_add(total, rn_mul(T.coef[q], f[q]));
    }
  }
  *score = total;
  return LS_OK;
}

// One group-table entry per thread: decode (group slot, tile-axis choices, stage
// mask); the entry is the product of the group's dimension counts (same fold as
// build_tab_kernel).  Products that do not fit 32 bits raise *overflow.
__global__ void build_sdt_kernel(const DTask* __restrict__ g, const int32_t* __restrict__ rows,
                                 uint32_t* __restrict__ tab, int32_t* __restrict__ overflow,
                                 unsigned int* __restrict__ gmax) {
  const DTask& T = *g;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T.sd_len) return;
  if (e < 4) {  // the ones row (group slots without dimensions)
    tab[e] = 1;
    return;
  }
  int G = -1;
  for (int q = 0; q < 8; ++q)
    if (rows[q] && e >= (int)T.sd_off[q] / 4 && e < (int)T.sd_off[q] / 4 + (rows[q] << T.sd_nb[q])) G = q;
  if (G < 0) return;
  const int loc = e - (int)T.sd_off[G] / 4;
  const uint32_t mask = (uint32_t)loc & ((1u << T.sd_nb[G]) - 1u);
  const uint32_t key = (uint32_t)loc >> T.sd_nb[G];
  int32_t prm[LS_MAX_PARAMS];
  for (int q = 0; q < LS_MAX_PARAMS; ++q) prm[q] = 1;
  for (int a = 0; a < T.sp_n; ++a) {
    const uint32_t stride = T.sd_S[a][G] >> (2 + T.sd_nb[G]);
    if (!stride) continue;
    const DAxis& ax = T.sp_ax[a];
    const uint32_t ch = (key / stride) % ax.n;
    prm[ax.param] = (int32_t)T.sp_vals[ax.voff + ch];
  }
  int32_t E[NSLOT], St[NSLOT];
  uint32_t exist;
  sim_slots(T, prm, 0u, E, St, exist);
  uint64_t F = 1;
  for (int j = 0; j < 4; ++j) {
    const int D = T.sd_gd[G][j];
    if (D < 0) continue;
    const uint32_t m = (mask >> T.sd_gx[G][j]) & ((1u << T.dim_nv[D]) - 1u);
    F *= (uint64_t)(uint32_t)dim_count(T, D, m, 0u, E, St, exist);
  }
  if (F > 0xFFFFFFFFull) {
    atomicExch(overflow, 1);
    F = 0;
  }
  atomicMax(&gmax[G], (unsigned int)F);
  tab[e] = (uint32_t)F;
}

// ---------------------------------------------------------------------------
// General trees: imperfect nests, sibling loops, accesses at
// any level; Tile / Reorder / Parallel transforms (Unroll / Vectorize and
// unrolled or vector base loops stay outside the device class).  One thread
// per candidate; the transformed tree lives in the thread's local memory.
// ---------------------------------------------------------------------------
constexpr int TR_N = 32;  // unified node ids: accesses, then loops (<= 16 each)

struct TreeCand {
  int8_t par[TR_N], first[TR_N], nxt[TR_N];
  int8_t ord[TR_N];                 // preorder of all nodes
  uint8_t pre[TR_N], pend[TR_N];    // preorder position, end of the subtree
  uint8_t dep[TR_N];
  uint8_t hs[NSLOT], hf[NSLOT];     // per loop j (node tr_na + j): var slot, flags
  int32_t he[NSLOT], hst[NSLOT];    //   extent, step
  int8_t grp[NSLOT];                //   access group (base loop id) hanging under it, -1 none
  int8_t nos[NSLOT];                // loop j of each var slot, -1 none
  int nl, nn, root;
};

// apply_schedule on the tree (ls/ir.py:361-474), same checks in the same order
__device__ int tree_apply(const DTask& T, const ls_record& r, TreeCand& c) {
  const int na = T.tr_na;
  c.nl = T.tr_nl;
  c.root = T.tr_root_first;
  for (int i = 0; i < na + c.nl; ++i) {
    c.par[i] = T.tr_parent[i];
    c.first[i] = T.tr_first[i];
    c.nxt[i] = T.tr_next[i];
  }
  for (int v = 0; v < NSLOT; ++v) c.nos[v] = -1;
  for (int j = 0; j < c.nl; ++j) {
    c.hs[j] = T.base_slot[j];
    c.he[j] = T.base_ext[j];
    c.hst[j] = T.base_step[j];
    c.hf[j] = T.base_flags[j];
    c.grp[j] = (int8_t)j;
    c.nos[T.base_slot[j]] = (int8_t)j;
  }
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.enable_bit >= 0 && !((r.flags >> xf.enable_bit) & 1u)) continue;
    const int j = xf.slot != NOSLOT ? c.nos[xf.slot] : -1;
    if (xf.kind == LS_XF_TILE || xf.kind == LS_XF_VECTORIZE) {
      if (j < 0 || xf.new_slot == NOSLOT) return LS_ST_NO_LOOP;
      const int32_t F = xf.param >= 0 ? (int32_t)rparam(r, xf.param) : xf.value;
      const int32_t E = c.he[j];
      if (xf.kind == LS_XF_VECTORIZE) {  // extent % width (ls/ir.py:463-468)
        if (F == 0) return LS_ST_VEC_ZERO;
        if (E % F != 0) return LS_ST_VEC_DIVIDE;
      }
      if (F < 1 || F > E) return LS_ST_TILE_RANGE;
      if (c.nl >= NSLOT) return LS_ST_OVERFLOW;
      const int u = c.nl++;
      const int nj = na + j, nu = na + u;
      c.hs[u] = xf.new_slot;
      c.he[u] = F;
      c.hst[u] = c.hst[j];
      c.hf[u] = xf.kind == LS_XF_VECTORIZE ? F_VEC : 0;
      c.hf[j] &= (uint8_t)~F_VEC;  // the outer loop keeps parallel / unrolled only (ls/ir.py:379-380)
      c.grp[u] = c.grp[j];
      c.grp[j] = -1;
      c.nos[xf.new_slot] = (int8_t)u;
      c.he[j] = (E + F - 1) / F;
      c.hst[j] *= F;
      c.first[nu] = c.first[nj];  // the inner loop takes the children (ls/ir.py:369-381)
      for (int ch = c.first[nu]; ch >= 0; ch = c.nxt[ch]) c.par[ch] = (int8_t)nu;
      c.first[nj] = (int8_t)nu;
      c.nxt[nu] = -1;
      c.par[nu] = (int8_t)nj;
    } else if (xf.kind == LS_XF_REORDER) {
      const int m = xf.n_order;
      if (m < 2) continue;
      int8_t ids[LS_MAX_ORDER];
      for (int q = 0; q < m; ++q) {  // find_loop of every name first (ls/ir.py:388)
        const int nib = (int)((r.perm >> (4 * (xf.perm_shift + q))) & 0xF);
        const int w = nib < m ? xf.order[nib] : NOSLOT;
        if (w == NOSLOT || c.nos[w] < 0) return LS_ST_NO_LOOP;
        ids[q] = c.nos[w];
      }
      uint32_t seen = 0;
      for (int q = 0; q < m; ++q) {
        if ((seen >> ids[q]) & 1u) return LS_ST_REORDER_MISSING;
        seen |= 1u << ids[q];
      }
      // the shallowest named loop, then down through only children (chain_ok, ls/ir.py:392-402)
      int top = -1, topd = 1 << 20;
      for (int q = 0; q < m; ++q) {
        int d = 0;
        for (int a = c.par[na + ids[q]]; a >= 0; a = c.par[a]) ++d;
        if (d < topd) topd = d, top = ids[q];
      }
      int8_t seq[LS_MAX_ORDER];
      seq[0] = (int8_t)top;
      for (int q = 1; q < m; ++q) {
        const int cur = na + seq[q - 1];
        const int ch = c.first[cur];
        if (ch < 0 || c.nxt[ch] >= 0 || ch < na || !((seen >> (ch - na)) & 1u)) return LS_ST_REORDER_CHAIN;
        seq[q] = (int8_t)(ch - na);
      }
      uint8_t hs[LS_MAX_ORDER], hf[LS_MAX_ORDER];
      int32_t he[LS_MAX_ORDER], hst[LS_MAX_ORDER];
      for (int q = 0; q < m; ++q) hs[q] = c.hs[ids[q]], hf[q] = c.hf[ids[q]], he[q] = c.he[ids[q]], hst[q] = c.hst[ids[q]];
      for (int q = 0; q < m; ++q) {  // position q of the chain takes the header of order[q] (ls/ir.py:406-412)
        const int j2 = seq[q];
        c.hs[j2] = hs[q], c.hf[j2] = hf[q], c.he[j2] = he[q], c.hst[j2] = hst[q];
        c.nos[hs[q]] = (int8_t)j2;
      }
    } else if (xf.kind == LS_XF_PARALLEL || xf.kind == LS_XF_UNROLL) {
      if (j < 0) return LS_ST_NO_LOOP;
      c.hf[j] |= xf.kind == LS_XF_PARALLEL ? F_PAR : F_UNR;
    } else {
      return LS_ST_UNSUPPORTED;
    }
  }
  // preorder numbering, depths, subtree ends
  c.nn = na + c.nl;
  int idx = 0, n = c.root, d = 0;
  while (n >= 0) {
    c.pre[n] = (uint8_t)idx;
    c.ord[idx++] = (int8_t)n;
    c.dep[n] = (uint8_t)d;
    if (n >= na && c.first[n] >= 0) {
      n = c.first[n];
      ++d;
      continue;
    }
    while (n >= 0) {
      c.pend[n] = (uint8_t)idx;
      if (c.nxt[n] >= 0) {
        n = c.nxt[n];
        break;
      }
      n = c.par[n];
      --d;
    }
  }
  return LS_OK;
}

// expr_range (ls/cache.py:80-96) with the loops of `L`'s subtree expanded (and L itself when full)
__device__ __forceinline__ SI tree_expr_range(const DTask& T, const DExpr& e, const TreeCand& c, uint32_t flags,
                                              int L, bool full) {
  SI acc;
  acc.lo = acc.hi = e.konst;
  acc.stride = 0;
  acc.count = 1;
  acc.exact = 1;
  const int na = T.tr_na;
  for (int k = 0; k < e.nt; ++k) {
    const DTerm& tm = T.term[e.t0 + k];
    if (!present(tm, flags)) continue;
    const int j = c.nos[tm.slot];
    if (j < 0) continue;
    const int nd = na + j;
    const bool in = (c.pre[nd] > c.pre[L] && c.pre[nd] < c.pend[L]) || (full && nd == L);
    if (!in) continue;
    const int32_t E = c.he[j];
    if (E == 1) continue;
    const int32_t dd = tm.coef * c.hst[j];
    SI s;
    s.lo = dd > 0 ? 0 : dd * (E - 1);
    s.hi = dd > 0 ? dd * (E - 1) : 0;
    s.stride = abs(dd);
    s.count = E;
    s.exact = 1;
    acc = si_sum(acc, s);
  }
  return acc;
}

// tensor_footprint (ls/cache.py:117-130): the union of the accesses of tensor t
// under loop node L in DFS order, product over dimensions
__device__ int64_t tree_footprint(const DTask& T, const TreeCand& c, uint32_t flags, int L, int t, bool full) {
  int64_t card = 1;
  for (int rr = 0; rr < T.t_rank[t]; ++rr) {
    SI u;
    bool any = false;
    for (int q = c.pre[L] + 1; q < c.pend[L]; ++q) {
      const int a = c.ord[q];
      if (a >= T.tr_na || T.acc_tensor[a] != t) continue;
      const SI x = tree_expr_range(T, T.expr[a][rr], c, flags, L, full);
      u = any ? si_union(u, x) : x;
      any = true;
    }
    card *= u.count;
  }
  return card;
}

// ---- emulated emission for trees with inlined (unrolled / vector) loops -------
// The mock emitter (ls/ir.py:557-659) inlines an unrolled loop `extent` times
// and a vector loop once, at the same depth; blocks split at labels and after
// branches (ls/asm.py:155-167).  The CPU features need the greedy loop_map over
// the emitted label blocks (ls/asm.py:250-294, copies of loops inside unrolled
// loops included) and schedule_block of every block (ls/ilp.py:131-204), so the
// emission is replayed block by block and each block is list-scheduled here.

// register / resource ids of the emitted text: vector regs 0..23, base regs
// 24 + decl % 6, their memory resources 30 + decl % 6, counters 36 + depth % 8,
// the PTX predicate 44
struct EInstr {
  uint8_t shape, nrd, nwr, pad;
  int8_t rd[6], wr[2];
};

constexpr int EM_MAXI = 128;   // instructions per block (more: LS_ST_UNSUPPORTED)
constexpr int EM_MAXE = 1024;  // dependence edges per block (more: LS_ST_UNSUPPORTED)

// reg_effects (ls/ilp.py:82-121) of one emitted instruction: operands as
// (kind, id) with kind 0 register, 1 memory operand (base register id), 2 immediate
__device__ void em_effects(int dialect, int shape, bool st_like, bool rmw, bool is_cmp, bool is_branch, bool mov_like,
                           int nops, const int8_t* okind, const int8_t* oid, int pred, EInstr& o) {
  o.shape = (uint8_t)shape;
  o.nrd = o.nwr = 0;
  if (pred >= 0) o.rd[o.nrd++] = (int8_t)pred;
  if (nops == 0 || is_branch) return;
  int mem = -1;
  for (int i = 0; i < nops; ++i)
    if (okind[i] == 1) {
      mem = i;
      break;
    }
  const bool store = st_like || (mem >= 0 && mem == nops - 1 && mov_like);
  const int dest = dialect == LS_DIALECT_X86_ATT ? nops - 1 : ((st_like && mem >= 0) ? mem : 0);
  for (int i = 0; i < nops; ++i) {
    if (okind[i] == 2) continue;
    if (i == mem) {
      o.rd[o.nrd++] = oid[i];  // the base register
      const int8_t res = (int8_t)(oid[i] + 6);
      if (i == dest && store)
        o.wr[o.nwr++] = res;
      else
        o.rd[o.nrd++] = res;
      continue;
    }
    if (i == dest && !is_cmp) {
      o.wr[o.nwr++] = oid[i];
      if (rmw) o.rd[o.nrd++] = oid[i];
    } else {
      o.rd[o.nrd++] = oid[i];
    }
  }
}

struct Emu {
  const DTask* T;
  const TreeCand* c;
  EInstr blk[EM_MAXI];
  int n;              // instructions in the open block
  int label;          // the open block starts at a label: loop node id (else -1)
  int nld, nst, nfma; // significant instructions in the open block
  int vreg;
  int cursor;         // loop_map cursor into the preorder non-inlined loops
  int nfor;
  int8_t forl[NSLOT];         // preorder non-inlined loops (loop index)
  int64_t trip[NSLOT];        // enclosing trip product of each of them
  int64_t ilp, n_ld, n_st, n_fma;
  int err;
};

__device__ void em_push(Emu& e, int shape, bool st_like, bool rmw, bool is_cmp, bool is_branch, bool mov_like, int nops,
                        const int8_t* ok, const int8_t* oi, int pred = -1) {
  if (e.n >= EM_MAXI) {
    e.err = LS_ST_UNSUPPORTED;
    return;
  }
  em_effects(e.T->tr_dialect, shape, st_like, rmw, is_cmp, is_branch, mov_like, nops, ok, oi, pred, e.blk[e.n++]);
}

// schedule_block (ls/ilp.py:131-204): RAW edges with latencies, WAR / WAW order edges, greedy issue
__device__ int64_t em_schedule(const Emu& e, int& err) {
  const DTask& T = *e.T;
  const int n = e.n;
  int16_t last_w[48];
  int16_t rhead[48];
  int16_t rnext[EM_MAXI * 6];
  int16_t rnode[EM_MAXI * 6];
  int nr = 0;
  for (int q = 0; q < 48; ++q) last_w[q] = rhead[q] = -1;
  int16_t eoff[EM_MAXI + 1], raw_end[EM_MAXI];
  int16_t edge[EM_MAXE];
  int ne = 0;
  for (int k = 0; k < n; ++k) {
    const EInstr& in = e.blk[k];
    eoff[k] = (int16_t)ne;
    for (int q = 0; q < in.nrd; ++q) {  // RAW: last writer of each read resource
      const int w = last_w[in.rd[q]];
      if (w < 0) continue;
      bool dup = false;
      for (int z = eoff[k]; z < ne; ++z) dup |= edge[z] == w;
      if (!dup) {
        if (ne >= EM_MAXE) {
          err = LS_ST_UNSUPPORTED;
          return 0;
        }
        edge[ne++] = (int16_t)w;
      }
    }
    raw_end[k] = (int16_t)ne;
    for (int q = 0; q < in.nwr; ++q) {  // WAW + WAR, minus the RAW predecessors
      const int res = in.wr[q];
      for (int z = -1; z < 0 || z >= 0;) {
        int pred;
        if (z == -1) {  // the last writer first, then the readers since it
          pred = last_w[res];
          z = rhead[res] >= 0 ? rhead[res] : -2;
        } else {
          pred = rnode[z] != k ? rnode[z] : -1;
          z = rnext[z] >= 0 ? rnext[z] : -2;
        }
        if (pred >= 0) {
          bool dup = false;
          for (int y = eoff[k]; y < ne; ++y) dup |= edge[y] == pred;
          if (!dup) {
            if (ne >= EM_MAXE) {
              err = LS_ST_UNSUPPORTED;
              return 0;
            }
            edge[ne++] = (int16_t)pred;
          }
        }
        if (z == -2) break;
      }
    }
    for (int q = 0; q < in.nwr; ++q) {
      last_w[in.wr[q]] = (int16_t)k;
      rhead[in.wr[q]] = -1;
    }
    for (int q = 0; q < in.nrd; ++q) {
      rnode[nr] = (int16_t)k;
      rnext[nr] = rhead[in.rd[q]];
      rhead[in.rd[q]] = (int16_t)nr;
      ++nr;
    }
  }
  eoff[n] = (int16_t)ne;
  int64_t issue[EM_MAXI];
  for (int k = 0; k < n; ++k) issue[k] = -1;
  int done = 0, first = 0;
  int64_t cycle = 0;
  while (done < n) {
    int issued = 0;
    int used[LS_I_COUNT] = {0};
    while (first < n && issue[first] >= 0) ++first;
    for (int i = first; i < n && issued < T.tr_issue; ++i) {
      if (issue[i] >= 0) continue;
      int64_t ready = 0;
      bool ok = true;
      for (int z = eoff[i]; z < eoff[i + 1] && ok; ++z) {
        const int p = edge[z];
        if (issue[p] < 0)
          ok = false;
        else
          ready = max(ready, issue[p] + (z < raw_end[i] ? (int64_t)T.tr_lat[e.blk[p].shape] : 1));
      }
      if (!ok || ready > cycle) continue;
      const int cls = T.tr_klass[e.blk[i].shape];
      const int cap = T.tr_ucap[cls];
      if (cap > 0 && used[cls] >= cap) continue;
      issue[i] = cycle;
      ++used[cls];
      ++issued;
      ++done;
    }
    ++cycle;
  }
  int64_t fin = 0;
  for (int k = 0; k < n; ++k) fin = max(fin, issue[k] + (int64_t)T.tr_lat[e.blk[k].shape]);
  return fin;
}

__device__ void em_end_block(Emu& e) {
  if (e.n == 0 || e.err) {
    e.n = 0;
    e.label = -1;
    return;
  }
  int64_t w = 1;
  if (e.label >= 0 && e.cursor < e.nfor) {  // greedy in-order loop_map (ls/asm.py:270-292)
    const int lp = e.forl[e.cursor];
    const int64_t bound = e.c->he[e.label - e.T->tr_na];
    if (bound == e.c->he[lp] || bound == (int64_t)e.c->he[lp] * e.c->hst[lp]) {
      w = e.trip[e.cursor];
      e.n_ld += (int64_t)e.nld * w;
      e.n_st += (int64_t)e.nst * w;
      e.n_fma += (int64_t)e.nfma * w;
      ++e.cursor;
    }
  }
  int err = 0;
  const int64_t cyc = em_schedule(e, err);
  if (err) e.err = err;
  e.ilp += cyc * w;
  e.n = 0;
  e.label = -1;
  e.nld = e.nst = e.nfma = 0;
}

// emit_body (ls/ir.py:584-612): loads, then fma + store per store
__device__ void em_body(Emu& e, int node) {
  const DTask& T = *e.T;
  const TreeCand& c = *e.c;
  const int tg = T.tr_target;
  int8_t lregs[MAXACC];
  int L = 0;
  for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch]) {
    if (ch >= T.tr_na || T.acc_store[ch]) continue;
    const int r = e.vreg++ % 16;
    lregs[L++] = (int8_t)r;
    const int8_t base = (int8_t)(24 + T.acc_decl[ch] % 6);
    if (tg == LS_TARGET_X86) {  // vmovups (B), %zmmR
      const int8_t ok[2] = {1, 0}, oi[2] = {base, (int8_t)r};
      em_push(e, LS_I_LOAD, false, false, false, false, true, 2, ok, oi);
    } else {  // ld1 {vR}, [B]  /  ld.global.f32 %fR, [B]
      const int8_t ok[2] = {0, 1}, oi[2] = {(int8_t)r, base};
      em_push(e, LS_I_LOAD, false, false, false, false, false, 2, ok, oi);
    }
    ++e.nld;
  }
  int j = 0;
  for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch]) {
    if (ch >= T.tr_na || !T.acc_store[ch]) continue;
    const int8_t acc = (int8_t)(16 + j % 8);
    const int8_t s1 = L ? lregs[(2 * j) % L] : 0, s2 = L ? lregs[(2 * j + 1) % L] : 1;
    const int8_t base = (int8_t)(24 + T.acc_decl[ch] % 6);
    if (tg == LS_TARGET_X86) {
      const int8_t ok[3] = {0, 0, 0}, oi[3] = {s1, s2, acc};  // vfmadd231ps S1, S2, A
      em_push(e, LS_I_FMA, false, true, false, false, false, 3, ok, oi);
      const int8_t sk[2] = {0, 1}, si[2] = {acc, base};        // vmovups A, (B)
      em_push(e, LS_I_STORE, false, false, false, false, true, 2, sk, si);
    } else if (tg == LS_TARGET_AARCH64) {
      const int8_t ok[3] = {0, 0, 0}, oi[3] = {acc, s1, s2};  // fmla A, S1, S2
      em_push(e, LS_I_FMA, false, true, false, false, false, 3, ok, oi);
      const int8_t sk[2] = {0, 1}, si[2] = {acc, base};        // st1 {A}, [B]
      em_push(e, LS_I_STORE, true, false, false, false, false, 2, sk, si);
    } else {
      const int8_t ok[4] = {0, 0, 0, 0}, oi[4] = {acc, s1, s2, acc};  // fma.rn.f32 A, S1, S2, A
      em_push(e, LS_I_FMA, false, true, false, false, false, 4, ok, oi);
      const int8_t sk[2] = {1, 0}, si[2] = {base, acc};                // st.global.f32 [B], A
      em_push(e, LS_I_STORE, true, false, false, false, false, 2, sk, si);
    }
    ++e.nfma;
    ++e.nst;
    ++j;
  }
}

__device__ void em_node(Emu& e, int node, int depth) {
  if (e.err) return;
  const DTask& T = *e.T;
  const TreeCand& c = *e.c;
  const int j = node - T.tr_na;
  const uint8_t fl = c.hf[j];
  const int tg = T.tr_target;
  if (fl & (F_UNR | F_VEC)) {  // inlined: extent copies (vector: one) at the same depth
    const int copies = (fl & F_VEC) ? 1 : c.he[j];
    for (int q = 0; q < copies && !e.err; ++q) {
      em_body(e, node);
      for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch])
        if (ch >= T.tr_na) em_node(e, ch, depth);
    }
    return;
  }
  const int8_t ctr = (int8_t)(36 + depth % 8);
  {  // counter init in the open block
    const int8_t ok[2] = {2, 0}, oi[2] = {0, ctr}, dk[2] = {0, 2}, di[2] = {ctr, 0};
    if (tg == LS_TARGET_X86)
      em_push(e, LS_I_INIT, false, false, false, false, true, 2, ok, oi);  // movq $0, C
    else
      em_push(e, LS_I_INIT, false, false, false, false, true, 2, dk, di);  // mov C, #0 / mov.u32 C, 0
  }
  em_end_block(e);  // the label starts a block
  e.label = node;
  em_body(e, node);
  for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch])
    if (ch >= T.tr_na) em_node(e, ch, depth + 1);
  if (tg == LS_TARGET_X86) {
    const int8_t ak[2] = {2, 0}, ai[2] = {0, ctr};
    em_push(e, LS_I_ADD, false, true, false, false, false, 2, ak, ai);    // addq $1, C
    em_push(e, LS_I_CMP, false, false, true, false, false, 2, ak, ai);    // cmpq $E, C
    em_push(e, LS_I_BRANCH, false, false, false, true, false, 1, ak, ai); // jne
  } else if (tg == LS_TARGET_AARCH64) {
    const int8_t ak[3] = {0, 0, 2}, ai[3] = {ctr, ctr, 0}, ck[2] = {0, 2}, ci[2] = {ctr, 0};
    em_push(e, LS_I_ADD, false, true, false, false, false, 3, ak, ai);    // add C, C, #1
    em_push(e, LS_I_CMP, false, false, true, false, false, 2, ck, ci);    // cmp C, #E
    em_push(e, LS_I_BRANCH, false, false, false, true, false, 1, ck, ci); // b.ne
  } else {
    const int8_t ak[3] = {0, 0, 2}, ai[3] = {ctr, ctr, 0}, sk[3] = {0, 0, 2}, si[3] = {44, ctr, 0};
    em_push(e, LS_I_ADD, false, true, false, false, false, 3, ak, ai);    // add.s32 C, C, 1
    em_push(e, LS_I_CMP, false, false, false, false, false, 3, sk, si);   // setp.lt.s32 P, C, E
    em_push(e, LS_I_BRANCH, false, false, false, true, false, 1, sk, si, 44);  // @P bra
  }
  em_end_block(e);  // a branch ends the block
}

// CPU features of a tree with inlined loops: n_fma, n_vload, n_vstore (count_simd over the
// matched label blocks) and ilp (every block scheduled, times its matched trip product)
__device__ int em_cpu_features(const DTask& T, const TreeCand& c, int64_t& nfma, int64_t& nld, int64_t& nst,
                               int64_t& ilp) {
  Emu e;
  e.T = &T;
  e.c = &c;
  e.n = 0;
  e.label = -1;
  e.nld = e.nst = e.nfma = 0;
  e.vreg = 0;
  e.cursor = 0;
  e.nfor = 0;
  e.ilp = e.n_ld = e.n_st = e.n_fma = 0;
  e.err = 0;
  // preorder non-inlined loops and their trip products over non-inlined ancestors (ls/asm.py:261-272)
  int64_t tp[NSLOT];
  for (int q = 0; q < c.nn; ++q) {
    const int L = c.ord[q];
    if (L < T.tr_na) continue;
    const int j = L - T.tr_na, p = c.par[L];
    const int64_t up = p >= 0 ? tp[p - T.tr_na] : 1;
    const bool inl = c.hf[j] & (F_UNR | F_VEC);
    tp[j] = inl ? up : up * c.he[j];
    if (!inl) {
      e.forl[e.nfor] = (int8_t)j;
      e.trip[e.nfor++] = tp[j];
    }
  }
  for (int n = c.root; n >= 0; n = c.nxt[n])
    if (n >= T.tr_na) em_node(e, n, 0);
  {
    const int8_t ok[1] = {2}, oi[1] = {0};
    em_push(e, LS_I_RET, false, false, false, true, false, 0, ok, oi);  // ret
  }
  em_end_block(e);
  if (e.err) return e.err;
  nfma = e.n_fma;
  nld = e.n_ld;
  nst = e.n_st;
  ilp = e.ilp;
  return LS_OK;
}

// thread_cycles in emission line order (ls/ptx.py:225-235) for a tree: inlined loops
// replay their body `copies` times at the same depth; a branching loop's init line
// weighs W' of its parent, its body and latch lines its own W'
__device__ double tree_ptx_node(const DTask& T, const TreeCand& c, const int64_t* Wp, int node, double work) {
  const double* pc = T.ptx_cost;
  const int na = T.tr_na, j = node - na, p = c.par[node];
  const uint8_t fl = c.hf[j];
  auto body = [&](double w) {
    const int g = c.grp[j];
    if (g < 0) return;
    for (int a = 0; a < T.tr_nld[g]; ++a) work = rn_add(work, rn_mul(pc[LS_I_LOAD], w));
    for (int a = 0; a < T.tr_nst[g]; ++a) {
      work = rn_add(work, rn_mul(pc[LS_I_FMA], w));
      work = rn_add(work, rn_mul(pc[LS_I_STORE], w));
    }
  };
  if (fl & (F_UNR | F_VEC)) {
    const int copies = (fl & F_VEC) ? 1 : c.he[j];
    for (int q = 0; q < copies; ++q) {
      body((double)Wp[j]);
      for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch])
        if (ch >= na) work = tree_ptx_node(T, c, Wp, ch, work);
    }
    return work;
  }
  work = rn_add(work, rn_mul(pc[LS_I_INIT], (double)(p >= 0 ? Wp[p - na] : 1)));
  body((double)Wp[j]);
  for (int ch = c.first[node]; ch >= 0; ch = c.nxt[ch])
    if (ch >= na) work = tree_ptx_node(T, c, Wp, ch, work);
  const double w = (double)Wp[j];
  work = rn_add(work, rn_mul(pc[LS_I_ADD], w));
  work = rn_add(work, rn_mul(pc[LS_I_CMP], w));
  work = rn_add(work, rn_mul(pc[LS_I_BRANCH], w));
  return work;
}

__device__ double tree_ptx_ordered(const DTask& T, const TreeCand& c, const int64_t* Wp) {
  double work = 0.0;
  for (int n = c.root; n >= 0; n = c.nxt[n])
    if (n >= T.tr_na) work = tree_ptx_node(T, c, Wp, n, work);
  return rn_add(work, T.ptx_cost[LS_I_RET]);
}

__device__ int eval_tree(const DTask& T, const ls_record& r, double* f, double* score) {
  TreeCand c;
  const int st = tree_apply(T, r, c);
  if (st) return st;
  const int na = T.tr_na, nT = T.n_tensors;
  const uint32_t flags = r.flags;
  const int64_t cap = T.cap;
  // ---- movement model (ls/cache.py:133-236), loops in reverse preorder (children first)
  int64_t dm[NSLOT][MAXT];
  uint8_t rb[NSLOT], pres[NSLOT];
  for (int q = c.nn - 1; q >= 0; --q) {
    const int L = c.ord[q];
    if (L < na) continue;
    const int j = L - na;
    int64_t m_dm[MAXT];
    uint32_t m_pres = 0, m_reuse = 0xFFu;
    for (int t = 0; t < nT; ++t) m_dm[t] = 0;
    for (int ch = c.first[L]; ch >= 0; ch = c.nxt[ch]) {
      if (ch < na) {
        const int t = T.acc_tensor[ch];
        m_pres |= 1u << t;
        m_dm[t] += 1;
      } else {
        const int k = ch - na;
        for (int t = 0; t < nT; ++t)
          if ((pres[k] >> t) & 1u) {
            m_pres |= 1u << t;
            m_dm[t] += dm[k][t];
            if (!((rb[k] >> t) & 1u)) m_reuse &= ~(1u << t);
          }
      }
    }
    int64_t single = 0, ffull[MAXT];
    uint32_t uses = 0;
    for (int t = 0; t < nT; ++t) {
      if (!((m_pres >> t) & 1u)) continue;
      single += tree_footprint(T, c, flags, L, t, false);
      ffull[t] = tree_footprint(T, c, flags, L, t, true);
      for (int q2 = c.pre[L] + 1; q2 < c.pend[L]; ++q2) {  // any access of t indexed by this loop's variable
        const int a = c.ord[q2];
        if (a >= na || T.acc_tensor[a] != t) continue;
        for (int rr = 0; rr < T.t_rank[t]; ++rr) {
          const DExpr& e = T.expr[a][rr];
          for (int k = 0; k < e.nt; ++k)
            if (present(T.term[e.t0 + k], flags) && T.term[e.t0 + k].slot == c.hs[j]) uses |= 1u << t;
        }
      }
    }
    if (single > cap) m_reuse &= uses | ~m_pres;
    for (int t = 0; t < nT; ++t) {
      if (!((m_pres >> t) & 1u)) continue;
      const int64_t per = (single <= cap || ((m_reuse >> t) & 1u)) ? ffull[t] : m_dm[t] * c.he[j];
      if (ffull[t] > cap) m_reuse &= ~(1u << t);
      dm[j][t] = per;
    }
    rb[j] = (uint8_t)m_reuse;
    pres[j] = (uint8_t)m_pres;
  }
  int64_t dmov = 0;
  for (int n = c.root; n >= 0; n = c.nxt[n]) {
    if (n < na) {
      dmov += 1;
    } else {
      for (int t = 0; t < nT; ++t)
        if ((pres[n - na] >> t) & 1u) dmov += dm[n - na][t];
    }
  }
  // ---- emitted code (ls/ir.py:557-659).  Per loop: W = trips of the enclosing branching
  // loops (inlined = unrolled or vector loops do not branch), W' the same with the PTX
  // counter-register wrap, copies = how often its code is emitted (unrolled ancestors),
  // Wv = product of enclosing extents with vector loops counting 1 (smem volume)
  int64_t W[NSLOT], Wp[NSLOT], cp[NSLOT], Wv[NSLOT];
  uint8_t height[NSLOT];
  for (int q = c.nn - 1; q >= 0; --q) {  // branching levels below: counter registers repeat every 8 depths
    const int L = c.ord[q];
    if (L < na) continue;
    int h = 0;
    for (int ch = c.first[L]; ch >= 0; ch = c.nxt[ch])
      if (ch >= na) h = max(h, height[ch - na] + ((c.hf[ch - na] & (F_UNR | F_VEC)) ? 0 : 1));
    height[L - na] = (uint8_t)h;
  }
  int64_t nld = 0, nst = 0, ilp = 0, ptx_loops = 0, wld = 0, wst = 0;
  const int64_t* ic = T.ptx_icost;
  int ntop = 0;
  for (int q = 0; q < c.nn; ++q) {
    const int L = c.ord[q];
    if (L < na) continue;
    const int j = L - na, p = c.par[L];
    const bool inl = c.hf[j] & (F_UNR | F_VEC);
    const int64_t Wpar = p >= 0 ? W[p - na] : 1, Wppar = p >= 0 ? Wp[p - na] : 1;
    const int64_t cpar = p >= 0 ? cp[p - na] * ((c.hf[p - na] & F_UNR) ? c.he[p - na] : 1) : 1;
    cp[j] = cpar;
    Wv[j] = (p >= 0 ? Wv[p - na] : 1) * ((c.hf[j] & F_VEC) ? 1 : c.he[j]);
    W[j] = inl ? Wpar : Wpar * c.he[j];
    Wp[j] = inl ? Wppar : Wppar * (height[j] >= 8 ? 1 : c.he[j]);  // no trip 8+ levels deep (ls/ptx.py:163-169)
    const int g = c.grp[j];
    const int64_t gl = g >= 0 ? T.tr_nld[g] : 0, gs = g >= 0 ? T.tr_nst[g] : 0;
    // the loop's own accesses are emitted copies(L) x (its extent if unrolled) times
    const int64_t acopies = cp[j] * ((c.hf[j] & F_UNR) ? c.he[j] : 1);
    wld += gl * acopies * Wp[j];
    wst += gs * acopies * Wp[j];
    if (inl) continue;
    if (p < 0) ++ntop;
    nld += gl * W[j];
    nst += gs * W[j];
    int nch = 0;
    for (int ch = c.first[L]; ch >= 0; ch = c.nxt[ch]) nch += ch >= na;
    if (T.family == LS_FAMILY_CPU) {
      // header block [group body + first child's init | own latch] x W, then between
      // consecutive child loops one init block and after the last one the latch block
      const int64_t hdr = nch ? (g >= 0 ? T.tr_c_hi[g] : T.c_init) : (g >= 0 ? T.tr_c_hl[g] : T.c_latch);
      ilp += hdr * W[j];
      if (nch) ilp += T.c_init * (nch - 1) + T.c_latch;
    } else {
      ptx_loops += cp[j] * (ic[LS_I_INIT] * Wppar + (ic[LS_I_ADD] + ic[LS_I_CMP] + ic[LS_I_BRANCH]) * Wp[j]);
    }
  }
  int nf;
  if (T.family == LS_FAMILY_CPU) {
    if (T.tr_inline) {  // inlined loops: replay the emission (greedy loop_map, every block scheduled)
      int64_t nfma;
      const int est = em_cpu_features(T, c, nfma, nld, nst, ilp);
      if (est) return est;
      f[0] = (double)nfma;
    } else {
      ilp += T.c_init * ntop + T.c_ret;  // the top-level init blocks and `ret`
      f[0] = (double)nst;
    }
    f[1] = (double)nld;
    f[2] = (double)nst;
    f[3] = (double)dmov;
    f[4] = (double)ilp;
    nf = LS_NFEAT_CPU;
  } else {
    double work;
    if (T.costs_integral) {
      work = (double)(ptx_loops + wld * ic[LS_I_LOAD] + wst * (ic[LS_I_FMA] + ic[LS_I_STORE]) + ic[LS_I_RET]);
    } else {  // thread_cycles in line order (ls/ptx.py:225-235): the emission replayed with its copies
      work = tree_ptx_ordered(T, c, Wp);
    }
    double smem = 0.0;
    if (T.has_shared) {  // smem_ops_feature (ls/ptx.py:310-327): vol = product of the enclosing extents
      for (int q = 0; q < c.nn; ++q) {
        const int a = c.ord[q];
        if (a >= na || !T.t_shared[T.acc_tensor[a]]) continue;
        const int p = c.par[a];
        const int64_t vol = p >= 0 ? Wv[p - na] : 1;
        // tid: `tid`, else the last preorder parallel loop indexing the access (ls/ptx.py:298-307)
        uint32_t used = 0;
        const int t = T.acc_tensor[a];
        for (int rr = 0; rr < T.t_rank[t]; ++rr) {
          const DExpr& e = T.expr[a][rr];
          for (int k = 0; k < e.nt; ++k)
            if (present(T.term[e.t0 + k], flags)) used |= 1u << T.term[e.t0 + k].slot;
        }
        int tid = -1;
        if (T.tid_slot >= 0 && ((used >> T.tid_slot) & 1u)) {
          tid = T.tid_slot;
        } else {
          for (int q2 = 0; q2 < c.nn; ++q2) {
            const int L = c.ord[q2];
            if (L >= na && (c.hf[L - na] & F_PAR) && ((used >> c.hs[L - na]) & 1u)) tid = c.hs[L - na];
          }
        }
        int64_t best = 1;
        if (tid >= 0 && c.nos[tid] >= 0) {
          const int lanes = min(T.warp_size, c.he[c.nos[tid]]);
          int64_t A = 0, B = 0;
          for (int rr = 0; rr < T.t_rank[t]; ++rr) {
            const DExpr& e = T.expr[a][rr];
            int64_t ct = 0;
            for (int k = 0; k < e.nt; ++k) {
              const DTerm& tm = T.term[e.t0 + k];
              if (present(tm, flags) && tm.slot == tid) ct += tm.coef;
            }
            A += (int64_t)e.konst * T.t_stride[t][rr];
            B += ct * T.t_stride[t][rr];
          }
          uint8_t cnt[64];
          for (int b = 0; b < T.banks; ++b) cnt[b] = 0;
          int64_t prev = 0;
          best = 0;
          for (int l = 0; l < lanes; ++l) {
            const int64_t num = (A + B * l) * T.t_eb[t];
            const int64_t w = num >= 0 ? num / 4 : -((-num + 3) / 4);
            if (l == 0 || w != prev) {
              int64_t b = w % T.banks;
              if (b < 0) b += T.banks;
              best = max(best, (int64_t)++cnt[b]);
            }
            prev = w;
          }
        }
        smem = rn_add(smem, (double)(vol * best));
      }
    }
    f[0] = work;
    f[1] = T.sm_underuse;
    f[2] = T.warp_slack;
    f[3] = smem;
    f[4] = (double)wst;
    f[5] = (double)wld;
    f[6] = (double)wst;
    nf = LS_NFEAT_GPU;
  }
  double total = 0.0;
  for (int q = 0; q < nf; ++q) {
    if (!(f[q] >= 0.0) || isinf(f[q])) return LS_ST_BAD_FEATURE;
    total = rn_add(total, rn_mul(T.coef[q], f[q]));
  }
  *score = total;
  return LS_OK;
}

// Per reorder choice: the transformed chain and the status of apply_fast with
// every tile factor 1 (always in range), i.e. what the reorder alone decides.
__global__ void build_pchain_kernel(const DTask* __restrict__ g, int32_t pax, uint64_t* __restrict__ chain,
                                    int32_t* __restrict__ pst) {
  extern __shared__ __align__(16) unsigned char dyn[];
  const DTask& T = *g;
  const int pc = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = pax >= 0 ? (int)T.sp_ax[pax].n : 1;
  FastCand c;
  c.ext = reinterpret_cast<int32_t*>(dyn) + threadIdx.x;
  if (pc >= n) return;
  ls_record r;
  memset(&r, 0, sizeof(r));
  for (int q = 0; q < LS_MAX_PARAMS; ++q) r.param[q] = 1;
  r.perm = pax >= 0 ? T.sp_vals[T.sp_ax[pax].voff + pc] : 0;
  const int st = apply_fast(T, r, c);
  pst[pc] = st;
  chain[pc] = st ? 0 : c.chain;
}

// One dimension-table entry per thread: decode (dimension, key, mask).
__global__ void build_tab_kernel(const DTask* __restrict__ g, int32_t* __restrict__ tab) {
  const DTask& T = *g;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T.tab_len) return;
  int D = -1;
  for (int q = 0; q < 16; ++q)
    if (T.ftab_len[q] > 0 && e >= T.ftab_off[q] && e < T.ftab_off[q] + T.ftab_len[q]) D = q;
  if (D < 0) {
    if (e == T.tab_one) tab[e] = 1;
    return;
  }
  const int nv = T.dim_nv[D];
  const int loc = e - T.ftab_off[D];
  const uint32_t mask = (uint32_t)loc & ((1u << nv) - 1u);
  int32_t key = loc >> nv;
  int32_t prm[LS_MAX_PARAMS];
  for (int q = 0; q < LS_MAX_PARAMS; ++q) prm[q] = 1;
  uint32_t flags = 0;
  for (int q = T.fk_n[D] - 1; q >= 0; --q) {
    const int32_t d = key % T.fk_rad[D][q];
    key /= T.fk_rad[D][q];
    const int src = T.fk_src[D][q];
    if (src < LS_MAX_PARAMS)
      prm[src] = d;
    else
      flags |= (uint32_t)d << (src - LS_MAX_PARAMS);
  }
  int32_t E[NSLOT], St[NSLOT];
  uint32_t exist;
  sim_slots(T, prm, flags, E, St, exist);
  tab[e] = dim_count(T, D, mask, flags, E, St, exist);
}

// One tensor-table entry per thread: decode (tensor, axis choices, mask of all
// the tensor's stage bits); the entry is the tensor footprint, the product of
// its dimension counts (ls/cache.py:117-130).
__global__ void build_ttab_kernel(const DTask* __restrict__ g, uint64_t* __restrict__ tt) {
  const DTask& T = *g;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T.tt_len) return;
  int t = -1;
  for (int q = 0; q < T.n_tensors && q < 4; ++q)
    if (e >= T.tt_off[q] && e < (int64_t)T.tt_off[q] + T.tt_len_t[q]) t = q;
  if (t < 0) return;
  const int nb = T.tt_nb[t];
  const uint32_t loc = (uint32_t)(e - T.tt_off[t]);
  const uint32_t mask = loc & ((1u << nb) - 1u);
  const uint32_t key = loc >> nb;
  int32_t prm[LS_MAX_PARAMS];
  for (int q = 0; q < LS_MAX_PARAMS; ++q) prm[q] = 1;
  uint32_t flags = 0;
  for (int a = 0; a < T.sp_n; ++a) {
    const uint32_t stride = T.tt_stride[t][a];
    if (!stride) continue;
    const DAxis& ax = T.sp_ax[a];
    const uint32_t c = (key / stride) % ax.n;
    if (ax.kind == LS_AX_BIT) {
      flags |= c << ax.bit;
      continue;
    }
    const uint64_t v = T.sp_vals[ax.voff + c];
    prm[ax.param] = (int32_t)v;
    if (ax.kind == LS_AX_VEC && v != 0) flags |= 1u << ax.bit;
  }
  int32_t E[NSLOT], St[NSLOT];
  uint32_t exist;
  sim_slots(T, prm, flags, E, St, exist);
  uint64_t F = 1;
  const int tb = T.dim_base[t * 4];
  for (int rr = 0; rr < T.t_rank[t]; ++rr) {
    const int D = t * 4 + rr;
    const uint32_t m = (mask >> (T.dim_base[D] - tb)) & ((1u << T.dim_nv[D]) - 1u);
    F *= (uint64_t)(uint32_t)dim_count(T, D, m, flags, E, St, exist);
  }
  tt[e] = F;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stage_task(DTask& s, const DTask* __restrict__ g) {
  const int4* src = reinterpret_cast<const int4*>(g);
  int4* dst = reinterpret_cast<int4*>(&s);
  const int n16 = __ldg(&g->task_bytes) / 16;  // header + used terms only
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(&src[i]);
  __syncthreads();
}

// Space path: the task header and its group tables staged together -- both
// sources addressed from global memory (no wait for the staged header), 16-byte
// loads, several in flight per thread, one barrier.  The table allocation is
// padded to 16 bytes.
__device__ __forceinline__ const int32_t* stage_space(unsigned char* dyn, const DTask* __restrict__ g) {
  const int tb = __ldg(&g->task_bytes);
  const int len = __ldg(&g->sd_len);
  const int4* ts = reinterpret_cast<const int4*>(__ldg(reinterpret_cast<const unsigned long long*>(&g->sd_tab)));
  const int n16 = tb / 16, tot = n16 + (len + 3) / 4;
  const int4* gs = reinterpret_cast<const int4*>(g);
  int4* d = reinterpret_cast<int4*>(dyn);  // header, then the tables at dyn + tb (tb % 16 == 0)
#pragma unroll 4
  for (int i = threadIdx.x; i < tot; i += blockDim.x) d[i] = __ldg(i < n16 ? gs + i : ts + (i - n16));
  __syncthreads();
  return reinterpret_cast<const int32_t*>(dyn + tb);
}

// Path selector of the scoring kernels: 0 generic, 1 tabulated with the table
// in global memory (L1/L2 resident), 2 tabulated with the table in shared memory.
template <int MODE>
__device__ __forceinline__ const int32_t* stage_tab(unsigned char* where, const DTask& T) {
  if constexpr (MODE == 2 || MODE == 4 || MODE == 5) {
    int32_t* dst = reinterpret_cast<int32_t*>(where);
    const int32_t* src = MODE == 2 ? T.tab : T.sd_tab;
    const int len = MODE == 2 ? T.tab_len : T.sd_len;
    for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = __ldg(&src[i]);
    __syncthreads();
    return dst;
  } else {
    return T.tab;
  }
}

__host__ __device__ inline size_t tab_smem_bytes(int mode, const DTask& T) {
  return mode == 2 ? align16(sizeof(int32_t) * (size_t)T.tab_len)
                   : (mode == 4 || mode == 5) ? align16(sizeof(int32_t) * (size_t)T.sd_len) : 0;
}
__host__ __device__ inline size_t state_bytes(int mode, int n_slots, int n_chain, int n_stage) {
  return mode == 0   ? cand_bytes(n_slots, n_chain, n_stage)
         : mode == 6 ? 0  // the tree path keeps its state in local memory
                     : align16(sizeof(int32_t) * (size_t)n_slots * TPB);
}

template <int TM, int RM, int MODE>
struct Evaluator {
  Cand c;
  FastCand fc;
  const int32_t* tab;
  __device__ __forceinline__ Evaluator(const DTask& T, unsigned char* state, const int32_t* tab_) : tab(tab_) {
    if constexpr (MODE == 0)
      c = carve(state, T);
    else
      fc.ext = reinterpret_cast<int32_t*>(state) + threadIdx.x;
  }
  __device__ __forceinline__ int operator()(const DTask& T, const ls_record& r, const uint32_t* kt, uint32_t pch,
                                            double* f, double* s) {
    if constexpr (MODE == 0)
      return eval_candidate<TM, RM>(T, r, c, f, s);
    else if constexpr (MODE == 6)
      return eval_tree(T, r, f, s);
    else if constexpr (MODE == 3)
      return eval_tensor<TM>(T, r, kt, fc, f, s);
    else
      return eval_fast<TM, RM, MODE == 2>(T, tab, r, fc, f, s);
  }
};

__device__ __forceinline__ ls_record load_record(const ls_record* __restrict__ recs, int64_t i) {
  const int4* p = reinterpret_cast<const int4*>(recs + i);
  int4 a = __ldg(p), b = __ldg(p + 1);
  ls_record r;
  memcpy(&r, &a, 16);
  memcpy(reinterpret_cast<char*>(&r) + 16, &b, 16);
  return r;
}

template <int SRC, bool KEYS>
__device__ __forceinline__ int load_cand(const DTask& T, const void* __restrict__ src, int pbytes, int64_t i,
                                         ls_record& r, uint32_t* kt, uint32_t& pch) {
  if constexpr (SRC == 0) {
    r = load_record(reinterpret_cast<const ls_record*>(src), i);
    return LS_OK;
  } else {
    const uint64_t x = pbytes == 4 ? (uint64_t)__ldg(reinterpret_cast<const unsigned int*>(src) + i)
                                   : (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(src) + i);
    return point_record<KEYS>(T, x, r, kt, pch);
  }
}

constexpr int min_blocks(int tm, int rm, int mode) { return mode == 6 ? 1 : mode ? 3 : (tm * rm <= 16 ? 3 : 1); }

template <int TM, int RM, int MODE, int SRC>
__global__ void __launch_bounds__(TPB, min_blocks(TM, RM, MODE))
    score_kernel(const DTask* __restrict__ gtask, const void* __restrict__ src, int pbytes, int64_t n,
                 double* __restrict__ scores, double* __restrict__ feats, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char dyn[];
  DTask& T = *reinterpret_cast<DTask*>(dyn);
  stage_task(T, gtask);
  unsigned char* p = dyn + T.task_bytes;
  const int32_t* tab = stage_tab<MODE>(p, T);
  p += tab_smem_bytes(MODE, T);
  Evaluator<TM, RM, MODE> ev(T, p, tab);
  const int nf = T.family == LS_FAMILY_CPU ? LS_NFEAT_CPU : LS_NFEAT_GPU;
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    ls_record r;
    uint32_t kt[4];
    double f[LS_NFEAT_GPU];
    double s = 0.0;
    int st;
    if constexpr (MODE == 4 || MODE == 5) {
      st = eval_space<TM, MODE == 5>(T, tab, load_point(src, pbytes, i), ev.fc, f, &s);
    } else {
      uint32_t pch = 0;
      st = load_cand<SRC, MODE == 3>(T, src, pbytes, i, r, kt, pch);
      if (st == LS_OK) st = ev(T, r, kt, pch, f, &s);
    }
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    if (scores) scores[i] = st ? nan : s;
    if (status) status[i] = st;
    if (feats)
      for (int q = 0; q < nf; ++q) feats[i * nf + q] = st ? nan : f[q];
  }
}

// ---- streaming top-k on (score, index) ------------------------------------
struct Key {
  unsigned long long s;
  long long i;
};
constexpr unsigned long long KEY_INF_S = ~0ull;
constexpr long long KEY_INF_I = LLONG_MAX;

__device__ __forceinline__ bool kless(const Key& a, const Key& b) {
  return a.s < b.s || (a.s == b.s && a.i < b.i);
}
__device__ __forceinline__ unsigned long long order_bits(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_order_bits(unsigned long long o) {
  unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)b);
}

constexpr int TK_MAXK = 1024;
#ifndef TOPK_CAP_SMALL
#define TOPK_CAP_SMALL 1
#endif

// Block top-k state in shared memory: header + a key buffer of `cap` keys
// (cap = 1024 or 2048, <= 8 per thread).  The buffer is an unsorted multiset of
// keys below `thr`; compaction keeps exactly the k smallest by radix selection
// of the k-th key (no sort), filtering in place through registers; only the
// final list of a launch is sorted.
struct __align__(16) TopkState {
  Key thr;
  int cnt, cap, cnt2, pad0;
  unsigned int hist[256];
  int sel_bucket, sel_rank, sel_count, pad;
  unsigned long long and_s, or_s, and_i, or_i;  // common-prefix reduction of the buffered keys
  __device__ __forceinline__ Key* buf() { return reinterpret_cast<Key*>(this + 1); }
  __device__ __forceinline__ const Key* buf() const { return reinterpret_cast<const Key*>(this + 1); }
};
__host__ __device__ constexpr size_t topk_state_bytes(int cap) {
  return sizeof(TopkState) + sizeof(Key) * (size_t)cap;
}

// Sort buf[0..cnt) (padded with +inf) and keep the k smallest; returns the kept
// count.  Used once per launch, on the final <= k keys.
__device__ int topk_compact(TopkState& S, int k, int cnt) {
  Key* const B = S.buf();
  int size0 = 2;
  while (size0 < cnt) size0 <<= 1;  // only the occupied power-of-two prefix needs sorting
  for (int i = cnt + threadIdx.x; i < size0; i += blockDim.x) {
    B[i].s = KEY_INF_S;
    B[i].i = KEY_INF_I;
  }
  __syncthreads();
  for (int size = 2; size <= size0; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < size0 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const Key a = B[lo], b = B[hi];
        if (kless(b, a) == up) {
          B[lo] = b;
          B[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  const int keep = cnt < k ? cnt : k;
  if (threadIdx.x == 0) {
    S.cnt = keep;
    if (keep == k) S.thr = B[k - 1];
  }
  __syncthreads();
  return keep;
}

// 8-bit digit d (0 = most significant) of the 128-bit key (s, i).
__device__ __forceinline__ unsigned key_digit(const Key& x, int d) {
  const unsigned long long w = d < 8 ? x.s : (unsigned long long)x.i;
  return (unsigned)(w >> (56 - 8 * (d & 7))) & 0xFFu;
}

// Keep exactly the k smallest keys of the buffer (all of them when cnt <= k)
// and set thr to the k-th: MSD radix selection of the k-th key over 8-bit
// digits of (score bits, index) until its bucket holds one key, then one
// filtering pass into the other buffer.  Keys are distinct (unique indices),
// so the k-th key and the kept set are unique.  Returns the kept count.
__device__ __forceinline__ unsigned long long warp_and64(unsigned long long x) {
  return ((unsigned long long)__reduce_and_sync(0xffffffffu, (unsigned)(x >> 32)) << 32) |
         __reduce_and_sync(0xffffffffu, (unsigned)x);
}
__device__ __forceinline__ unsigned long long warp_or64(unsigned long long x) {
  return ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(x >> 32)) << 32) |
         __reduce_or_sync(0xffffffffu, (unsigned)x);
}

// Warp-aggregated append: one atomic per warp for the lanes with pred set;
// returns the lane's slot (or -1).  All 32 lanes of the warp must call it.
template <typename C>
__device__ __forceinline__ int warp_append(C* ctr, bool pred) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return -1;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  C b = 0;
  if (lane == leader) b = atomicAdd(ctr, (C)__popc(m));
  b = __shfl_sync(0xffffffffu, b, leader);
  return pred ? (int)b + __popc(m & ((1u << lane) - 1u)) : -1;
}

__device__ int topk_select(TopkState& S, int k) {
  const int c = S.cnt;
  if (c <= k) return c;
  const Key* const B = S.buf();
  const int lane = threadIdx.x & 31;
  const int c_up = (c + blockDim.x - 1) / blockDim.x * blockDim.x;  // warp-uniform trip count
  // digits every buffered key shares are skipped: AND / OR of the keys
  if (threadIdx.x == 0) {
    S.and_s = S.and_i = ~0ull;
    S.or_s = S.or_i = 0ull;
  }
  __syncthreads();
  {
    unsigned long long as = ~0ull, os = 0, ai = ~0ull, oi = 0;
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      const Key x = B[j];
      as &= x.s;
      os |= x.s;
      ai &= (unsigned long long)x.i;
      oi |= (unsigned long long)x.i;
    }
    as = warp_and64(as);
    os = warp_or64(os);
    ai = warp_and64(ai);
    oi = warp_or64(oi);
    if (lane == 0) {
      atomicAnd(&S.and_s, as);
      atomicOr(&S.or_s, os);
      atomicAnd(&S.and_i, ai);
      atomicOr(&S.or_i, oi);
    }
  }
  __syncthreads();
  unsigned long long ps = 0, pi = 0, ms = 0, mi = 0;  // known digits of the k-th key (block-uniform)
  int d0;
  {
    const unsigned long long xs = S.and_s ^ S.or_s, xi = S.and_i ^ S.or_i;
    if (xs) {
      d0 = __clzll((long long)xs) / 8;
      ms = d0 ? ~0ull << (64 - 8 * d0) : 0ull;
      ps = S.and_s & ms;
    } else {
      ms = ~0ull;
      ps = S.and_s;
      d0 = xi ? 8 + __clzll((long long)xi) / 8 : 16;
      mi = d0 > 8 && d0 < 16 ? ~0ull << (64 - 8 * (d0 - 8)) : (d0 == 16 ? ~0ull : 0ull);
      pi = S.and_i & mi;
    }
  }
  int rank = k;  // rank of the k-th key among keys matching the known digits
  for (int d = d0; d < 16; ++d) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) S.hist[b] = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < c_up; j += blockDim.x) {  // warp-aggregated histogram
      unsigned dig = 0x100u;
      if (j < c) {
        const Key x = B[j];
        if ((x.s & ms) == ps && ((unsigned long long)x.i & mi) == pi) dig = key_digit(x, d);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      if (dig < 0x100u && (__ffs(peers) - 1) == lane) atomicAdd(&S.hist[dig], (unsigned)__popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      unsigned h[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) sum += (h[q] = S.hist[8 * l + q]);
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
      }
      const unsigned excl = incl - sum;
      if (excl < (unsigned)rank && (unsigned)rank <= incl) {
        unsigned cum = excl;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (cum + h[q] >= (unsigned)rank) {
            S.sel_bucket = 8 * l + q;
            S.sel_rank = rank - (int)cum;
            S.sel_count = (int)h[q];
            break;
          }
          cum += h[q];
        }
      }
    }
    __syncthreads();
    const unsigned long long b = (unsigned long long)S.sel_bucket;
    const int sh = 56 - 8 * (d & 7);
    if (d < 8) {
      ps |= b << sh;
      ms |= 0xFFull << sh;
    } else {
      pi |= b << sh;
      mi |= 0xFFull << sh;
    }
    rank = S.sel_rank;
    const bool done = S.sel_count == 1;
    __syncthreads();
    if (done) break;
  }
  // the k-th key is the only one matching the selected digits
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    const Key x = B[j];
    if ((x.s & ms) == ps && ((unsigned long long)x.i & mi) == pi) S.thr = x;
  }
  if (threadIdx.x == 0) S.cnt2 = 0;
  __syncthreads();
  const Key thr = S.thr;
  // in place, 4 keys per thread per chunk: a chunk's reads end (barrier) before
  // its writes, and writes land below the keys read so far, so they never reach
  // a later chunk's unread keys
  Key* const W = S.buf();
  for (int base = 0; base < c; base += 4 * blockDim.x) {
    Key keep[4];
    bool kp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = base + threadIdx.x + q * blockDim.x;
      kp[q] = false;
      if (j < c) {
        keep[q] = B[j];
        kp[q] = !kless(thr, keep[q]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int slot = warp_append(&S.cnt2, kp[q]);
      if (slot >= 0) W[slot] = keep[q];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) S.cnt = S.cnt2;
  __syncthreads();
  return k;
}

__device__ __forceinline__ void topk_init(TopkState& S, int cap) {
  if (threadIdx.x == 0) {
    S.cap = cap;
    S.cnt = 0;
    S.thr.s = KEY_INF_S;
    S.thr.i = KEY_INF_I;
  }
  __syncthreads();
}

// Insert-if-better without a barrier; the block synchronises only when the
// buffer could overflow within the next round (`safe` rounds are free).
__device__ __forceinline__ void topk_offer(TopkState& S, bool has, const Key& key, int k, int& safe) {
  if (has && kless(key, S.thr)) {  // rare after the first rounds: a plain atomic beats a warp vote
    const int slot = atomicAdd(&S.cnt, 1);
    S.buf()[slot] = key;
  }
  if (--safe > 0) return;
  __syncthreads();
  int c = S.cnt;
  const bool open = S.thr.s == KEY_INF_S && S.thr.i == KEY_INF_I;
  __syncthreads();
  // select when another round could overflow, and as soon as k keys exist
  // without a threshold (an early threshold keeps later inserts rare)
  if (c > S.cap - (int)blockDim.x || (open && c > k)) c = topk_select(S, k);
  safe = (S.cap - c) / (int)blockDim.x;
}

constexpr int TK_GROUP = 16;  // blocks per first-level merge group
constexpr int TK_DYN_CTR = 1023;  // tickets[] slot of the dynamic round counter
constexpr int TK_FIN_CTR = 1022;  // tickets[] slot of the two-stage finish ticket
constexpr int TK_MAXGRID = 2048;  // two-stage minima slots (grid <= topk_buf(k) <= 2048); slot TK_MAXGRID = T

// Phase timestamps of the fused kernel (LS_TRACE=1, tools/ only): per block
// [start, staged, main loop done, block list written, group merged, final written].
constexpr int TR_SLOTS = 9;  // 8 timestamps + the SM id
// (the trace buffer is a kernel parameter: no global load at kernel start when off)
__device__ __forceinline__ void trace_mark(unsigned long long* g_trace, int slot) {
  if (g_trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[blockIdx.x * TR_SLOTS + slot] = t;
    if (slot == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_trace[blockIdx.x * TR_SLOTS + 8] = sm;
    }
  }
}

__device__ __forceinline__ Key ld_key_cg(const Key* p) {
  Key k;
  k.s = __ldcg(reinterpret_cast<const unsigned long long*>(p));
  k.i = __ldcg(reinterpret_cast<const long long*>(p) + 1);
  return k;
}

// Merge m keys from global memory into the block's buffer (streamed, k kept).
// (sorted: the kept keys end ascending; otherwise they stay an unsorted set)
// Keys are loaded in chunks of cap - k (four per thread in flight), appended
// below the running threshold, and a selection follows each chunk.
__device__ int merge_into(TopkState& S, const Key* src, int64_t m, int k, bool sorted) {
  topk_init(S, S.cap);
  const int chunk = S.cap - k;
  for (int64_t base = 0; base < m; base += chunk) {
    const int64_t lim = min(m, base + chunk);
    for (int64_t j0 = base; j0 < lim; j0 += 4 * (int64_t)blockDim.x) {
      Key key[4];
      bool has[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i = j0 + q * (int64_t)blockDim.x + threadIdx.x;
        has[q] = i < lim;
        if (has[q]) key[q] = ld_key_cg(src + i);
      }
      const Key thr = S.thr;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int slot =
            warp_append(&S.cnt, has[q] && !(key[q].s == KEY_INF_S && key[q].i == KEY_INF_I) && kless(key[q], thr));
        if (slot >= 0) S.buf()[slot] = key[q];
      }
    }
    __syncthreads();
    topk_select(S, k);
  }
  __syncthreads();
  const int kept = min(S.cnt, k);
  return sorted ? topk_compact(S, k, kept) : kept;
}

__device__ void write_keys(const TopkState& S, int kept, int k, Key* out) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    Key o;
    if (j < kept) {
      o = S.buf()[j];
    } else {
      o.s = KEY_INF_S;
      o.i = KEY_INF_I;
    }
    out[j] = o;
  }
}

// Write the kept keys ascending as (score, index), +inf / -1 padded to k.
// kept <= blockDim: every thread ranks one key by counting the smaller ones
// (keys are distinct); otherwise a bitonic sort.
__device__ void write_sorted(TopkState& S, int kept, int k, double* __restrict__ out_s, int64_t* __restrict__ out_i) {
  if (kept <= (int)blockDim.x) {
    __syncthreads();
    if ((int)threadIdx.x < kept) {
      const Key x = S.buf()[threadIdx.x];
      int r = 0;
      for (int j = 0; j < kept; ++j) r += kless(S.buf()[j], x) ? 1 : 0;
      out_s[r] = from_order_bits(x.s);
      out_i[r] = x.i;
    }
  } else {
    kept = topk_compact(S, k, kept);
    for (int j = threadIdx.x; j < kept; j += blockDim.x) {
      out_s[j] = from_order_bits(S.buf()[j].s);
      out_i[j] = S.buf()[j].i;
    }
  }
  for (int j = kept + threadIdx.x; j < k; j += blockDim.x) {
    out_s[j] = __longlong_as_double(0x7ff0000000000000ll);
    out_i[j] = -1;
  }
}

// Smallest of the block's kept keys (+inf when none) to *out.
__device__ void write_block_min(const TopkState& S, int kept, Key* out) {
  __shared__ Key wmin[TPB / 32];
  Key m;
  m.s = KEY_INF_S;
  m.i = KEY_INF_I;
  for (int j = threadIdx.x; j < kept; j += blockDim.x) {
    const Key x = S.buf()[j];
    if (kless(x, m)) m = x;
  }
  for (int off = 16; off > 0; off >>= 1) {
    Key o;
    o.s = __shfl_down_sync(0xffffffffu, m.s, off);
    o.i = __shfl_down_sync(0xffffffffu, m.i, off);
    if (kless(o, m)) m = o;
  }
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (kless(wmin[w], m)) m = wmin[w];
    *out = m;
  }
}

// Sort B[0..cnt) ascending in shared memory (bitonic over the next power of two,
// +inf padded; B must hold it).
__device__ void bitonic_sort(Key* B, int cnt) {
  int size0 = 2;
  while (size0 < cnt) size0 <<= 1;
  for (int i = cnt + threadIdx.x; i < size0; i += blockDim.x) {
    B[i].s = KEY_INF_S;
    B[i].i = KEY_INF_I;
  }
  __syncthreads();
  for (int size = 2; size <= size0; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < size0 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const Key a = B[lo], b = B[hi];
        if (kless(b, a) == up) {
          B[lo] = b;
          B[hi] = a;
        }
      }
      __syncthreads();
    }
}

// Second stage of the fused top-k when k is small next to the grid (the
// fused kernel wrote every block's k best and its minimum).  T = the k-th
// smallest block minimum bounds the global k-th key from above (the k minima
// are k real keys <= T), so only list keys <= T can be in the answer: every
// block finds T, filters its share of the lists into `surv`, and the last
// block ranks the survivors (~k of them) into the sorted output.
__global__ void __launch_bounds__(TPB) merge_filter_kernel(const Key* __restrict__ block_out,
                                                           const Key* __restrict__ mins, int nblk, int k,
                                                           Key* __restrict__ surv, unsigned int* __restrict__ ctr,
                                                           double* __restrict__ out_s, int64_t* __restrict__ out_i,
                                                           int cap, unsigned long long* __restrict__ n_valid,
                                                           unsigned long long* __restrict__ wvalid,
                                                           unsigned long long* __restrict__ g_trace) {
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ unsigned int s_ticket;
  __shared__ Key s_T;
  TopkState& S = *reinterpret_cast<TopkState*>(raw);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scoring grid is complete and visible
  trace_mark(g_trace, 4);
  // the first chunk of this block's list is loaded while T is read (independent loads)
  const unsigned int* cnts = reinterpret_cast<const unsigned int*>(mins + TK_MAXGRID + 1);
  int cb0 = (int)blockIdx.x < nblk ? (int)__ldcg(cnts + blockIdx.x) : 0;
  Key x0;
  x0.s = KEY_INF_S;
  x0.i = KEY_INF_I;
  if ((int)threadIdx.x < cb0) x0 = ld_key_cg(block_out + (int64_t)blockIdx.x * cap + threadIdx.x);
  // T: published by the scoring grid's (3/4 grid)-th finisher; else the k-th smallest block minimum
  Key* B = S.buf();
  __shared__ int s_n;
  if (threadIdx.x == 0) {
    S.cap = cap;  // merge_into (many survivors) streams in chunks of cap - k
    s_n = 0;
    s_T = ld_key_cg(mins + TK_MAXGRID);
    if (s_T.s == KEY_INF_S) s_T.i = KEY_INF_I;
  }
  __syncthreads();
  if (s_T.s == KEY_INF_S) {
    for (int j0 = 0; j0 < nblk; j0 += blockDim.x) {  // block-uniform trip count (warp appends)
      const int j = j0 + threadIdx.x;
      Key x;
      x.s = KEY_INF_S;
      if (j < nblk) x = ld_key_cg(mins + j);
      const int slot = warp_append(&s_n, x.s != KEY_INF_S);
      if (slot >= 0) B[slot] = x;
    }
    __syncthreads();
    const int nm = s_n;
    if (nm > k) {  // radix selection of the k-th minimum (the block buffer's select, no sort)
      if (threadIdx.x == 0) S.cnt = nm;
      __syncthreads();
      topk_select(S, k);
      if (threadIdx.x == 0) s_T = S.thr;
    }
    __syncthreads();
  }
  const Key T = s_T;  // +inf (no filtering) when there are at most k minima
  trace_mark(g_trace, 5);
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {  // block b's list: cnts[b] keys at b * cap
    const int cb = b == (int)blockIdx.x ? cb0 : (int)__ldcg(cnts + b);
    const Key* lst = block_out + (int64_t)b * cap;
    for (int j0 = 0; j0 < cb; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      Key x;
      x.s = KEY_INF_S;
      x.i = KEY_INF_I;
      if (j0 == 0 && b == (int)blockIdx.x) x = x0;
      else if (j < cb) x = ld_key_cg(lst + j);
      const int slot = warp_append(&ctr[0], j < cb && !kless(T, x));
      if (slot >= 0) surv[slot] = x;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(&ctr[1], 1u);
  __syncthreads();
  trace_mark(g_trace, 6);
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  const int c = (int)__ldcg(&ctr[0]);
  // every scoring block is done: the valid count is final (read now, off the tail's critical path)
  const unsigned long long v_final = threadIdx.x == 0 ? __ldcg(wvalid) : 0ull;
  if (g_trace && threadIdx.x == 0) g_trace[blockIdx.x * TR_SLOTS + 3] = (1ull << 63) | (unsigned long long)c;
  Key* buf = S.buf();
  if (c <= (int)blockDim.x) {  // rank the survivors directly; the k smallest land at their rank
    __syncthreads();
    if ((int)threadIdx.x < c) buf[threadIdx.x] = ld_key_cg(surv + threadIdx.x);
    __syncthreads();
    if ((int)threadIdx.x < c) {
      const Key x = buf[threadIdx.x];
      int r = 0;
      for (int q = 0; q < c; ++q) r += kless(buf[q], x) ? 1 : 0;
      if (r < k) {
        out_s[r] = from_order_bits(x.s);
        out_i[r] = x.i;
      }
    }
    for (int j = c + threadIdx.x; j < k; j += blockDim.x) {
      out_s[j] = __longlong_as_double(0x7ff0000000000000ll);
      out_i[j] = -1;
    }
  } else {
    write_sorted(S, merge_into(S, surv, c, k, false), k, out_s, out_i);
  }
  if (threadIdx.x == 0) {  // the count out; the counters back to zero for the next launch
    if (n_valid) *n_valid = v_final;
    *wvalid = 0ull;
    ctr[0] = 0;
    ctr[1] = 0;
    ctr[TK_DYN_CTR] = 0;
    ctr[TK_FIN_CTR] = 0;
  }
  for (int j = threadIdx.x; j <= nblk; j += blockDim.x) {  // minima slots (and T) back to +inf
    Key* m = const_cast<Key*>(mins) + (j < nblk ? j : TK_MAXGRID);
    m->s = KEY_INF_S;
    m->i = KEY_INF_I;
  }
  trace_mark(g_trace, 7);
}

// Fused pass: score every record, keep the block's k best, then merge the
// block lists in a two-level tree inside the same launch: the last block of
// each group of TK_GROUP merges its group, the last group merger writes the
// final k (threadfence + ticket counters; no second kernel).
template <int TM, int RM, int MODE, int SRC>
__global__ void __launch_bounds__(TPB, min_blocks(TM, RM, MODE)) score_topk_kernel(
    const DTask* __restrict__ gtask, const void* __restrict__ src, int pbytes, int64_t n, int64_t base_index, int k,
    Key* __restrict__ block_out, Key* __restrict__ group_out, unsigned int* __restrict__ tickets,
    double* __restrict__ out_s, int64_t* __restrict__ out_i, unsigned long long* __restrict__ n_valid, int cap,
    Key* __restrict__ mins, unsigned long long* __restrict__ wvalid, unsigned long long* __restrict__ g_trace) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ unsigned int s_ticket;
  DTask& T = *reinterpret_cast<DTask*>(dyn);
  trace_mark(g_trace, 0);
  const int32_t* tab;
  if constexpr (MODE == 4 || MODE == 5) {
    tab = stage_space(dyn, gtask);
  } else {
    stage_task(T, gtask);
    tab = stage_tab<MODE>(dyn + T.task_bytes, T);
  }
  unsigned char* p = dyn + T.task_bytes + tab_smem_bytes(MODE, T);
  TopkState& S = *reinterpret_cast<TopkState*>(p);
  Evaluator<TM, RM, MODE> ev(T, p + align16(topk_state_bytes(cap)), tab);
  topk_init(S, cap);
  trace_mark(g_trace, 1);
  unsigned int valid = 0;
  int safe = 1;
  // Rounds of TPB candidates.  Each block owns a contiguous static share of
  // 3/4 of all rounds; the rest are handed out one round at a time from a
  // global counter (tickets[TK_DYN_CTR]), so blocks the SM's warp scheduler
  // favours take more of them and every SM finishes together.  The round after
  // next is known one round ahead (block-uniform), so the next round's points
  // are prefetched; a dynamic round's base is published through s_nb at a
  // barrier.
  __shared__ int64_t s_nb[2], s_first[2];
  unsigned int* const dyn_ctr = tickets + TK_DYN_CTR;
  const int64_t rounds = (n + TPB - 1) / TPB;
  const int64_t st_rounds = rounds * 3 / 4 / gridDim.x;  // static rounds per block
  const int64_t dyn0 = st_rounds * gridDim.x * TPB;     // first dynamically distributed candidate
  const int64_t sb0 = (int64_t)blockIdx.x * st_rounds * TPB;
  auto round_base = [&](int64_t r) -> int64_t {  // thread 0: base of the block's round r
    return r < st_rounds ? sb0 + r * TPB : dyn0 + (int64_t)atomicAdd(dyn_ctr, 1u) * TPB;
  };
  if (threadIdx.x == 0) {
    s_first[0] = round_base(0);
    s_first[1] = round_base(1);
  }
  __syncthreads();
  int64_t base = s_first[0], nb = s_first[1];
  uint64_t xn = 0;  // space path: the next point, loaded one round ahead
  if constexpr (MODE == 4 || MODE == 5)
    if (base + threadIdx.x < n) xn = load_point(src, pbytes, base + threadIdx.x);
  for (int64_t r = 0; base < n; ++r) {
    const bool dyn = r + 2 >= st_rounds;  // block-uniform: round r + 2 is dynamic
    if (dyn && threadIdx.x == 0) s_nb[r & 1] = round_base(r + 2);
    const int64_t i = base + threadIdx.x;
    bool has = false;
    Key key;
    if (i < n) {
      ls_record r_;
      uint32_t kt[4];
      double f[LS_NFEAT_GPU];
      double s;
      int st;
      if constexpr (MODE == 4 || MODE == 5) {
        const uint64_t x = xn;
        if (nb + threadIdx.x < n) xn = load_point(src, pbytes, nb + threadIdx.x);
        st = eval_space<TM, MODE == 5>(T, tab, x, ev.fc, f, &s);
      } else {
        uint32_t pch = 0;
        st = load_cand<SRC, MODE == 3>(T, src, pbytes, i, r_, kt, pch);
        if (st == LS_OK) st = ev(T, r_, kt, pch, f, &s);
      }
      if (st == LS_OK) {
        key.s = order_bits(s);
        key.i = base_index + i;
        has = true;
        ++valid;
      }
    }
    topk_offer(S, has, key, k, safe);
    base = nb;
    if (dyn) {
      __syncthreads();
      nb = s_nb[r & 1];
    } else {
      nb = sb0 + (r + 2) * TPB;
    }
  }
  for (int off = 16; off > 0; off >>= 1) valid += __shfl_down_sync(0xffffffffu, valid, off);
  if ((threadIdx.x & 31) == 0 && valid) atomicAdd(wvalid, (unsigned long long)valid);
  __syncthreads();
  trace_mark(g_trace, 2);
  if (mins) {  // second stage (merge_filter_kernel): the whole buffer, a superset of the
               // block's k best (a key leaves it only below k smaller ones), its count and minimum
    asm volatile("griddepcontrol.launch_dependents;");  // the merge launch may be scheduled now
    const int cnt = S.cnt;
    Key* dst = block_out + (int64_t)blockIdx.x * cap;
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) dst[j] = S.buf()[j];
    if (threadIdx.x == 0) reinterpret_cast<unsigned int*>(mins + TK_MAXGRID + 1)[blockIdx.x] = (unsigned)cnt;
    write_block_min(S, cnt, mins + blockIdx.x);
    // The (3/4 grid)-th block to get here bounds the merge early, while the rest
    // still score: T = the k-th smallest minimum present in the slots (>= 3/4 grid
    // >= 3k are, fenced before their tickets).  Slots are +inf (absent) or a finished
    // block's minimum -- a torn read of one still lies at or above a real key of
    // that block -- so T has k real keys at or below it: an upper bound of the
    // global k-th key.  The merge kernel resets every slot after use.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(&tickets[TK_FIN_CTR], 1u);
    __syncthreads();
    if (s_ticket == gridDim.x * 3 / 4 - 1) {
      Key* B = S.buf();
      if (threadIdx.x == 0) S.cnt = 0;
      __syncthreads();
      for (int j0 = 0; j0 < (int)gridDim.x; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        Key x;
        x.s = KEY_INF_S;
        if (j < (int)gridDim.x) x = ld_key_cg(mins + j);
        const int slot = warp_append(&S.cnt, x.s != KEY_INF_S);
        if (slot >= 0) B[slot] = x;
      }
      __syncthreads();
      if (S.cnt > k) {
        topk_select(S, k);
        if (threadIdx.x == 0) {
          mins[TK_MAXGRID].i = S.thr.i;
          mins[TK_MAXGRID].s = S.thr.s;
        }
      }
    }
    trace_mark(g_trace, 3);
    return;
  }
  const int kept0 = topk_select(S, k);
  write_keys(S, kept0, k, block_out + (int64_t)blockIdx.x * k);
  trace_mark(g_trace, 3);

  // ---- level 1: last block of the group merges the group's lists
  const int g = blockIdx.x / TK_GROUP;
  const int ngroups = (gridDim.x + TK_GROUP - 1) / TK_GROUP;
  const int gsize = min(TK_GROUP, (int)gridDim.x - g * TK_GROUP);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(&tickets[g], 1u);
  __syncthreads();
  if (s_ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  int kept = merge_into(S, block_out + (int64_t)g * TK_GROUP * k, (int64_t)gsize * k, k, false);
  write_keys(S, kept, k, group_out + (int64_t)g * k);
  trace_mark(g_trace, 4);
  // ---- level 2: last group merger writes the final list
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(&tickets[ngroups], 1u);
  __syncthreads();
  if (s_ticket != (unsigned)(ngroups - 1)) return;
  __threadfence();
  kept = merge_into(S, group_out, (int64_t)ngroups * k, k, false);
  write_sorted(S, kept, k, out_s, out_i);
  if (threadIdx.x == 0) {  // the count out; every counter back to zero for the next launch
    const unsigned long long v = atomicExch(wvalid, 0ull);
    if (n_valid) *n_valid = v;
    for (int q = 0; q <= ngroups; ++q) tickets[q] = 0;
    tickets[TK_DYN_CTR] = 0;
  }
  trace_mark(g_trace, 5);
}

// Merge m keys (any order, +inf padded) into the k best, written as (score, index).
// Input either packed keys (in) or parallel (score, index) lists (idx < 0 = empty slot),
// converted on the fly: no staging buffer.
__global__ void __launch_bounds__(TPB) merge_keys_kernel(const Key* __restrict__ in, const double* __restrict__ in_s,
                                                         const int64_t* __restrict__ in_i, int64_t m, int k,
                                                         double* __restrict__ out_s, int64_t* __restrict__ out_i,
                                                         int cap) {
  extern __shared__ __align__(16) unsigned char raw[];
  TopkState& S = *reinterpret_cast<TopkState*>(raw);
  topk_init(S, cap);
  int safe = 1;
  for (int64_t base = 0; base < m; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool has = false;
    Key key;
    if (i < m) {
      if (in) {
        key = in[i];
        has = !(key.s == KEY_INF_S && key.i == KEY_INF_I);
      } else {
        key.i = in_i[i];
        has = key.i >= 0;
        key.s = has ? order_bits(in_s[i]) : KEY_INF_S;
      }
    }
    topk_offer(S, has, key, k, safe);
  }
  __syncthreads();
  write_sorted(S, topk_select(S, k), k, out_s, out_i);
}

__global__ void lists_to_keys_kernel(const double* __restrict__ s, const int64_t* __restrict__ idx, int64_t m,
                                     Key* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  Key k;
  if (idx[i] < 0) {
    k.s = KEY_INF_S;
    k.i = KEY_INF_I;
  } else {
    k.s = order_bits(s[i]);
    k.i = idx[i];
  }
  out[i] = k;
}

// Body-replication factor of every transformable record (U_inner, or all
// unrolled extents when no loop branches), into an open-addressing set.
__global__ void __launch_bounds__(TPB) collect_unroll_kernel(const DTask* __restrict__ gtask,
                                                             const ls_record* __restrict__ recs, int64_t n,
                                                             unsigned long long* __restrict__ set, int cap) {
  extern __shared__ __align__(16) unsigned char dyn[];
  DTask& T = *reinterpret_cast<DTask*>(dyn);
  stage_task(T, gtask);
  Cand c = carve(dyn + T.task_bytes, T);
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    const ls_record r = load_record(recs, i);
    if (apply_transforms(T, r, c)) continue;
    int64_t R = 1, Uin = 1;
    int k = 0;
    for (int p = 0; p < c.n; ++p) {
      const uint8_t fl = c.Fl(c.C(p));
      if (fl & F_VEC) continue;
      if (fl & F_UNR) {
        R *= c.E(c.C(p));
        Uin *= c.E(c.C(p));
      } else {
        Uin = 1;
        ++k;
      }
    }
    const unsigned long long key = (unsigned long long)(k ? Uin : R);
    unsigned int h = (unsigned int)((key * 0x9E3779B97F4A7C15ull) >> 40) % (unsigned)cap;
    int probe = 0;
    for (; probe < cap; ++probe) {
      const unsigned long long prev = atomicCAS(&set[h], 0ull, key);
      if (prev == 0ull || prev == key) break;
      h = (h + 1) % (unsigned)cap;
    }
    if (probe == cap) atomicExch(&set[cap], 1ull);  // set full: reported, never dropped silently
  }
}

// ---------------------------------------------------------------------------
// host: task construction
// ---------------------------------------------------------------------------
namespace {

struct HTerm {
  int var;
  int64_t coef;
  uint32_t req;
};

constexpr int64_t TAB_MAX_ENTRIES = 1 << 22;  // 16 MiB of int32 counts per task
constexpr int64_t TT_MAX_ENTRIES = 1 << 21;   // 16 MiB of uint64 footprints per task

// Record params / enable bits that can change each slot's extent/step
// (Tile/Vectorize on the slot or on the loop it was split from).
void slot_deps(const DTask& T, uint32_t* dep_p, uint32_t* dep_b, int64_t* ub, int64_t* pbound) {
  for (int v = 0; v < NSLOT; ++v) dep_p[v] = dep_b[v] = 0, ub[v] = 0;
  for (int q = 0; q < LS_MAX_PARAMS; ++q) pbound[q] = 0;
  for (int p = 0; p < T.n_base; ++p) ub[T.base_slot[p]] = T.base_ext[p];
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.kind != LS_XF_TILE && xf.kind != LS_XF_VECTORIZE) continue;
    if (xf.slot == NOSLOT || xf.new_slot == NOSLOT) continue;  // always fails
    const uint32_t pm = xf.param >= 0 ? (1u << xf.param) : 0u;
    const uint32_t bm = xf.enable_bit >= 0 ? (1u << xf.enable_bit) : 0u;
    dep_p[xf.slot] |= pm;
    dep_b[xf.slot] |= bm;
    dep_p[xf.new_slot] = dep_p[xf.slot];
    dep_b[xf.new_slot] = dep_b[xf.slot];
    if (xf.param >= 0) pbound[xf.param] = std::max(pbound[xf.param], ub[xf.slot]);
    ub[xf.new_slot] = ub[xf.slot];
  }
}

// dependencies of dimension D (4x4 layout): its variables' slots + its optional terms
void dim_deps(const DTask& T, int D, const uint32_t* dep_p, const uint32_t* dep_b, uint32_t& pm, uint32_t& bm) {
  const int t = D / 4, rr = D % 4;
  pm = bm = 0;
  for (int x = 0; x < T.dim_nv[D]; ++x) {
    pm |= dep_p[T.dim_var[D][x]];
    bm |= dep_b[T.dim_var[D][x]];
  }
  for (int a = 0; a < T.t_nu[t]; ++a) {
    const DExpr& e = T.expr[T.t_uacc[t][a]][rr];
    for (int z = 0; z < e.nt; ++z) bm |= T.term[e.t0 + z].req;
  }
}

// Tensor tables for the points path: key = the choices of the space axes that
// can change one of the tensor's dimension counts (mixed radix), row = all of
// the tensor's stage bits.  Needs the dimension-table plan (T.fast).
bool plan_tensor_tables(DTask& T) {
  T.tt_len = 0;
  if (!T.fast || T.sp_n < 1 || T.n_tensors > 4) return false;
  uint32_t dep_p[NSLOT], dep_b[NSLOT];
  int64_t ub[NSLOT], pbound[LS_MAX_PARAMS];
  slot_deps(T, dep_p, dep_b, ub, pbound);
  int64_t off = 0;
  for (int t = 0; t < 4; ++t) {
    T.tt_off[t] = T.tt_len_t[t] = T.tt_nb[t] = T.tt_sh[t] = T.tt_mk[t] = 0;
    for (int a = 0; a < LS_MAX_AXES; ++a) T.tt_stride[t][a] = 0;
    if (t >= T.n_tensors) continue;
    uint32_t pm = 0, bm = 0;
    int nb = 0;
    for (int rr = 0; rr < T.t_rank[t]; ++rr) {
      uint32_t p, b;
      dim_deps(T, t * 4 + rr, dep_p, dep_b, p, b);
      pm |= p;
      bm |= b;
      nb += T.dim_nv[t * 4 + rr];
    }
    if (nb > 20) return false;
    int64_t keys = 1;
    for (int a = T.sp_n - 1; a >= 0; --a) {
      const DAxis& ax = T.sp_ax[a];
      const bool hit = ((ax.kind == LS_AX_PARAM || ax.kind == LS_AX_VEC) && ((pm >> ax.param) & 1u)) ||
                       ((ax.kind == LS_AX_VEC || ax.kind == LS_AX_BIT) && ((bm >> ax.bit) & 1u));
      if (!hit) continue;
      T.tt_stride[t][a] = (uint32_t)keys;
      keys *= ax.n;
      if (keys > TT_MAX_ENTRIES) return false;
    }
    const int64_t len = keys << nb;
    if (off + len > TT_MAX_ENTRIES) return false;
    T.tt_off[t] = (uint32_t)off;
    T.tt_len_t[t] = (uint32_t)len;
    T.tt_nb[t] = (uint32_t)nb;
    T.tt_sh[t] = (uint32_t)T.dim_base[t * 4];
    T.tt_mk[t] = ((1u << nb) - 1u) << 3;

    off += len;
  }
  T.tt_len = (int32_t)off;
  return off > 0;
}
constexpr int64_t TAB_SMEM_MAX_BYTES = 16384;

// Eligibility of the space-specialised points path: unconditional
// tiles on existing loops, then at most one reorder; tile-factor and reorder axes
// only; no unroll/vector marks, shared tensors or optional terms.  pax: the
// reorder axis (-1: none).
bool plan_space(DTask& T, int& pax) {
  pax = -1;
  if (!T.fast || T.tt_len <= 0 || T.has_shared || T.has_optional || T.base_unr || T.base_vec) return false;
  if (T.family == LS_FAMILY_GPU && !T.costs_integral) return false;
  uint32_t exist = T.base_exist;
  int ntile = 0, last_tile = -1, reorder = -1;
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.enable_bit >= 0) return false;
    if (xf.kind == LS_XF_TILE) {
      if (xf.slot == NOSLOT || xf.new_slot == NOSLOT || !((exist >> xf.slot) & 1u) || ((exist >> xf.new_slot) & 1u))
        return false;
      exist |= 1u << xf.new_slot;
      ++ntile;
      last_tile = x;
    } else if (xf.kind == LS_XF_REORDER) {
      if (reorder >= 0) return false;
      reorder = x;
    } else {
      return false;
    }
  }
  if (reorder >= 0 && reorder < last_tile) return false;
  if (T.n_base + ntile > MAXCH) return false;
  for (int a = 0; a < T.sp_n; ++a) {
    if (T.sp_ax[a].kind == LS_AX_PERM) {
      if (pax >= 0) return false;
      pax = a;
    } else if (T.sp_ax[a].kind != LS_AX_PARAM) {
      return false;
    }
  }
  T.sp_nchain = T.n_base + ntile;
  return true;
}

constexpr int64_t SD_MAX_ENTRIES = 8192;  // 32 KiB of shared memory

// Static tiles of the space path: every Tile is driven by exactly one tile axis
// and splits a base loop that no earlier Tile split, so each choice fixes the
// inner extent F and the outer extent ceil(E/F) (ls/ir.py:361-382) and whether
// F is out of range.  ext[voff + c] per choice of the tile axes (indexed like
// sp_vals; other axes' entries unused).
void plan_static_tiles(DTask& T, const ls_space_desc* sp, std::vector<uint64_t>& ext) {
  T.sp_static = 0;
  int ntile = 0;
  for (int x = 0; x < T.n_xf; ++x) ntile += T.xf[x].kind == LS_XF_TILE;
  uint32_t split = 0;  // base slots already split
  int covered = 0;
  size_t nvals = 0;
  for (int a = 0; a < sp->n_axes; ++a) nvals += sp->axes[a].kind == LS_AX_BIT ? 0 : sp->axes[a].n_choices;
  ext.assign(std::max<size_t>(1, nvals), 0);
  for (int x = 0; x < T.n_xf; ++x) {
    const DXform& xf = T.xf[x];
    if (xf.kind != LS_XF_TILE) continue;
    if (xf.param < 0) return;
    int axis = -1, naxes = 0;
    for (int a = 0; a < T.sp_n; ++a)
      if (T.sp_ax[a].kind == LS_AX_PARAM && T.sp_ax[a].param == xf.param) axis = a, ++naxes;
    if (naxes != 1) return;
    int base = -1;
    for (int p = 0; p < T.n_base; ++p)
      if (T.base_slot[p] == xf.slot) base = p;
    if (base < 0 || ((split >> xf.slot) & 1u)) return;
    split |= 1u << xf.slot;
    const int64_t Ev = T.base_ext[base];
    const DAxis& ax = T.sp_ax[axis];
    for (uint32_t c = 0; c < ax.n; ++c) {
      const int64_t F = (int64_t)sp->axes[axis].values[c];
      const bool bad = F < 1 || F > Ev;
      const int64_t outer = bad ? 1 : (Ev + F - 1) / F;
      ext[ax.voff + c] = (uint64_t)(F & 0xFFFF) | ((uint64_t)outer << 16) | (bad ? (1ull << 63) : 0ull);
    }
    T.sp_tslot[axis] = xf.slot;
    T.sp_tnew[axis] = xf.new_slot;
    ++covered;
  }
  T.sp_n_untiled = 0;
  for (int p = 0; p < T.n_base; ++p)
    if (!((split >> T.base_slot[p]) & 1u)) {
      T.sp_untiled[T.sp_n_untiled] = T.base_slot[p];
      T.sp_untiled_pos[T.sp_n_untiled++] = (uint8_t)p;
    }
  for (int a = 0; a < T.sp_n; ++a) {  // every tile axis must drive a tile
    if (T.sp_ax[a].kind != LS_AX_PARAM) continue;
    bool used = false;
    for (int x = 0; x < T.n_xf; ++x) used |= T.xf[x].kind == LS_XF_TILE && T.xf[x].param == T.sp_ax[a].param;
    if (!used) return;
  }
  T.sp_static = covered == ntile ? 1 : 0;
}

// Group tables of the space path.  Every tensor's dimensions
// whose count can vary are split into at most two groups (one when the whole
// tensor fits), each with a table of 64-entry rows (stage mask <= 6 bits) keyed
// by the choices of the tile axes that can change one of its dimensions; the
// split minimising the entries is taken.  rows[g] = row count of group slot g.
bool plan_space_groups(DTask& T, int32_t* rows) {
  uint32_t dep_p[NSLOT], dep_b[NSLOT];
  int64_t ub[NSLOT], pb[LS_MAX_PARAMS];
  slot_deps(T, dep_p, dep_b, ub, pb);
  memset(T.sd_S, 0, sizeof(T.sd_S));
  memset(T.vb8, 0, sizeof(T.vb8));
  memset(T.sd_gd, -1, sizeof(T.sd_gd));
  memset(T.sd_gx, 0, sizeof(T.sd_gx));
  memset(T.sd_nb, 0, sizeof(T.sd_nb));
  for (int g = 0; g < 8; ++g) T.sd_off[g] = 0, rows[g] = 0;
  if (T.n_tensors > 4) return false;
  int64_t off = 4;  // entries 0..3: the ones row
  for (int t = 0; t < T.n_tensors; ++t) {
    int dims[4], nd = 0;
    uint32_t pmask[4];
    for (int rr = 0; rr < T.t_rank[t]; ++rr) {
      const int D = t * 4 + rr;
      bool varies = false;
      for (int x = 0; x < T.dim_nv[D]; ++x) varies |= ub[T.dim_var[D][x]] > 1;
      if (!varies && T.dim_count0[D] == 1) continue;  // the count stays 1
      uint32_t pm, bm;
      dim_deps(T, D, dep_p, dep_b, pm, bm);
      pmask[nd] = pm;
      dims[nd++] = D;
    }
    // choose the split (bit j of `sel`: dimension j goes to group 1) with the fewest entries
    int64_t best = -1;
    int best_sel = 0;
    for (int sel = 0; sel < (1 << nd); ++sel) {
      if (nd && (sel >> (nd - 1)) & 1) continue;  // symmetric splits: the last dimension stays in group 0
      int64_t total = 0;
      bool ok = true;
      for (int j = 0; j < 2 && ok; ++j) {
        uint32_t pm = 0;
        int nb = 0, members = 0;
        for (int q = 0; q < nd; ++q)
          if (((sel >> q) & 1) == j) pm |= pmask[q], nb += T.dim_nv[dims[q]], ++members;
        if (!members) continue;
        if (nb > 6) ok = false;
        int64_t keys = 1;
        for (int a = 0; a < T.sp_n && ok; ++a)
          if (T.sp_ax[a].kind == LS_AX_PARAM && ((pm >> T.sp_ax[a].param) & 1u)) keys *= T.sp_ax[a].n;
        total += keys << nb;
        if (total > SD_MAX_ENTRIES) ok = false;
      }
      if (ok && (best < 0 || total < best)) best = total, best_sel = sel;
    }
    if (best < 0) return false;
    for (int j = 0; j < 2; ++j) {
      const int G = 2 * t + j;
      uint32_t pm = 0;
      int nb = 0, m = 0;
      for (int q = 0; q < nd; ++q) {
        if (((best_sel >> q) & 1) != j) continue;
        const int D = dims[q];
        T.sd_gd[G][m] = (int8_t)D;
        T.sd_gx[G][m] = (int8_t)nb;
        for (int x = 0; x < T.dim_nv[D]; ++x) T.vb8[T.dim_var[D][x]] |= 1ull << (8 * G + 2 + nb + x);
        nb += T.dim_nv[D];
        pm |= pmask[q];
        ++m;
      }
      if (!m) continue;
      T.sd_nb[G] = (int8_t)nb;
      int64_t keys = 1;
      for (int a = T.sp_n - 1; a >= 0; --a) {
        const DAxis& ax = T.sp_ax[a];
        if (ax.kind != LS_AX_PARAM || !((pm >> ax.param) & 1u)) continue;
        T.sd_S[a][G] = (uint32_t)((keys << nb) * 4);
        keys *= ax.n;
      }
      if (off + (keys << nb) > SD_MAX_ENTRIES) return false;
      T.sd_off[G] = (uint32_t)(off * 4);
      rows[G] = (int32_t)keys;
      off += keys << nb;
    }
  }
  T.sd_len = (int32_t)off;
  return true;
}

// Decide whether the task can use the tabulated path and lay out its table
// (DESIGN.md §3.5).  A dimension's key is every record field that can change
// the extent/step of one of its variables (Tile/Vectorize factors applied to
// the variable or its ancestors, and their enable bits) plus the enable bits
// of its optional terms.
void plan_tabulated(const ls_task_desc& d, DTask& T, int RM, const std::vector<int64_t>& count_bound) {
  T.fast = 0;
  T.tab_len = 0;
  if (RM != 4 || T.n_stage + 3 > 64) return;
  for (int t = 0; t < T.n_tensors; ++t) {  // footprints are unsigned 64-bit products on this path
    double b = 1.0;
    for (int rr = 0; rr < T.t_rank[t]; ++rr) b *= (double)count_bound[t * RM + rr];
    if (b >= 9.0e18) return;
  }
  uint32_t dep_p[NSLOT], dep_b[NSLOT];
  int64_t ub[NSLOT], bound[LS_MAX_PARAMS];
  slot_deps(T, dep_p, dep_b, ub, bound);
  for (int q = 0; q < LS_MAX_PARAMS; ++q) T.fk_bound[q] = (int32_t)bound[q];
  int64_t off = 0;
  for (int D = 0; D < 16; ++D) {
    T.ftab_off[D] = 0;
    T.ftab_len[D] = 0;
    T.fk_n[D] = 0;
    const int t = D / 4, rr = D % 4;
    T.fsel[D] = 0;
    if (t >= T.n_tensors || rr >= T.t_rank[t]) continue;  // points at the constant-1 entry (below)
    uint32_t pm, bm;
    const int nv = T.dim_nv[D];
    dim_deps(T, D, dep_p, dep_b, pm, bm);
    int64_t len = 1;
    int nd = 0;
    for (int q = 0; q < LS_MAX_PARAMS; ++q) {
      if (!((pm >> q) & 1u)) continue;
      if (nd == 3) return;
      T.fk_src[D][nd] = (int8_t)q;
      T.fk_rad[D][nd] = (int32_t)(bound[q] + 1);
      len *= bound[q] + 1;
      ++nd;
      if (len > TAB_MAX_ENTRIES) return;
    }
    for (int b = 0; b < 24; ++b) {
      if (!((bm >> b) & 1u)) continue;
      if (nd == 3) return;
      T.fk_src[D][nd] = (int8_t)(LS_MAX_PARAMS + b);
      T.fk_rad[D][nd] = 2;
      len *= 2;
      ++nd;
    }
    if (bm >> 24) return;  // enable bits >= 24 do not fit the key encoding
    len <<= nv;
    if (off + len > TAB_MAX_ENTRIES) return;
    T.fk_n[D] = (int8_t)nd;
    T.ftab_off[D] = (int32_t)off;
    T.ftab_len[D] = (int32_t)len;
    // stage bits sit at dim_base + 3 + x, so (mall >> (dim_base + 1)) & (mask << 2) is a byte offset
    T.fsel[D] = (uint32_t)(T.dim_base[D] + 1) | ((((1u << nv) - 1u) << 2) << 8);
    off += len;
  }
  T.tab_one = (int32_t)off++;  // the count of a dimension slot the layout does not use: 1
  for (int D = 0; D < 16; ++D)
    if (T.ftab_len[D] == 0) T.ftab_off[D] = T.tab_one;
  for (int v = 0; v < NSLOT; ++v) T.vbits[v] = 0;
  for (int D = 0; D < 16; ++D)
    for (int x = 0; x < T.dim_nv[D]; ++x) T.vbits[T.dim_var[D][x]] |= 1ull << (T.dim_base[D] + 3 + x);
  T.chain0 = ~0ull;
  T.base_exist = T.base_unr = T.base_vec = T.base_par = 0;
  for (int p = 0; p < T.n_base; ++p) {
    const int v = T.base_slot[p];
    T.chain0 = (T.chain0 & ~(15ull << (4 * p))) | ((uint64_t)v << (4 * p));
    T.base_exist |= 1u << v;
    if (T.base_flags[p] & F_UNR) T.base_unr |= 1u << v;
    if (T.base_flags[p] & F_VEC) T.base_vec |= 1u << v;
    if (T.base_flags[p] & F_PAR) T.base_par |= 1u << v;
  }
  T.tab_len = (int32_t)off;
  T.tab_smem = (int64_t)sizeof(int32_t) * off <= TAB_SMEM_MAX_BYTES ? 1 : 0;
  T.fast = 1;
}

int build_task(const ls_task_desc& d, DTask& T, std::vector<int>& load_t, std::vector<int>& store_t) {
  memset(&T, 0, sizeof(T));
  if (d.abi_version != LS_ABI_VERSION) return fail(LS_E_ARG, "abi_version mismatch");
  if (d.n_nodes <= 0 || d.n_nodes > LS_MAX_NODES || d.n_tensors < 1 || d.n_tensors > LS_MAX_TENSORS ||
      d.n_vars < 1 || d.n_vars > LS_MAX_VARS || d.n_xforms < 0 || d.n_xforms > LS_MAX_XFORMS)
    return fail(LS_E_ARG, "descriptor counts out of range");
  if (!((d.family == LS_FAMILY_CPU && (d.target == LS_TARGET_X86 || d.target == LS_TARGET_AARCH64)) ||
        (d.family == LS_FAMILY_GPU && d.target == LS_TARGET_PTX)))
    return fail(LS_E_UNSUPPORTED, "family/target combination not supported");
  // ---- loops and accesses in preorder; a perfect chain (loops 0..L-1 each the only child
  //      of the previous, every access under the last) takes the chain kernels, any other
  //      tree the tree kernel
  std::vector<int> loop_nodes, acc_nodes;
  for (int i = 0; i < d.n_nodes; ++i) {
    if (d.nodes[i].parent < -1 || d.nodes[i].parent >= i) return fail(LS_E_ARG, "nodes must be in preorder");
    if (d.nodes[i].parent >= 0 && d.nodes[d.nodes[i].parent].kind != LS_NODE_LOOP)
      return fail(LS_E_ARG, "parent of a node must be a loop");
    (d.nodes[i].kind == LS_NODE_LOOP ? loop_nodes : acc_nodes).push_back(i);
  }
  const int nl = (int)loop_nodes.size(), na = (int)acc_nodes.size();
  bool chain = nl >= 1;
  for (int p = 0; p < nl && chain; ++p) chain = loop_nodes[p] == p && d.nodes[p].parent == p - 1;
  for (int a = 0; a < na && chain; ++a) chain = d.nodes[acc_nodes[a]].parent == nl - 1;
  T.tree = chain ? 0 : 1;
  if (nl == 0 || nl > MAXCH) return fail(LS_E_UNSUPPORTED, "program must have 1..16 loops");
  if (na < 1 || na > MAXACC) return fail(LS_E_UNSUPPORTED, "program must hold 1..16 accesses");
  if (T.tree) {  // inlined loops: the emission is emulated per candidate
    for (int p = 0; p < nl; ++p)
      if (d.nodes[loop_nodes[p]].unrolled || d.nodes[loop_nodes[p]].vector_width) T.tr_inline = 1;
    for (int x = 0; x < d.n_xforms; ++x)
      if (d.xforms[x].kind == LS_XF_UNROLL || d.xforms[x].kind == LS_XF_VECTORIZE) T.tr_inline = 1;
  }
  for (int x = 0; x < d.n_xforms; ++x) {
    const ls_xform& s = d.xforms[x];
    if (s.var >= d.n_vars || s.new_var >= d.n_vars || s.param >= LS_MAX_PARAMS || s.enable_bit >= 32 ||
        s.n_order < 0 || s.n_order > LS_MAX_ORDER || s.perm_shift < 0 || s.perm_shift + s.n_order > 16)
      return fail(LS_E_ARG, "bad transform slot");
  }
  // ---- variable slots: only names that can exist (base loops and tile/vectorize inner loops)
  std::vector<int> slot_of(LS_MAX_VARS, NOSLOT);
  int ns = 0;
  auto add_slot = [&](int v) {
    if (v >= 0 && slot_of[v] == NOSLOT) slot_of[v] = ns++;
  };
  for (int p = 0; p < nl; ++p) add_slot(d.nodes[loop_nodes[p]].var);
  for (int x = 0; x < d.n_xforms; ++x)
    if ((d.xforms[x].kind == LS_XF_TILE || d.xforms[x].kind == LS_XF_VECTORIZE) && d.xforms[x].var >= 0)
      add_slot(d.xforms[x].new_var);
  if (ns > NSLOT) return fail(LS_E_UNSUPPORTED, "transformed chain could exceed 16 loops");
  auto S_ = [&](int v) -> uint8_t { return v < 0 ? NOSLOT : (uint8_t)slot_of[v]; };

  T.n_base = nl;
  std::vector<int64_t> span(LS_MAX_VARS, 0);  // step * extent of each variable's base loop
  int ntile = 0;
  for (int p = 0; p < nl; ++p) {
    const ls_node& n = d.nodes[loop_nodes[p]];
    if (n.var < 0 || n.var >= d.n_vars || n.extent < 1 || n.step < 1 || n.extent >= (1 << 30) ||
        n.step >= (1 << 30))
      return fail(LS_E_ARG, "bad loop node");
    T.base_slot[p] = S_(n.var);
    T.base_ext[p] = n.extent;
    T.base_step[p] = n.step;
    T.base_flags[p] = (uint8_t)((n.parallel ? F_PAR : 0) | (n.unrolled ? F_UNR : 0) | (n.vector_width ? F_VEC : 0));
    span[n.var] = (int64_t)n.step * n.extent;
  }
  T.n_xf = d.n_xforms;
  for (int x = 0; x < d.n_xforms; ++x) {
    const ls_xform& s = d.xforms[x];
    DXform& o = T.xf[x];
    o.kind = (int8_t)s.kind;
    o.slot = S_(s.var);
    o.new_slot = (s.kind == LS_XF_TILE || s.kind == LS_XF_VECTORIZE) && s.var >= 0 ? S_(s.new_var) : NOSLOT;
    o.param = (int8_t)s.param;
    o.value = s.value;
    o.enable_bit = (int8_t)s.enable_bit;
    o.n_order = (int8_t)s.n_order;
    o.perm_shift = (int8_t)s.perm_shift;
    for (int j = 0; j < s.n_order; ++j) o.order[j] = S_(s.order[j]);
    if (s.kind == LS_XF_TILE || s.kind == LS_XF_VECTORIZE) ++ntile;
  }
  // ---- symbolic expression rewrite: final term lists with enable requirements
  // (_rewrite_exprs ls/ir.py:350-358 applied for every Tile/Vectorize of the template)
  std::vector<std::vector<std::vector<HTerm>>> ex(na);
  for (int a = 0; a < na; ++a) {
    const ls_node& n = d.nodes[acc_nodes[a]];
    if (n.tensor < 0 || n.tensor >= d.n_tensors) return fail(LS_E_ARG, "bad tensor index");
    const int rank = d.tensors[n.tensor].rank;
    if (rank < 1 || rank > MAXRANK) return fail(LS_E_ARG, "bad rank");
    ex[a].resize(rank);
    for (int k = 0; k < rank; ++k)
      for (int t = 0; t < n.idx[k].n_terms; ++t) {
        const int v = n.idx[k].terms[t].var;
        if (v < 0 || v >= d.n_vars || slot_of[v] == NOSLOT) return fail(LS_E_ARG, "index term on a non-loop var");
        ex[a][k].push_back({v, n.idx[k].terms[t].coef, 0u});
      }
  }
  for (int x = 0; x < d.n_xforms; ++x) {
    const ls_xform& s = d.xforms[x];
    if (s.kind != LS_XF_TILE && s.kind != LS_XF_VECTORIZE) continue;
    if (s.var < 0 || s.new_var < 0) continue;  // target never exists: every candidate fails there
    const uint32_t bit = s.enable_bit >= 0 ? (1u << s.enable_bit) : 0u;
    span[s.new_var] = span[s.var];
    for (auto& acc : ex)
      for (auto& e : acc) {
        std::vector<HTerm> add;
        for (auto& t : e)
          if (t.var == s.var) add.push_back({s.new_var, t.coef, t.req | bit});
        for (auto& t : add) e.push_back(t);
      }
  }
  int nt = 0;
  std::vector<std::vector<int64_t>> ebound(na, std::vector<int64_t>(MAXRANK, 0));
  for (int a = 0; a < na; ++a) {
    const ls_node& n = d.nodes[acc_nodes[a]];
    T.acc_tensor[a] = (uint8_t)n.tensor;
    T.acc_store[a] = (uint8_t)n.is_store;
    for (size_t k = 0; k < ex[a].size(); ++k) {
      auto& e = ex[a][k];
      std::stable_sort(e.begin(), e.end(),
                       [&](const HTerm& x, const HTerm& y) { return d.var_rank[x.var] < d.var_rank[y.var]; });
      // |value| <= |konst| + sum |coef| * step * (extent - 1); tiling keeps step*extent
      // below 2x its previous value, so 2^(tiles+1) bounds every candidate
      int64_t bound = std::llabs((int64_t)n.idx[k].konst);
      for (auto& t : e) bound += std::llabs(t.coef) * span[t.var] * (2ll << ntile);
      if (bound >= (1ll << 30)) return fail(LS_E_UNSUPPORTED, "index range exceeds the device int32 model");
      ebound[a][k] = bound;
      if (nt + (int)e.size() > MAXTERM) return fail(LS_E_UNSUPPORTED, "too many index terms");
      T.expr[a][k].konst = n.idx[k].konst;
      T.expr[a][k].t0 = (int16_t)nt;
      T.expr[a][k].nt = (int16_t)e.size();
      for (auto& t : e) T.term[nt++] = {(int32_t)t.coef, t.req, (int32_t)slot_of[t.var]};
    }
  }
  T.n_terms = nt;
  T.n_acc = na;
  // ---- tensors in first-appearance order, deduplicated consecutive accesses
  std::vector<int> order;
  for (int a = 0; a < na; ++a)
    if (std::find(order.begin(), order.end(), (int)T.acc_tensor[a]) == order.end()) order.push_back(T.acc_tensor[a]);
  T.n_tensors = (int)order.size();
  int L = 0, S = 0;
  for (int a = 0; a < na; ++a) {
    if (T.acc_store[a]) {
      ++S;
      store_t.push_back(T.acc_tensor[a]);
    } else {
      ++L;
      load_t.push_back(T.acc_tensor[a]);
    }
  }
  T.L = L;
  T.S = S;
  int max_rank = 0;
  for (int t : order) max_rank = std::max(max_rank, (int)d.tensors[t].rank);
  const int RM = (T.n_tensors <= 4 && max_rank <= 4) ? 4 : MAXRANK;
  T.layout_rm = RM;
  for (int D = 0; D < MAXD; ++D) T.dim_count0[D] = 1;
  std::vector<int> decl_of(order.begin(), order.end());
  for (int a = 0; a < na; ++a)
    T.acc_tensor[a] = (uint8_t)(std::find(order.begin(), order.end(), (int)T.acc_tensor[a]) - order.begin());
  int n_stage = 0;
  for (int t = 0; t < T.n_tensors; ++t) {
    const ls_tensor& td = d.tensors[decl_of[t]];
    T.t_rank[t] = (uint8_t)td.rank;
    T.t_eb[t] = (uint8_t)td.elem_bytes;
    T.t_shared[t] = (uint8_t)(td.shared != 0);
    if (td.shared && d.family == LS_FAMILY_GPU) T.has_shared = 1;
    int64_t stride = 1;
    for (int k = td.rank - 1; k >= 0; --k) {
      T.t_stride[t][k] = stride;
      stride *= td.dims[k];
    }
    int nu = 0, last = -1;
    for (int a = 0; a < na; ++a) {
      if (T.acc_tensor[a] != t) continue;
      T.t_nacc[t]++;
      bool same = last >= 0;
      for (int k = 0; same && k < td.rank; ++k) {
        const ls_expr& x = d.nodes[acc_nodes[a]].idx[k];
        const ls_expr& y = d.nodes[acc_nodes[last]].idx[k];
        same = x.konst == y.konst && x.n_terms == y.n_terms &&
               memcmp(x.terms, y.terms, sizeof(ls_term) * x.n_terms) == 0;
      }
      if (!same) T.t_uacc[t][nu++] = (uint8_t)a;
      last = a;
    }
    T.t_nu[t] = (uint8_t)nu;
    for (int k = 0; k < td.rank; ++k) {
      const int D = t * RM + k;
      // nothing expanded: union of the accesses' constant points (ls/cache.py:80-96)
      int64_t lo = 0, hi = 0, str = 0, cnt = 1;
      bool exact = true;
      for (int q = 0; q < nu; ++q) {
        const int64_t v = T.expr[T.t_uacc[t][q]][k].konst;
        if (q == 0) {
          lo = hi = v;
          continue;
        }
        if (lo == v && hi == v && str == 0 && cnt == 1 && exact) continue;
        const int64_t nlo = std::min(lo, v), nhi = std::max(hi, v);
        auto gcd = [](int64_t a, int64_t b) {
          while (b) {
            int64_t t2 = a % b;
            a = b;
            b = t2;
          }
          return a;
        };
        const int64_t g = gcd(str, std::llabs(lo - v));
        const int64_t est = g ? (nhi - nlo) / g + 1 : 1;
        cnt = std::min(est, cnt + 1);
        lo = nlo;
        hi = nhi;
        str = g;
        exact = false;
      }
      T.dim_count0[D] = (int32_t)cnt;
      // the dimension's loop variables (any term of any of its accesses)
      int nv = 0;
      for (int q = 0; q < nu; ++q) {
        const DExpr& e = T.expr[T.t_uacc[t][q]][k];
        for (int z = 0; z < e.nt; ++z) {
          const int s = T.term[e.t0 + z].slot;
          bool have = false;
          for (int j = 0; j < nv; ++j) have |= T.dim_var[D][j] == s;
          if (have) continue;
          if (nv >= MAXDV) {
            if (T.tree) break;  // the chain kernels' per-dimension stages; unused on trees
            return fail(LS_E_UNSUPPORTED, "more than 8 loop variables in one tensor dimension");
          }
          T.dim_var[D][nv] = (uint8_t)s;
          T.slot_dnib[s][D / 16] |= (uint64_t)(nv + 1) << (4 * (D % 16));
          ++nv;
        }
      }
      T.dim_nv[D] = (uint8_t)nv;
      T.dim_base[D] = (uint8_t)n_stage;
      n_stage += nv;
    }
  }
  if (n_stage > MAXSTAGE && !T.tree) return fail(LS_E_UNSUPPORTED, "too many (dimension, variable) pairs");
  T.n_stage = n_stage;
  T.n_slots = ns;
  for (int q = 0; q < nt; ++q) T.has_optional |= T.term[q].req != 0;
  for (int a = 0; a < na; ++a)
    for (int k = 0; k < T.t_rank[T.acc_tensor[a]]; ++k)
      for (int z = 0; z < T.expr[a][k].nt; ++z)
        T.t_vmask[T.acc_tensor[a]] |= 1u << T.term[T.expr[a][k].t0 + z].slot;
  T.n_chain = std::min(MAXCH, nl + ntile);
  {  // |count| of a dimension <= hi - lo + 1 <= 2 * range bound + 1 (ls/cache.py:46-77)
    std::vector<int64_t> cb(MAXD, 1);
    for (int a = 0; a < na; ++a)
      for (int k = 0; k < T.t_rank[T.acc_tensor[a]]; ++k) {
        const int D = T.acc_tensor[a] * RM + k;
        cb[D] = std::max(cb[D], 2 * ebound[a][k] + 1);
      }
    if (!T.tree) plan_tabulated(d, T, RM, cb);
  }
  T.task_bytes = (int32_t)align16(offsetof(DTask, term) + sizeof(DTerm) * (size_t)nt);
  // ---- arch
  T.family = d.family;
  T.cap = d.cache_capacity;
  for (int q = 0; q < LS_NFEAT_GPU; ++q) T.coef[q] = d.coef[q];
  T.costs_integral = 1;
  for (int q = 0; q < LS_I_COUNT; ++q) {
    T.ptx_cost[q] = d.ptx_cost[q];
    const double c = d.ptx_cost[q];
    if (c != std::floor(c) || std::fabs(c) > 1e12) T.costs_integral = 0;
    T.ptx_icost[q] = (int64_t)c;
  }
  T.sm_underuse = d.sm_underuse;
  T.warp_slack = d.warp_slack;
  T.tid_slot = d.tid_var >= 0 && slot_of[d.tid_var] != NOSLOT ? slot_of[d.tid_var] : -1;
  T.banks = d.banks > 0 ? d.banks : 32;
  T.warp_size = d.warp_size > 0 ? d.warp_size : 32;
  if (T.banks > 64) return fail(LS_E_UNSUPPORTED, "more than 64 banks");
  if (d.family == LS_FAMILY_CPU) {
    if (d.issue_width < 1) return fail(LS_E_ARG, "issue_width < 1");
    for (int q = 0; q < LS_I_COUNT; ++q)
      if (d.klass[q] < 0 || d.klass[q] >= LS_I_COUNT) return fail(LS_E_ARG, "bad class id");
    lsb::fixed_block_cycles(d, &T.c_init, &T.c_latch, &T.c_ret);
  }
  if (T.tree) {  // ---- the base tree over unified ids and the per-loop access groups
    std::vector<int> id_of(d.n_nodes);
    for (int a = 0; a < na; ++a) id_of[acc_nodes[a]] = a;
    for (int p = 0; p < nl; ++p) id_of[loop_nodes[p]] = na + p;
    for (int i = 0; i < 32; ++i) T.tr_parent[i] = T.tr_first[i] = T.tr_next[i] = -1;
    T.tr_root_first = -1;
    std::vector<int> last_child(32, -1);
    int last_top = -1;
    for (int i = 0; i < d.n_nodes; ++i) {  // preorder: children appear in order
      const int id = id_of[i], par = d.nodes[i].parent;
      const int pid = par >= 0 ? id_of[par] : -1;
      T.tr_parent[id] = (int8_t)pid;
      int& prev = pid >= 0 ? last_child[pid] : last_top;
      if (prev < 0) {
        if (pid >= 0)
          T.tr_first[pid] = (int8_t)id;
        else
          T.tr_root_first = id;
      } else {
        T.tr_next[prev] = (int8_t)id;
      }
      prev = id;
    }
    T.tr_nl = nl;
    T.tr_na = na;
    for (int a = 0; a < na; ++a) T.acc_decl[a] = (uint8_t)d.nodes[acc_nodes[a]].tensor;
    T.tr_target = d.target;
    T.tr_dialect = d.dialect;
    T.tr_issue = d.issue_width;
    for (int q = 0; q < LS_I_COUNT; ++q) {
      T.tr_lat[q] = d.lat[q];
      T.tr_klass[q] = d.klass[q];
      T.tr_ucap[q] = d.unit_cap[q];
    }
    for (int p = 0; p < nl; ++p) {  // the group of base loop p: its direct accesses, loads then stores
      std::vector<int> lt, st;
      for (int a = 0; a < na; ++a)
        if (d.nodes[acc_nodes[a]].parent == loop_nodes[p])
          (d.nodes[acc_nodes[a]].is_store ? st : lt).push_back(d.nodes[acc_nodes[a]].tensor);
      T.tr_nld[p] = (uint8_t)lt.size();
      T.tr_nst[p] = (uint8_t)st.size();
      if (d.family == LS_FAMILY_CPU) {
        T.tr_c_hi[p] = lsb::group_block_cycles(d, lt, st, false);
        T.tr_c_hl[p] = lsb::group_block_cycles(d, lt, st, true);
      }
    }
  }
  return LS_E_OK;
}

int upload(ls_task* t) {
  DTask* dnew = nullptr;
  DUnroll* dtab = nullptr;
  CUDA_TRY(cudaMalloc(&dtab, sizeof(DUnroll) * std::max<size_t>(1, t->utab.size())));
  CUDA_TRY(cudaMemcpy(dtab, t->utab.data(), sizeof(DUnroll) * t->utab.size(), cudaMemcpyHostToDevice));
  t->host.u_tab = dtab;
  t->host.n_u = (int32_t)t->utab.size();
  for (const DUnroll& e : t->utab)
    if (e.u == 1) t->host.c_inner1 = e.c_inner;
  CUDA_TRY(cudaMalloc(&dnew, sizeof(DTask)));
  CUDA_TRY(cudaMemcpy(dnew, &t->host, sizeof(DTask), cudaMemcpyHostToDevice));
  if (t->d_task) t->retired.push_back(t->d_task);
  t->retired.push_back(dtab);
  t->d_task = dnew;
  return LS_E_OK;
}

// Body-replication products above this are outside the device class: their candidates report
// LS_ST_UNROLL_TABLE (the block of U body copies is list-scheduled on the host, O(U) instructions).
constexpr int64_t LS_UNROLL_MAX = 65536;

int add_unroll(ls_task* t, const int64_t* us, int n) {
  bool changed = false;
  for (int i = 0; i < n; ++i) {
    int64_t U = us[i];
    if (U < 1 || U > LS_UNROLL_MAX) continue;
    bool have = false;
    for (auto& e : t->utab) have |= e.u == U;
    if (have) continue;
    DUnroll e;
    e.u = U;
    if (t->desc.family == LS_FAMILY_CPU) {
      e.c_inner = lsb::body_block_cycles(t->desc, t->load_t, t->store_t, U, true);
      e.c_all = lsb::body_block_cycles(t->desc, t->load_t, t->store_t, U, false);
    } else {
      e.c_inner = e.c_all = 0;
    }
    t->utab.push_back(e);
    changed = true;
  }
  if (!changed && t->d_task) return LS_E_OK;
  std::sort(t->utab.begin(), t->utab.end(), [](const DUnroll& a, const DUnroll& b) { return a.u < b.u; });
  return upload(t);
}

int grid_for(const ls_task* t, int64_t n, int per_sm) {
  const int64_t want = (n + TPB - 1) / TPB;
  const int64_t cap = (int64_t)t->num_sms * std::max(per_sm, 1);
  return (int)std::max<int64_t>(1, std::min(want, cap));
}

// 0 generic, 1 tabulated (table in global memory), 2 tabulated (table in shared memory),
// 3 tensor tables (points), 4 space-specialised (points)
int mode_of(const ls_task* t, bool points = false) {
  if (t->host.tree) return 6;
  if (t->path == LS_PATH_GENERIC || !t->host.fast) return 0;
  if (points && t->host.sp_ok && t->path != LS_PATH_TABULATED) return t->host.sp_narrow ? 5 : 4;
  if (points && t->host.tt_ok) return 3;
  return t->host.tab_smem ? 2 : 1;
}

size_t smem_score(const DTask& T, int mode) {
  return (size_t)T.task_bytes + tab_smem_bytes(mode, T) + state_bytes(mode, T.n_slots, T.n_chain, T.n_stage);
}
// the fused kernel's buffer must hold k plus one round of inserts
int topk_buf(int k) { return TOPK_CAP_SMALL && k <= 1024 - TPB ? 1024 : 2048; }
size_t smem_topk(const DTask& T, int k, int mode) { return smem_score(T, mode) + align16(topk_state_bytes(topk_buf(k))); }

using ScoreFn = void (*)(const DTask*, const void*, int, int64_t, double*, double*, int32_t*);
using TopkFn = void (*)(const DTask*, const void*, int, int64_t, int64_t, int, Key*, Key*, unsigned int*, double*,
                       int64_t*, unsigned long long*, int, Key*, unsigned long long*, unsigned long long*);

template <int SRC>
ScoreFn score_fn_src(const DTask& T, int mode) {
  if constexpr (SRC == 1) {
    if (mode == 4) {
      switch (T.n_tensors) {
        case 1: return score_kernel<1, 4, 4, 1>;
        case 2: return score_kernel<2, 4, 4, 1>;
        case 3: return score_kernel<3, 4, 4, 1>;
        default: return score_kernel<4, 4, 4, 1>;
      }
    }
    if (mode == 5) {
      switch (T.n_tensors) {
        case 1: return score_kernel<1, 4, 5, 1>;
        case 2: return score_kernel<2, 4, 5, 1>;
        case 3: return score_kernel<3, 4, 5, 1>;
        default: return score_kernel<4, 4, 5, 1>;
      }
    }
    if (mode == 3) return score_kernel<4, 4, 3, 1>;
  }
  if (mode == 6) return score_kernel<4, 4, 6, SRC>;
  if (mode == 1) return score_kernel<4, 4, 1, SRC>;
  if (mode == 2) return score_kernel<4, 4, 2, SRC>;
  return T.layout_rm == 4 ? score_kernel<4, 4, 0, SRC> : score_kernel<MAXT, MAXRANK, 0, SRC>;
}
template <int SRC>
TopkFn topk_fn_src(const DTask& T, int mode) {
  if constexpr (SRC == 1) {
    if (mode == 4) {
      switch (T.n_tensors) {
        case 1: return score_topk_kernel<1, 4, 4, 1>;
        case 2: return score_topk_kernel<2, 4, 4, 1>;
        case 3: return score_topk_kernel<3, 4, 4, 1>;
        default: return score_topk_kernel<4, 4, 4, 1>;
      }
    }
    if (mode == 5) {
      switch (T.n_tensors) {
        case 1: return score_topk_kernel<1, 4, 5, 1>;
        case 2: return score_topk_kernel<2, 4, 5, 1>;
        case 3: return score_topk_kernel<3, 4, 5, 1>;
        default: return score_topk_kernel<4, 4, 5, 1>;
      }
    }
    if (mode == 3) return score_topk_kernel<4, 4, 3, 1>;
  }
  if (mode == 6) return score_topk_kernel<4, 4, 6, SRC>;
  if (mode == 1) return score_topk_kernel<4, 4, 1, SRC>;
  if (mode == 2) return score_topk_kernel<4, 4, 2, SRC>;
  return T.layout_rm == 4 ? score_topk_kernel<4, 4, 0, SRC> : score_topk_kernel<MAXT, MAXRANK, 0, SRC>;
}
ScoreFn score_fn(const DTask& T, int mode, int pbytes) {
  return pbytes ? score_fn_src<1>(T, mode) : score_fn_src<0>(T, mode);
}
TopkFn topk_fn(const DTask& T, int mode, int pbytes) {
  return pbytes ? topk_fn_src<1>(T, mode) : topk_fn_src<0>(T, mode);
}

// Dynamic shared-memory limit and resident blocks per SM of a kernel on the
// current device (cached per (device, kernel): the attribute and occupancy
// queries cost host time on every scoring call).  cudaFuncSetAttribute acts on
// the current device only, so each device gets its own entry.  The limit only
// ever grows, so a cached launch at a smaller size stays valid after a larger
// one.  Returns -1 (with ls_last_error set) when the attribute cannot be set.
struct KernAttr {
  int device;
  const void* fn;
  size_t limit;                                  // MaxDynamicSharedMemorySize set so far
  std::vector<std::pair<size_t, int>> occ;       // (dynamic smem, blocks per SM)
};
template <typename K>
int kernel_prepare(K kernel, size_t smem, bool want_occupancy) {
  static std::mutex mu;
  static std::vector<KernAttr> cache;
  const void* f = reinterpret_cast<const void*>(kernel);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(LS_E_CUDA, "cudaGetDevice failed"), -1;
  std::lock_guard<std::mutex> g(mu);
  KernAttr* e = nullptr;
  for (auto& c : cache)
    if (c.device == dev && c.fn == f) e = &c;
  if (!e) {
    cache.push_back({dev, f, 0, {}});
    e = &cache.back();
  }
  if (smem > e->limit) {
    const cudaError_t r = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r != cudaSuccess) {
      cudaGetLastError();
      return fail(LS_E_CUDA, std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize=") + std::to_string(smem) +
                                 "): " + cudaGetErrorString(r)),
             -1;
    }
    e->limit = smem;
  }
  if (!want_occupancy) return 1;
  for (auto& o : e->occ)
    if (o.first == smem) return o.second;
  int b = 0;
  const cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, TPB, smem);
  if (r != cudaSuccess) {
    cudaGetLastError();
    return fail(LS_E_CUDA, std::string("cudaOccupancyMaxActiveBlocksPerMultiprocessor: ") + cudaGetErrorString(r)), -1;
  }
  b = std::max(b, 1);
  e->occ.push_back({smem, b});
  return b;
}
template <typename K>
int blocks_per_sm(K kernel, size_t smem) {
  return kernel_prepare(kernel, smem, true);
}
#define BPS_TRY(var, kernel, smem)           \
  const int var = blocks_per_sm(kernel, smem); \
  if (var < 0) return LS_E_CUDA

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* ls_last_error(void) { return g_err.c_str(); }
int ls_abi_version(void) { return LS_ABI_VERSION; }

int ls_task_create(const ls_task_desc* desc, int device, ls_task** out) {
  if (!desc || !out) return fail(LS_E_ARG, "null argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  ls_task* t = new ls_task();
  t->desc = *desc;
  t->device = device;
  t->d_task = nullptr;
  int rc = build_task(*desc, t->host, t->load_t, t->store_t);
  if (rc) {
    delete t;
    return rc;
  }
  cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (t->host.tree) {  // the tree kernels recurse (emission replay, line-order PTX) and list-schedule in local memory
    size_t lim = 0;
    cudaDeviceGetLimit(&lim, cudaLimitStackSize);
    if (lim < 20480) CUDA_TRY(cudaDeviceSetLimit(cudaLimitStackSize, 20480));
  }
  {  // keep stream-ordered workspace allocations cached across calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  t->path = LS_PATH_AUTO;
  t->d_tab = nullptr;
  if (t->host.fast) {
    if (cudaMalloc(&t->d_tab, sizeof(int32_t) * std::max(1, t->host.tab_len)) != cudaSuccess) {
      delete t;
      return fail(LS_E_NOMEM, "cannot allocate the dimension-count table");
    }
    t->host.tab = t->d_tab;
  }
  int64_t one = 1;
  rc = add_unroll(t, &one, 1);
  if (rc == LS_E_OK && t->host.fast && t->host.tab_len > 0) {
    build_tab_kernel<<<(t->host.tab_len + 255) / 256, 256>>>(t->d_task, t->d_tab);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(LS_E_CUDA, std::string("build_tab_kernel: ") + cudaGetErrorString(e));
  }
  if (rc) {
    if (t->d_tab) cudaFree(t->d_tab);
    delete t;
    return rc;
  }
  *out = t;
  return LS_E_OK;
}

int ls_task_set_path(ls_task* t, int32_t path) {
  if (!t || path < LS_PATH_AUTO || path > LS_PATH_SPACE) return fail(LS_E_ARG, "bad argument");
  if ((path == LS_PATH_TABULATED || path == LS_PATH_SPACE) && !t->host.fast)
    return fail(LS_E_UNSUPPORTED, "task is not eligible for the tabulated path");
  t->path = path;
  return LS_E_OK;
}

int ls_task_path(const ls_task* t) {
  if (!t) return LS_E_ARG;
  const int m = mode_of(t);
  return (m >= 1 && m <= 3) ? LS_PATH_TABULATED : LS_PATH_GENERIC;
}

int ls_task_points_path(const ls_task* t) {
  if (!t) return LS_E_ARG;
  const int m = mode_of(t, true);
  return (m == 4 || m == 5) ? LS_PATH_SPACE : (m >= 1 && m <= 3) ? LS_PATH_TABULATED : LS_PATH_GENERIC;
}

int ls_task_destroy(ls_task* t) {
  if (!t) return LS_E_OK;
  cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  for (void* p : t->retired) cudaFree(p);
  if (t->d_task) cudaFree(t->d_task);
  if (t->d_tab) cudaFree(t->d_tab);
  if (t->stage) cudaFreeHost(t->stage);
  if (t->ws) cudaFree(t->ws);
  delete t;
  return LS_E_OK;
}

int ls_task_num_features(const ls_task* t) {
  return t ? (t->desc.family == LS_FAMILY_CPU ? LS_NFEAT_CPU : LS_NFEAT_GPU) : LS_E_ARG;
}

int ls_task_prepare_unroll(ls_task* t, const int64_t* u, int32_t n) {
  if (!t || (n && !u)) return fail(LS_E_ARG, "null argument");
  std::lock_guard<std::mutex> g(t->mu);
  CUDA_TRY(cudaSetDevice(t->device));
  return add_unroll(t, u, n);
}

int ls_collect_unroll(ls_task* t, const ls_record* d_records, int64_t n, int64_t* h_values, int32_t cap,
                      int32_t* h_count, void* stream) {
  if (!t || !h_values || !h_count || cap < 1) return fail(LS_E_ARG, "bad argument");
  if (t->host.tree) {  // no Unroll on the tree path: nothing to prepare
    *h_count = 0;
    return LS_E_OK;
  }
  CUDA_TRY(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int slots = 16384;  // distinct products per batch; one more slot flags a full set
  unsigned long long* set = nullptr;
  CUDA_TRY(cudaMallocAsync(&set, sizeof(unsigned long long) * (slots + 1), s));
  CUDA_TRY(cudaMemsetAsync(set, 0, sizeof(unsigned long long) * (slots + 1), s));
  if (n > 0) {
    const size_t sm = smem_score(t->host, 0);
    BPS_TRY(bps, collect_unroll_kernel, sm);
    collect_unroll_kernel<<<grid_for(t, n, bps), TPB, sm, s>>>(
        t->d_task, d_records, n, set, slots);
    CUDA_TRY(cudaGetLastError());
  }
  std::vector<unsigned long long> h(slots + 1);
  CUDA_TRY(cudaMemcpyAsync(h.data(), set, sizeof(unsigned long long) * (slots + 1), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaFreeAsync(set, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (h[slots]) return fail(LS_E_UNSUPPORTED, "more than 16384 distinct unroll products in one batch");
  int c = 0, distinct = 0;
  for (int q = 0; q < slots; ++q)
    if (h[q]) {
      ++distinct;
      if (c < cap) h_values[c++] = (int64_t)h[q];
    }
  if (distinct > cap) return fail(LS_E_ARG, "h_values holds fewer entries than the distinct unroll products");
  std::sort(h_values, h_values + c);
  *h_count = c;
  return LS_E_OK;
}

static int score_device(ls_task* t, const void* d_src, int pbytes, int64_t n, double* d_scores, double* d_features,
                        int32_t* d_status, cudaStream_t s) {
  const int mode = mode_of(t, pbytes != 0);
  const ScoreFn fn = score_fn(t->host, mode, pbytes);
  const size_t sm = smem_score(t->host, mode);
  BPS_TRY(bps, fn, sm);
  fn<<<grid_for(t, n, bps), TPB, sm, s>>>(t->d_task, d_src, pbytes, n, d_scores, d_features,
                                                            d_status);
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

int ls_score(ls_task* t, const ls_record* d_records, int64_t n, double* d_scores, double* d_features,
             int32_t* d_status, void* stream) {
  if (!t || n < 0 || (n && !d_records)) return fail(LS_E_ARG, "bad argument");
  if (n == 0) return LS_E_OK;
  CUDA_TRY(cudaSetDevice(t->device));
  return score_device(t, d_records, 0, n, d_scores, d_features, d_status, (cudaStream_t)stream);
}

static int check_points(const ls_task* t, int32_t pbytes) {
  if (pbytes != 4 && pbytes != 8) return fail(LS_E_ARG, "point_bytes must be 4 or 8");
  if (t->host.sp_n < 1) return fail(LS_E_ARG, "no schedule space attached (ls_task_set_space)");
  return LS_E_OK;
}

int ls_score_points(ls_task* t, const void* d_points, int32_t pbytes, int64_t n, double* d_scores,
                    double* d_features, int32_t* d_status, void* stream) {
  if (!t || n < 0 || (n && !d_points)) return fail(LS_E_ARG, "bad argument");
  if (int rc = check_points(t, pbytes)) return rc;
  if (n == 0) return LS_E_OK;
  CUDA_TRY(cudaSetDevice(t->device));
  return score_device(t, d_points, pbytes, n, d_scores, d_features, d_status, (cudaStream_t)stream);
}

// Workspace: [4 KiB of self-resetting counters (tickets) | the valid count] [key lists]
// [outputs when h_out].  The launch leaves every counter at zero, so a workspace cached
// on the task is reused on the same stream without a memset.  h_out != null: the top-k
// scores, indices and the valid count come back in one copy to h_out (count in a 16-byte
// slot, then [k] f64, [k] i64).
constexpr size_t WS_CTR_BYTES = 4096 + 16;
// then the two-stage minima slots + T (+inf between launches: 0xFF fill, reset by the merge)
// and the block-list counts, at a fixed offset so no other layout ever overlaps them
constexpr size_t WS_MIN_KEYS = TK_MAXGRID + 1;
constexpr size_t WS_FIXED_BYTES = WS_CTR_BYTES + 16 * WS_MIN_KEYS + 4 * TK_MAXGRID;
static cudaError_t ws_init(unsigned char* ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(ws, 0, WS_CTR_BYTES, s);
  return e != cudaSuccess ? e : cudaMemsetAsync(ws + WS_CTR_BYTES, 0xFF, 16 * WS_MIN_KEYS, s);
}

static int topk_device(ls_task* t, const void* d_src, int pbytes, int64_t n, int64_t base_index, int32_t k,
                       double* d_top_scores, int64_t* d_top_index, unsigned long long* d_valid, cudaStream_t s,
                       void* h_out = nullptr) {
  const int mode = mode_of(t, pbytes != 0);
  const TopkFn fn = topk_fn(t->host, mode, pbytes);
  const size_t sm = smem_topk(t->host, k, mode);
  BPS_TRY(bps, fn, sm);
  const int grid = n > 0 ? grid_for(t, n, bps) : 1;
  const int ngroups = (grid + TK_GROUP - 1) / TK_GROUP;
  // two-stage merge (block-minima bound, merge_filter_kernel) when the grid has plenty of
  // blocks per answer key; else the in-kernel merge tree
  const bool two = 4 * k <= grid && grid <= topk_buf(k) && grid <= TK_MAXGRID;
  // two-stage: [grid] buffers of topk_buf(k) keys and as many survivor slots
  const size_t keys_bytes = sizeof(Key) * (two ? (size_t)grid * 2 * topk_buf(k) : ((size_t)grid + ngroups) * k);
  const size_t out_bytes = h_out ? 16 + 16 * (size_t)k : 0;
  const size_t ws_bytes = WS_FIXED_BYTES + keys_bytes + out_bytes;
  // The workspace lease: the task's cached block (grown on demand) unless another call holds it
  // or it belongs to another stream, else a private block.  Released on every exit path; a call
  // that fails after its first launch leaves the cached block marked for re-initialisation (its
  // self-resetting counters may not have been reset).
  struct Lease {
    ls_task* t;
    cudaStream_t s;
    unsigned char* ws = nullptr;
    unsigned long long* tr = nullptr;
    bool cached = false, launched = false, ok = false;
    ~Lease() {
      if (tr) cudaFree(tr);
      if (cached) {
        std::lock_guard<std::mutex> g(t->mu);
        t->ws_busy = false;
        if (launched && !ok) t->ws_dirty = true;
      } else if (ws) {
        cudaFreeAsync(ws, s);
      }
    }
  } L{t, s};
  {
    std::lock_guard<std::mutex> g(t->mu);
    if (!t->ws_busy && (!t->ws || t->ws_stream == s)) {
      if (t->ws_bytes < ws_bytes) {  // grow (the old block is freed in its stream's order)
        if (t->ws) cudaFreeAsync(t->ws, t->ws_stream);
        t->ws = nullptr;
        t->ws_bytes = 0;
        CUDA_TRY(cudaMallocAsync(&t->ws, ws_bytes, s));
        t->ws_bytes = ws_bytes;
        t->ws_stream = s;
        t->ws_dirty = true;
      }
      if (t->ws_dirty) {
        CUDA_TRY(ws_init(t->ws, s));
        t->ws_dirty = false;
      }
      t->ws_busy = true;
      L.ws = t->ws;
      L.cached = true;
    }
  }
  if (!L.cached) {  // concurrent call or another stream: a private workspace
    CUDA_TRY(cudaMallocAsync(&L.ws, ws_bytes, s));
    CUDA_TRY(ws_init(L.ws, s));
  }
  unsigned char* const ws = L.ws;
  unsigned int* tickets = reinterpret_cast<unsigned int*>(ws);
  unsigned long long* wvalid = reinterpret_cast<unsigned long long*>(ws + 4096);
  Key* block_out = reinterpret_cast<Key*>(ws + WS_FIXED_BYTES);
  Key* group_out = block_out + (size_t)grid * (two ? topk_buf(k) : k);  // tree: group lists; two-stage: survivors
  Key* mins = two ? reinterpret_cast<Key*>(ws + WS_CTR_BYTES) : nullptr;
  unsigned char* out = ws + WS_FIXED_BYTES + keys_bytes;
  if (h_out) {
    d_valid = reinterpret_cast<unsigned long long*>(out);
    d_top_scores = reinterpret_cast<double*>(out + 16);
    d_top_index = reinterpret_cast<int64_t*>(d_top_scores + k);
  }
  const char* tr_env = getenv("LS_TRACE");
  if (tr_env && tr_env[0] == '1') {  // phase timestamps to stderr (profiling aid)
    CUDA_TRY(cudaMalloc(&L.tr, sizeof(unsigned long long) * TR_SLOTS * grid));
    CUDA_TRY(cudaMemset(L.tr, 0, sizeof(unsigned long long) * TR_SLOTS * grid));
  }
  unsigned long long* const tr = L.tr;
  L.launched = true;
  fn<<<grid, TPB, sm, s>>>(t->d_task, d_src, pbytes, n, base_index, k, block_out, group_out, tickets, d_top_scores,
                           d_top_index, d_valid, topk_buf(k), mins, wvalid, tr);
  CUDA_TRY(cudaGetLastError());
  if (two) {
    const size_t msm = topk_state_bytes(topk_buf(k));
    if (kernel_prepare(merge_filter_kernel, msm, false) < 0) return LS_E_CUDA;
    const int g2 = grid;  // one block list each
    // programmatic dependent launch: the merge is queued behind the scoring
    // launch's tail (its blocks wait in griddepcontrol.wait for the scoring
    // grid's completion and memory), not behind a full kernel boundary
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g2);
    cfg.blockDim = dim3(TPB);
    cfg.dynamicSmemBytes = msm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const Key* cbo = block_out;
    const Key* cmins = mins;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, merge_filter_kernel, cbo, cmins, grid, k, group_out, tickets, d_top_scores,
                                d_top_index, topk_buf(k), d_valid, wvalid, tr));
  }
  if (h_out) CUDA_TRY(cudaMemcpyAsync(h_out, out, out_bytes, cudaMemcpyDeviceToHost, s));
  L.ok = true;
  if (tr) {
    std::vector<unsigned long long> h((size_t)TR_SLOTS * grid);
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaMemcpy(h.data(), tr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, surv = 0;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[b * TR_SLOTS]);
    for (int b = 0; b < grid; ++b)
      if (h[b * TR_SLOTS + 3] >> 63) surv = h[b * TR_SLOTS + 3] & ~(1ull << 63), h[b * TR_SLOTS + 3] = 0;
    double avg[8] = {0}, mx[8] = {0};
    for (int q = 0; q < 8; ++q) {
      int cnt = 0;
      for (int b = 0; b < grid; ++b)
        if (h[b * TR_SLOTS + q] > t0) {
          const double v = (double)(h[b * TR_SLOTS + q] - t0) / 1e3;
          avg[q] += v, mx[q] = std::max(mx[q], v), ++cnt;
        }
      if (cnt) avg[q] /= cnt;
    }
    fprintf(stderr, "LS_TRACE n=%lld grid=%d us(avg/max): staged %.1f/%.1f main %.1f/%.1f listed %.1f/%.1f | "
            "tree group %.1f final %.1f | two-stage start %.1f T %.1f filtered %.1f final %.1f survivors %llu\n",
            (long long)n, grid, avg[1], mx[1], avg[2], mx[2], avg[3], mx[3], mx[4], mx[5], mx[4], mx[5], mx[6],
            mx[7], surv);
    if (getenv("LS_TRACE_BLOCKS")) {  // per-block main-loop ends
      std::vector<std::pair<double, int>> e;
      for (int b = 0; b < grid; ++b)
        if (h[b * TR_SLOTS + 2] > t0) e.push_back({(double)(h[b * TR_SLOTS + 2] - t0) / 1e3, b});
      std::sort(e.begin(), e.end());
      fprintf(stderr, "LS_TRACE blocks (main end us, block, sm, start us):");
      for (size_t q = 0; q < e.size(); q += std::max<size_t>(1, e.size() / 24)) {
        const int b = e[q].second;
        fprintf(stderr, " %.1f/%d/%llu/%.1f", e[q].first, b, h[b * TR_SLOTS + 8], (double)(h[b * TR_SLOTS] - t0) / 1e3);
      }
      if (!e.empty()) {
        const int b = e.back().second;
        fprintf(stderr, " | max %.1f/%d/%llu/%.1f", e.back().first, b, h[b * TR_SLOTS + 8],
                (double)(h[b * TR_SLOTS] - t0) / 1e3);
      }
      fprintf(stderr, "\n");
    }
  }
  return LS_E_OK;
}

static int score_topk_any(ls_task* t, const void* d_src, int pbytes, int64_t n, int64_t base_index, int32_t k,
                          double* d_top_scores, int64_t* d_top_index, int64_t* d_n_valid, cudaStream_t s) {
  CUDA_TRY(cudaSetDevice(t->device));
  // the launch writes the count (no memset): d_n_valid may be null
  return topk_device(t, d_src, pbytes, n, base_index, k, d_top_scores, d_top_index,
                     reinterpret_cast<unsigned long long*>(d_n_valid), s);
}

int ls_score_topk(ls_task* t, const ls_record* d_records, int64_t n, int64_t base_index, int32_t k,
                  double* d_top_scores, int64_t* d_top_index, int64_t* d_n_valid, void* stream) {
  if (!t || n < 0 || (n && !d_records) || !d_top_scores || !d_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  return score_topk_any(t, d_records, 0, n, base_index, k, d_top_scores, d_top_index, d_n_valid,
                        (cudaStream_t)stream);
}

int ls_score_topk_points(ls_task* t, const void* d_points, int32_t pbytes, int64_t n, int64_t base_index, int32_t k,
                         double* d_top_scores, int64_t* d_top_index, int64_t* d_n_valid, void* stream) {
  if (!t || n < 0 || (n && !d_points) || !d_top_scores || !d_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  if (int rc = check_points(t, pbytes)) return rc;
  return score_topk_any(t, d_points, pbytes, n, base_index, k, d_top_scores, d_top_index, d_n_valid,
                        (cudaStream_t)stream);
}

int ls_task_set_space(ls_task* t, const ls_space_desc* sp) {
  if (!t || !sp || sp->n_axes < 1 || sp->n_axes > LS_MAX_AXES) return fail(LS_E_ARG, "bad space");
  std::vector<uint64_t> vals;
  DAxis ax[LS_MAX_AXES];
  memset(ax, 0, sizeof(ax));
  for (int a = 0; a < sp->n_axes; ++a) {
    const ls_axis& x = sp->axes[a];
    if (x.kind < LS_AX_PARAM || x.kind > LS_AX_BIT || x.n_choices < 1) return fail(LS_E_ARG, "bad axis");
    if ((x.kind == LS_AX_PARAM || x.kind == LS_AX_VEC) && (x.param < 0 || x.param >= LS_MAX_PARAMS))
      return fail(LS_E_ARG, "bad axis param slot");
    if ((x.kind == LS_AX_VEC || x.kind == LS_AX_BIT) && (x.bit < 0 || x.bit >= 32)) return fail(LS_E_ARG, "bad axis bit");
    if (x.kind == LS_AX_BIT && x.n_choices > 2) return fail(LS_E_ARG, "on/off axis with more than 2 choices");
    if (x.kind != LS_AX_BIT && !x.values) return fail(LS_E_ARG, "axis without values");
    ax[a].kind = (int8_t)x.kind;
    ax[a].param = (int8_t)x.param;
    ax[a].bit = (int8_t)x.bit;
    ax[a].n = (uint32_t)x.n_choices;
    ax[a].voff = (uint32_t)vals.size();
    ax[a].magic = x.n_choices >= 2 ? (~0ull / (uint64_t)x.n_choices) + 1 : 0;
    if (x.kind != LS_AX_BIT)
      for (int c = 0; c < x.n_choices; ++c) {
        if ((x.kind == LS_AX_PARAM || x.kind == LS_AX_VEC) && x.values[c] > 0xFFFFu)
          return fail(LS_E_ARG, "factor/width above 65535");
        vals.push_back(x.values[c]);
      }
  }
  std::lock_guard<std::mutex> g(t->mu);
  CUDA_TRY(cudaSetDevice(t->device));
  uint64_t* dv = nullptr;
  CUDA_TRY(cudaMalloc(&dv, sizeof(uint64_t) * std::max<size_t>(1, vals.size())));
  if (!vals.empty()) CUDA_TRY(cudaMemcpy(dv, vals.data(), sizeof(uint64_t) * vals.size(), cudaMemcpyHostToDevice));
  t->retired.push_back(dv);
  t->host.sp_n = sp->n_axes;
  t->host.sp_vals = dv;
  memcpy(t->host.sp_ax, ax, sizeof(ax));
  t->host.tt_ok = 0;
  t->host.tt = nullptr;
  const bool tables = plan_tensor_tables(t->host);
  uint64_t* dtt = nullptr;
  if (tables) {
    CUDA_TRY(cudaMalloc(&dtt, sizeof(uint64_t) * (size_t)t->host.tt_len));
    t->retired.push_back(dtt);
    t->host.tt = dtt;
  }
  if (int rc = upload(t)) return rc;
  t->host.sp_ok = 0;
  if (tables) {
    build_ttab_kernel<<<(unsigned)((t->host.tt_len + 255) / 256), 256>>>(t->d_task, dtt);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    t->host.tt_ok = 1;
    int pax = -1;
    int32_t rows[16] = {0};
    std::vector<uint64_t> ext;
    if (plan_space(t->host, pax) && plan_space_groups(t->host, rows)) {
      plan_static_tiles(t->host, sp, ext);
      uint64_t* dext = nullptr;
      if (t->host.sp_static) {
        CUDA_TRY(cudaMalloc(&dext, sizeof(uint64_t) * ext.size()));
        t->retired.push_back(dext);
        CUDA_TRY(cudaMemcpy(dext, ext.data(), sizeof(uint64_t) * ext.size(), cudaMemcpyHostToDevice));
        t->host.sp_ext = dext;
      }
      const int np = pax >= 0 ? (int)t->host.sp_ax[pax].n : 1;
      uint64_t* dch = nullptr;
      int32_t *dst = nullptr, *drows = nullptr, *dovf = nullptr;
      uint32_t* dsd = nullptr;
      CUDA_TRY(cudaMalloc(&dch, sizeof(uint64_t) * np));
      t->retired.push_back(dch);
      CUDA_TRY(cudaMalloc(&dst, sizeof(int32_t) * np));
      t->retired.push_back(dst);
      CUDA_TRY(cudaMalloc(&dsd, sizeof(int32_t) * ((t->host.sd_len + 3) & ~3)));  // 16-byte staging loads
      t->retired.push_back(dsd);
      CUDA_TRY(cudaMalloc(&drows, sizeof(rows) + sizeof(int32_t) * 9));
      t->retired.push_back(drows);
      CUDA_TRY(cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice));
      dovf = drows + 16;
      CUDA_TRY(cudaMemset(dovf, 0, sizeof(int32_t) * 9));  // overflow flag + per-group maxima
      if (int rc = upload(t)) return rc;
      const size_t sm = sizeof(int32_t) * NSLOT * TPB;
      build_pchain_kernel<<<(np + TPB - 1) / TPB, TPB, sm>>>(t->d_task, pax, dch, dst);
      CUDA_TRY(cudaGetLastError());
      build_sdt_kernel<<<(t->host.sd_len + 255) / 256, 256>>>(t->d_task, drows, dsd, dovf,
                                                              reinterpret_cast<unsigned int*>(dovf + 1));
      CUDA_TRY(cudaGetLastError());
      int32_t ovf_g[9] = {0};
      CUDA_TRY(cudaMemcpy(ovf_g, dovf, sizeof(ovf_g), cudaMemcpyDeviceToHost));
      const int32_t ovf = ovf_g[0];
      {  // MODE 5 (32-bit walk): every footprint, their sum and every movement below 2^32.
        // A dimension count with variables S expanded is at most (unique accesses) x the product of
        // their extents (_si_sum counts <= the product, _si_union <= the sum), so a footprint is
        // <= K_t * P^m_t and a movement <= max(accesses, K_t) * P^m_t, with P the product of all
        // transformed extents, K_t = unique accesses ^ rank, m_t = most dimensions sharing a variable.
        const unsigned int* gm = reinterpret_cast<const unsigned int*>(ovf_g + 1);
        double fsum = 0, prod = 1;
        bool divides = true;
        for (int q = 0; q < t->host.n_base; ++q) prod *= t->host.base_ext[q];
        for (int a = 0; a < t->host.sp_n; ++a)
          if (t->host.sp_ax[a].kind == LS_AX_PARAM)
            for (uint32_t c = 0; c < t->host.sp_ax[a].n; ++c) {
              const uint64_t F = sp->axes[a].values[c];
              int base = -1;
              for (int q = 0; q < t->host.n_base; ++q)
                for (int x = 0; x < t->host.n_xf; ++x)
                  if (t->host.xf[x].kind == LS_XF_TILE && t->host.xf[x].param == t->host.sp_ax[a].param &&
                      t->host.base_slot[q] == t->host.xf[x].slot)
                    base = q;
              if (base < 0 || F == 0 || t->host.base_ext[base] % (int64_t)F != 0) divides = false;
            }
        if (!divides) prod *= std::pow(2.0, (double)t->host.sp_n);  // ceil(E/F) * F < 2E per tile
        bool fits = t->host.sp_static && t->host.cap < 4294967295ll;
        for (int q = 0; q < t->host.n_tensors; ++q) {
          fsum += (double)std::max(1u, gm[2 * q]) * (double)std::max(1u, gm[2 * q + 1]);
          int m = 1;
          for (int v = 0; v < NSLOT; ++v) {
            int dims = 0;
            for (int r = 0; r < t->host.t_rank[q]; ++r)
              for (int x = 0; x < t->host.dim_nv[q * 4 + r]; ++x) dims += t->host.dim_var[q * 4 + r][x] == v;
            m = std::max(m, dims);
          }
          const double K = std::pow((double)t->host.t_nu[q], (double)t->host.t_rank[q]);
          if (std::max((double)t->host.t_nacc[q], K) * std::pow(prod, (double)m) >= 4294967295.0) fits = false;
        }
        // the Horner sum of the prefix products is <= (chain length) * P
        t->host.sp_narrow = fits && fsum < 4294967295.0 && prod * (t->host.sp_nchain + 1) < 4294967295.0;
      }
      t->host.sp_chain = dch;
      t->host.sp_pstat = dst;
      t->host.sd_tab = reinterpret_cast<const int32_t*>(dsd);
      t->host.sp_ok = ovf ? 0 : 1;  // a group product beyond 32 bits: keep the tensor-table path
    }
    return upload(t);
  }
  return LS_E_OK;
}

static int merge_launch(const Key* keys, const double* d_scores, const int64_t* d_index, int64_t m, int32_t k_out,
                        double* d_out_scores, int64_t* d_out_index, cudaStream_t s) {
  const size_t msm = topk_state_bytes(topk_buf(k_out));
  if (kernel_prepare(merge_keys_kernel, msm, false) < 0) return LS_E_CUDA;
  merge_keys_kernel<<<1, TPB, msm, s>>>(keys, d_scores, d_index, m, k_out, d_out_scores, d_out_index, topk_buf(k_out));
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

int ls_topk_merge(const double* d_scores, const int64_t* d_index, int32_t n_lists, int32_t k_in, int32_t k_out,
                  double* d_out_scores, int64_t* d_out_index, void* stream) {
  if (!d_scores || !d_index || n_lists < 0 || k_in < 0 || k_out < 1 || k_out > TK_MAXK || !d_out_scores ||
      !d_out_index)
    return fail(LS_E_ARG, "bad argument");
  return merge_launch(nullptr, d_scores, d_index, (int64_t)n_lists * k_in, k_out, d_out_scores, d_out_index,
                      (cudaStream_t)stream);
}

int ls_topk_merge_keys(const ls_topk_key* d_keys, int64_t m, int32_t k_out, double* d_out_scores,
                       int64_t* d_out_index, void* stream) {
  if ((m > 0 && !d_keys) || m < 0 || k_out < 1 || k_out > TK_MAXK || !d_out_scores || !d_out_index)
    return fail(LS_E_ARG, "bad argument");
  static_assert(sizeof(ls_topk_key) == sizeof(Key), "ls_topk_key layout");
  return merge_launch(reinterpret_cast<const Key*>(d_keys), nullptr, nullptr, m, k_out, d_out_scores, d_out_index,
                      (cudaStream_t)stream);
}

int ls_topk_to_keys(const double* d_scores, const int64_t* d_index, int64_t m, ls_topk_key* d_keys, void* stream) {
  if (m < 0 || (m > 0 && (!d_scores || !d_index || !d_keys))) return fail(LS_E_ARG, "bad argument");
  if (m == 0) return LS_E_OK;
  lists_to_keys_kernel<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      d_scores, d_index, m, reinterpret_cast<Key*>(d_keys));
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

// Host buffers that are page-locked and mapped (cudaHostAlloc / torch pin_memory under UVA)
// are read by the scoring kernel itself over the host link: the host->device transfer of the
// candidates overlaps the scoring with no staging copy.  Returns the device alias or null.
static const void* mapped_alias(const void* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

static int score_topk_mapped(ls_task* t, const void* d_alias, int pbytes, int64_t n, int64_t base_index, int32_t k,
                             double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid, cudaStream_t s) {
  // pinned staging block: count (16 B slot) | scores | indices, filled by one D2H copy; the task's
  // cached block unless another host call holds it (then a private one), released on every path
  struct Stage {
    ls_task* t;
    unsigned char* p = nullptr;
    bool own = false;
    ~Stage() {
      if (own) {
        if (p) cudaFreeHost(p);
      } else if (p) {
        std::lock_guard<std::mutex> g(t->mu);
        t->stage_busy = false;
      }
    }
  } S{t};
  const size_t need = 16 + 16 * (size_t)k;
  {
    std::lock_guard<std::mutex> g(t->mu);
    if (!t->stage_busy) {
      if (t->stage_bytes < need) {
        if (t->stage) cudaFreeHost(t->stage);
        t->stage = nullptr;
        t->stage_bytes = 0;
        CUDA_TRY(cudaMallocHost(&t->stage, need));
        t->stage_bytes = need;
      }
      t->stage_busy = true;
      S.p = t->stage;
    }
  }
  if (!S.p) {  // concurrent host call on this task: a private staging block
    S.own = true;
    CUDA_TRY(cudaMallocHost(&S.p, need));
  }
  const int rc = topk_device(t, d_alias, pbytes, n, base_index, k, nullptr, nullptr, nullptr, s, S.p);
  if (rc != LS_E_OK) return rc;
  CUDA_TRY(cudaStreamSynchronize(s));
  unsigned long long hv = 0;
  memcpy(&hv, S.p, 8);
  memcpy(h_top_scores, S.p + 16, sizeof(double) * k);
  memcpy(h_top_index, S.p + 16 + 8 * (size_t)k, sizeof(int64_t) * k);
  if (h_n_valid) *h_n_valid = (int64_t)hv;
  return LS_E_OK;
}

// Host buffers that are not mapped: chunks are copied on a side stream into two
// device buffers (the copy of chunk c+1 overlaps the scoring of chunk c), every
// chunk gets its own fused top-k, and the chunk lists are merged.  Every stream,
// event and buffer is owned by `R` and released (after the work it backs has
// drained) on every exit path.
static int score_topk_host_any(ls_task* t, const void* h_src, int pbytes, int64_t n, int64_t base_index, int32_t k,
                               double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid, cudaStream_t s) {
  CUDA_TRY(cudaSetDevice(t->device));
  if (n > 0)
    if (const void* alias = mapped_alias(h_src))
      return score_topk_mapped(t, alias, pbytes, n, base_index, k, h_top_scores, h_top_index, h_n_valid, s);
  const size_t esz = pbytes ? (size_t)pbytes : sizeof(ls_record);
  const int64_t CH = (int64_t)((8u << 20) / esz);  // 8 MiB chunks
  const int64_t nch = std::max<int64_t>(1, (n + CH - 1) / CH);
  struct Res {
    cudaStream_t s, cp = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // start, ready[2], freed[2]
    std::vector<void*> bufs;
    ~Res() {
      cudaStreamSynchronize(s);  // the queued work that uses the buffers has drained
      if (cp) cudaStreamSynchronize(cp);
      for (void* p : bufs) cudaFree(p);
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      if (cp) cudaStreamDestroy(cp);
    }
    cudaError_t alloc(void** p, size_t bytes) {
      const cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 16), s);
      if (e == cudaSuccess) bufs.push_back(*p);
      return e;
    }
  } R{s};
  CUDA_TRY(cudaStreamCreateWithFlags(&R.cp, cudaStreamNonBlocking));
  for (auto& e : R.ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t ev_start = R.ev[0], *ready = R.ev + 1, *freed = R.ev + 3;
  unsigned char* buf[2] = {nullptr, nullptr};
  double *ls = nullptr, *out_s = nullptr;
  int64_t *li = nullptr, *out_i = nullptr;
  unsigned long long* valid = nullptr;
  for (int b = 0; b < 2; ++b)
    CUDA_TRY(R.alloc((void**)&buf[b], esz * (size_t)std::min(CH, std::max<int64_t>(n, 1))));
  CUDA_TRY(R.alloc((void**)&ls, sizeof(double) * nch * k));
  CUDA_TRY(R.alloc((void**)&li, sizeof(int64_t) * nch * k));
  CUDA_TRY(R.alloc((void**)&valid, sizeof(unsigned long long) * nch));  // one count per chunk
  CUDA_TRY(R.alloc((void**)&out_s, sizeof(double) * k));
  CUDA_TRY(R.alloc((void**)&out_i, sizeof(int64_t) * k));
  CUDA_TRY(cudaEventRecord(ev_start, s));
  CUDA_TRY(cudaStreamWaitEvent(R.cp, ev_start, 0));
  const unsigned char* src = reinterpret_cast<const unsigned char*>(h_src);
  for (int64_t c = 0; c < nch; ++c) {
    const int b = (int)(c & 1);
    const int64_t off = c * CH, m = std::min(CH, n - off);
    if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(R.cp, freed[b], 0));
    if (m > 0) CUDA_TRY(cudaMemcpyAsync(buf[b], src + off * esz, esz * m, cudaMemcpyHostToDevice, R.cp));
    CUDA_TRY(cudaEventRecord(ready[b], R.cp));
    CUDA_TRY(cudaStreamWaitEvent(s, ready[b], 0));
    if (int rc = topk_device(t, buf[b], pbytes, std::max<int64_t>(m, 0), base_index + off, k, ls + c * k, li + c * k,
                             valid + c, s))
      return rc;
    CUDA_TRY(cudaEventRecord(freed[b], s));
  }
  if (int rc = ls_topk_merge(ls, li, (int32_t)nch, k, k, out_s, out_i, s)) return rc;
  CUDA_TRY(cudaMemcpyAsync(h_top_scores, out_s, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(h_top_index, out_i, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
  std::vector<unsigned long long> hvs((size_t)nch, 0);
  CUDA_TRY(cudaMemcpyAsync(hvs.data(), valid, sizeof(unsigned long long) * nch, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  unsigned long long hv = 0;
  for (unsigned long long v : hvs) hv += v;
  if (h_n_valid) *h_n_valid = (int64_t)hv;
  return LS_E_OK;
}

int ls_score_topk_host(ls_task* t, const ls_record* h_records, int64_t n, int64_t base_index, int32_t k,
                       double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid, void* stream) {
  if (!t || n < 0 || (n && !h_records) || !h_top_scores || !h_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  return score_topk_host_any(t, h_records, 0, n, base_index, k, h_top_scores, h_top_index, h_n_valid,
                             (cudaStream_t)stream);
}

int ls_score_topk_points_host(ls_task* t, const void* h_points, int32_t pbytes, int64_t n, int64_t base_index,
                              int32_t k, double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid,
                              void* stream) {
  if (!t || n < 0 || (n && !h_points) || !h_top_scores || !h_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  if (int rc = check_points(t, pbytes)) return rc;
  return score_topk_host_any(t, h_points, pbytes, n, base_index, k, h_top_scores, h_top_index, h_n_valid,
                             (cudaStream_t)stream);
}

}  // extern "C"

// ES generation loop on device
#include "es.cuh"
