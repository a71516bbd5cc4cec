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

#pragma once
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
  // packed walk (MODE 5): a tensor's two group offsets in one word (group 2t in
  // the low half, 2t + 1 in the high half; every table offset < 2^16), advanced per loop level
  // by one add of the level's packed stage bytes
  int32_t sp_pack, pad9;
  uint32_t sd_offp[4];                   // packed first-row offsets per tensor
  uint32_t sd_Sp[LS_MAX_AXES][4];        // packed byte stride of one choice of each tile axis
  uint32_t sp_vbp[NSLOT][4];             // per loop slot: packed stage bytes of tensors 0..2, tensor-use bits
  uint32_t sp_vbp3[NSLOT];               // per loop slot: packed stage bytes of tensor 3
  const uint64_t* sp_rchain;             // per reorder choice: the chain innermost loop first
  // tile-point rows (MODE 5): the reorder axis is the last axis, so a point is tile point * choices
  // + reorder choice; one 32-byte row per tile point holds the tiled extents (F | ceil(E/F) << 16
  // per tile axis; 0 = a factor out of range) and the packed first-row offsets per tensor
  int32_t sp_tp_ok, sp_ntile;
  uint32_t sp_total;                     // points in the space (< 2^32)
  int32_t sp_pax;                        // the reorder axis (the last one) or -1
  uint8_t sp_tj_new[4], sp_tj_slot[4];   // slots the j-th tile axis writes (inner F, outer ceil(E/F))
  const uint4* sp_tp;                    // [tile points][2]
  const uint4* sp_crow;                  // per reorder choice: {innermost-first chain lo, hi, status, 0}
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

// Entries per group-table row: the 2^nb stage masks plus LS_SD_PAD padding
// entries, so rows start on different banks and lanes reading the same stage mask of different
// rows (the common case within a warp) do not conflict.
#ifndef LS_SD_PAD
#define LS_SD_PAD 1
#endif
__host__ __device__ inline int sd_row_len(int nb) { return (1 << nb) + LS_SD_PAD; }
// the tabulated path's dimension-count rows, padded the same way
__host__ __device__ inline int tab_row_len(int nv) { return (1 << nv) + LS_SD_PAD; }

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
static __device__ int apply_transforms(const DTask& T, const ls_record& r, Cand& c) {
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
static __device__ int apply_fast(const DTask& T, const ls_record& r, FastCand& c) {
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
    kb[D] = 4u * (uint32_t)(T.ftab_off[D] + k * tab_row_len(T.dim_nv[D]));
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
static __device__ void sim_slots(const DTask& T, const int32_t* prm, uint32_t flags, int32_t* E, int32_t* St,
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
static __device__ int32_t dim_count(const DTask& T, int D, uint32_t mask, uint32_t flags, const int32_t* E, const int32_t* St,
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
// Points are 3-, 4- or 8-byte little-endian unsigned integers (3: packed, for spaces below
// 2^24 points -- a quarter less to move over the host link than 4-byte points).
__device__ __forceinline__ uint64_t load_point(const void* __restrict__ src, int pbytes, int64_t i) {
  if (pbytes == 4) return (uint64_t)__ldg(reinterpret_cast<const unsigned int*>(src) + i);
  if (pbytes == 3) {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(src) + 3 * i;
    return (uint64_t)__ldg(b) | ((uint64_t)__ldg(b + 1) << 8) | ((uint64_t)__ldg(b + 2) << 16);
  }
  return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(src) + i);
}

// The point of candidate b + lane of a warp-aligned round base b (b % 32 == 0), or 0 past n.
// Warp-cooperative (every lane calls it): 3-byte points are read as the warp's 24 aligned
// words (one coalesced 96-byte request -- over the host link, byte loads would fetch every
// sector three times) and reassembled with two shuffles.
__device__ __forceinline__ uint64_t load_point_warp(const void* __restrict__ src, int pbytes, int64_t b, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t p0 = b + (threadIdx.x & ~31);  // the warp's first point
  if (pbytes != 3) return p0 + lane < n ? load_point(src, pbytes, p0 + lane) : 0;
  const unsigned char* bytes = reinterpret_cast<const unsigned char*>(src);
  const int64_t B0 = 3 * p0, Bend = 3 * n;  // B0 % 96 == 0: word aligned
  uint32_t w = 0;
  const int64_t wb = B0 + 4 * lane;
  if (lane < 24 && wb < Bend) {
    if (wb + 4 <= Bend) {
      w = __ldg(reinterpret_cast<const unsigned int*>(bytes + wb));
    } else {  // the buffer ends inside this word
      for (int q = 0; q < (int)(Bend - wb); ++q) w |= (uint32_t)__ldg(bytes + wb + q) << (8 * q);
    }
  }
  const int a = (3 * lane) >> 2, sh = (3 * lane & 3) * 8;
  const uint32_t lo = __shfl_sync(0xffffffffu, w, a), hi = __shfl_sync(0xffffffffu, w, a + 1);
  return p0 + lane < n ? (uint64_t)(__funnelshift_r(lo, hi, sh) & 0xFFFFFFu) : 0;
}

// SRC 2 (points in mapped pinned host memory): a round's TPB points are read by the block as
// one run of aligned 16-byte loads (pbytes * TPB / 16 loader threads: full 128-byte lines over
// the host link, ~20% more link throughput than the warps' 96-byte pieces of 3-byte points),
// one round ahead, staged into shared memory at the round boundary.
constexpr int PTS_STAGE_LOADS = 8 * TPB / 16;  // loader slots for the widest (8-byte) points
__device__ __forceinline__ uint4 load_round_chunk(const void* __restrict__ src, int pbytes, int64_t b, int64_t n) {
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  const int64_t o = b * pbytes + 16 * (int64_t)threadIdx.x, end = n * pbytes;
  if ((int)threadIdx.x >= pbytes * TPB / 16 || o >= end) return v;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(src) + o;
  if (o + 16 <= end) return __ldg(reinterpret_cast<const uint4*>(p));
  uint32_t w[4] = {0u, 0u, 0u, 0u};  // the buffer ends inside this chunk
  for (int q = 0; q < (int)(end - o); ++q) w[q >> 2] |= (uint32_t)__ldg(p + q) << (8 * (q & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ uint64_t staged_point(const uint4* buf, int pbytes) {
  const unsigned char* b = reinterpret_cast<const unsigned char*>(buf);
  const int t = threadIdx.x;
  if (pbytes == 4) return reinterpret_cast<const uint32_t*>(b)[t];
  if (pbytes == 8) return reinterpret_cast<const unsigned long long*>(b)[t];
  const int o = 3 * t;  // two aligned words around the 3 bytes
  const uint32_t lo = reinterpret_cast<const uint32_t*>(b)[o >> 2], hi = reinterpret_cast<const uint32_t*>(b)[(o >> 2) + 1];
  return __funnelshift_r(lo, hi, (o & 3) * 8) & 0xFFFFFFu;
}

__device__ __forceinline__ int space_score(const DTask& T, int n, int64_t P, int64_t H, int64_t dmov, double* f,
                                           double* score);

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
  return space_score(T, n, (int64_t)P, (int64_t)H, dmov, f, score);
}

// Features and score of a space-path candidate from the walk's products (ls/cost.py:132-161;
// closed forms of DESIGN.md §3.6).
__device__ __forceinline__ int space_score(const DTask& T, int n, int64_t P, int64_t H, int64_t dmov, double* f,
                                           double* score) {
  const bool cpu = T.family == LS_FAMILY_CPU;
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

// MODE 5 with packed group offsets (T.sp_pack): the same decode, walk and closed forms as
// eval_space<TM, true> with the per-level work cut down --
//   * a tensor's two group-table offsets live in one register (16 bits each) and advance by one
//     add of the level's packed stage bytes (a variable's stage bits are disjoint from every
//     other's, so the OR of eval_space is an add); each half is a shared-memory address;
//   * the chain is stored innermost-first and the walk is unrolled over chain positions (the
//     chain length is uniform across the launch), so nibble extraction uses constant shifts,
//     the PTX counter-register wrap is a constant condition and the reuse flags stay predicates;
//   * the tensors using the level's variable come with the packed stage bytes (one 16-byte
//     shared load per level);
//   * the extents of untiled base loops are written once per thread (Evaluator).
// Bit-identical to eval_space<TM, true> (tests: every BASELINE space on the points paths).
template <int TM>
__device__ __forceinline__ int eval_space_packed(const DTask& T, const int32_t* __restrict__ sdt, uint64_t x,
                                                 FastCand& c, double* f, double* score) {
  uint32_t kp[TM];
  uint32_t pch = 0;
  uint4 crow;
  if (T.sp_tp_ok) {  // tile-point row: one division, two 16-byte loads
    if (x >= T.sp_total) return LS_ST_POINT_RANGE;
    const uint32_t x32 = (uint32_t)x;
    uint32_t tp = x32;
    if (T.sp_pax >= 0) {
      const DAxis& ax = T.sp_ax[T.sp_pax];
      if (ax.n > 1) {
        tp = (uint32_t)(((uint64_t)x32 * (uint32_t)(ax.magic >> 32) + __umulhi(x32, (uint32_t)ax.magic)) >> 32);
        pch = x32 - tp * (uint32_t)ax.n;
      } else {
        tp = x32;
      }
    }
    // the tile-point row and the reorder choice's chain row, issued together (one latency)
    const uint4 w = __ldg(T.sp_tp + 2 * (size_t)tp);
    const uint4 kw = __ldg(T.sp_tp + 2 * (size_t)tp + 1);
    crow = __ldg(T.sp_crow + pch);
    if (w.x == 0u) return LS_ST_TILE_RANGE;
    const int nt = T.sp_ntile;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= nt) break;  // uniform
      const uint32_t wj = j == 0 ? w.x : j == 1 ? w.y : j == 2 ? w.z : w.w;
      c.E(T.sp_tj_new[j]) = (int32_t)(wj & 0xFFFFu);
      c.E(T.sp_tj_slot[j]) = (int32_t)(wj >> 16);
    }
#pragma unroll
    for (int t = 0; t < TM; ++t) kp[t] = t == 0 ? kw.x : t == 1 ? kw.y : t == 2 ? kw.z : kw.w;
  } else {
#pragma unroll
  for (int t = 0; t < TM; ++t) kp[t] = T.sd_offp[t];
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
    for (int t = 0; t < TM; ++t) kp[t] += ch * T.sd_Sp[a][t];
    // Tile (ls/ir.py:361-382) of a base loop: F and ceil(E/F) per choice
    const uint64_t e = __ldg(reinterpret_cast<const unsigned long long*>(T.sp_ext) + ax.voff + ch);
    if (e >> 63) return LS_ST_TILE_RANGE;
    c.E(T.sp_tnew[a]) = (int32_t)(e & 0xFFFFu);
    c.E(T.sp_tslot[a]) = (int32_t)((e >> 16) & 0x7FFFFFFFu);
  }
  }
  if (!T.sp_tp_ok) crow = __ldg(T.sp_crow + pch);
  if (crow.z) return (int)crow.z;
  const uint64_t rchain = (uint64_t)crow.x | ((uint64_t)crow.y << 32);
  const int n = T.sp_nchain;
  // offsets relative to the dynamic shared memory base (the tables sit at dyn + task_bytes,
  // DESIGN.md §3.6): a lookup is one mask/shift and one shared load
  extern __shared__ __align__(16) unsigned char dyn[];
  const uint32_t tbo = (uint32_t)(reinterpret_cast<const unsigned char*>(sdt) - dyn);
#pragma unroll
  for (int t = 0; t < TM; ++t) kp[t] += tbo | (tbo << 16);
  auto fp = [&](uint32_t o) -> uint32_t {
    return *reinterpret_cast<const uint32_t*>(dyn + (o & 0xFFFFu)) * *reinterpret_cast<const uint32_t*>(dyn + (o >> 16));
  };
  uint32_t Fb[TM], dm[TM];
  bool ru[TM];
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    Fb[t] = fp(kp[t]);
    dm[t] = (uint32_t)T.t_nacc[t];
    ru[t] = true;
  }
  const uint32_t cap = (uint32_t)T.cap;
  const bool cpu = T.family == LS_FAMILY_CPU;
  const uint32_t* const vbp = &T.sp_vbp[0][0];
  uint32_t P = 1, H = 0;  // product of the extents; Horner sum of the outer prefix products (< 2^32 proven)
#ifdef LS_WALK_PIPE
  int vn = (int)(rchain & 15u);
  uint32_t En = (uint32_t)c.E(vn);
  uint4 rown = *reinterpret_cast<const uint4*>(vbp + 4 * vn);
#endif
#pragma unroll
  for (int q = 0; q < LS_MAX_CHAIN; ++q) {  // chain position p = n - 1 - q, innermost first
    if (q >= n) break;                        // uniform
#ifdef LS_WALK_PIPE
    const int v = vn;
    const uint32_t E = En;
    const uint4 row = rown;
    if (q + 1 < n) {  // the next level's extent and stage bytes, one level ahead
      vn = (int)((rchain >> (4 * (q + 1))) & 15u);
      En = (uint32_t)c.E(vn);
      rown = *reinterpret_cast<const uint4*>(vbp + 4 * vn);
    }
#else
    const int v = (int)((rchain >> (4 * q)) & 15u);
    const uint32_t E = (uint32_t)c.E(v);
    const uint4 row = *reinterpret_cast<const uint4*>(vbp + 4 * v);
#endif
    const uint32_t use = row.w;
    uint32_t single = 0;
#pragma unroll
    for (int t = 0; t < TM; ++t) single += Fb[t];
    const bool over = single > cap;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const uint32_t add = t == 0 ? row.x : t == 1 ? row.y : t == 2 ? row.z : T.sp_vbp3[v];
      kp[t] += add;
      const uint32_t Ff = fp(kp[t]);
      // r0 = ru && (!over || uses); keep Ff when !over || r0 == !over || (ru && uses);
      // ru' = r0 && Ff <= cap (bitwise on predicates: no short-circuit branches)
      const bool ub = (use & (1u << t)) != 0u;
      const bool keep = !over | (ru[t] & ub);
      dm[t] = keep ? Ff : dm[t] * E;
      ru[t] = ru[t] & (!over | ub) & (Ff <= cap);
      Fb[t] = Ff;
    }
    const uint32_t Ee = (cpu || q < 8) ? E : 1u;  // PTX: no trip for loops 8+ levels above the innermost
    if (q > 0) H = Ee * (1 + H);
    P *= Ee;
  }
  int64_t dmov = 0;
#pragma unroll
  for (int t = 0; t < TM; ++t) dmov += (int64_t)dm[t];
  return space_score(T, n, (int64_t)P, (int64_t)H, dmov, f, score);
}

// The space kernels' evaluator: MODE 5 takes the packed walk (LS_WALK_OLD: the reference
// formulation, for A/B runs).
template <int TM, int MODE>
__device__ __forceinline__ int eval_space_mode(const DTask& T, const int32_t* __restrict__ sdt, uint64_t x,
                                               FastCand& c, double* f, double* s) {
#ifndef LS_WALK_OLD
  if constexpr (MODE == 5) return eval_space_packed<TM>(T, sdt, x, c, f, s);
#endif
  return eval_space<TM, MODE == 5>(T, sdt, x, c, f, s);
}

// One group-table entry per thread: decode (group slot, tile-axis choices, stage
// mask); the entry is the product of the group's dimension counts (same fold as
// build_tab_kernel).  Products that do not fit 32 bits raise *overflow.
#ifdef LS_MAIN_TU
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
    if (rows[q] && e >= (int)T.sd_off[q] / 4 && e < (int)T.sd_off[q] / 4 + rows[q] * sd_row_len(T.sd_nb[q])) G = q;
  if (G < 0) return;
  const int loc = e - (int)T.sd_off[G] / 4;
  const int rl = sd_row_len(T.sd_nb[G]);
  const uint32_t mask = (uint32_t)(loc % rl);
  const uint32_t key = (uint32_t)(loc / rl);
  if (mask >> T.sd_nb[G]) {  // the row's padding entry (never read)
    tab[e] = 0;
    return;
  }
  int32_t prm[LS_MAX_PARAMS];
  for (int q = 0; q < LS_MAX_PARAMS; ++q) prm[q] = 1;
  for (int a = 0; a < T.sp_n; ++a) {
    const uint32_t stride = T.sd_S[a][G] / (4u * (uint32_t)rl);
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
#endif  // LS_MAIN_TU

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
static __device__ int tree_apply(const DTask& T, const ls_record& r, TreeCand& c) {
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
static __device__ int64_t tree_footprint(const DTask& T, const TreeCand& c, uint32_t flags, int L, int t, bool full) {
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
static __device__ void em_effects(int dialect, int shape, bool st_like, bool rmw, bool is_cmp, bool is_branch, bool mov_like,
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

static __device__ void em_push(Emu& e, int shape, bool st_like, bool rmw, bool is_cmp, bool is_branch, bool mov_like, int nops,
                        const int8_t* ok, const int8_t* oi, int pred = -1) {
  if (e.n >= EM_MAXI) {
    e.err = LS_ST_UNSUPPORTED;
    return;
  }
  em_effects(e.T->tr_dialect, shape, st_like, rmw, is_cmp, is_branch, mov_like, nops, ok, oi, pred, e.blk[e.n++]);
}

// schedule_block (ls/ilp.py:131-204): RAW edges with latencies, WAR / WAW order edges, greedy issue
static __device__ int64_t em_schedule(const Emu& e, int& err) {
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

static __device__ void em_end_block(Emu& e) {
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
static __device__ void em_body(Emu& e, int node) {
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

static __device__ void em_node(Emu& e, int node, int depth) {
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
static __device__ int em_cpu_features(const DTask& T, const TreeCand& c, int64_t& nfma, int64_t& nld, int64_t& nst,
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
static __device__ double tree_ptx_node(const DTask& T, const TreeCand& c, const int64_t* Wp, int node, double work) {
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

static __device__ double tree_ptx_ordered(const DTask& T, const TreeCand& c, const int64_t* Wp) {
  double work = 0.0;
  for (int n = c.root; n >= 0; n = c.nxt[n])
    if (n >= T.tr_na) work = tree_ptx_node(T, c, Wp, n, work);
  return rn_add(work, T.ptx_cost[LS_I_RET]);
}

static __device__ int eval_tree(const DTask& T, const ls_record& r, double* f, double* score) {
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
#ifdef LS_MAIN_TU
__global__ void build_pchain_kernel(const DTask* __restrict__ g, int32_t pax, uint64_t* __restrict__ chain,
                                    int32_t* __restrict__ pst, uint64_t* __restrict__ rchain,
                                    uint4* __restrict__ crow) {
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
  uint64_t rc = 0;  // innermost loop first
  for (int q = 0; q < c.n && !st; ++q) rc |= ((c.chain >> (4 * (c.n - 1 - q))) & 15ull) << (4 * q);
  rchain[pc] = rc;
  crow[pc] = make_uint4((uint32_t)rc, (uint32_t)(rc >> 32), (uint32_t)st, 0u);
}
#endif  // LS_MAIN_TU

// One dimension-table entry per thread: decode (dimension, key, mask).
#ifdef LS_MAIN_TU
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
  const int rl = tab_row_len(nv);
  const uint32_t mask = (uint32_t)(loc % rl);
  int32_t key = loc / rl;
  if (mask >> nv) {  // the row's padding entry (never read)
    tab[e] = 0;
    return;
  }
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
#endif  // LS_MAIN_TU

// One tensor-table entry per thread: decode (tensor, axis choices, mask of all
// the tensor's stage bits); the entry is the tensor footprint, the product of
// its dimension counts (ls/cache.py:117-130).
#ifdef LS_MAIN_TU
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
#endif  // LS_MAIN_TU

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
    if constexpr (MODE == 5)  // base loops no tile splits: their extents never change
      for (int q = 0; q < T.sp_n_untiled; ++q) fc.E(T.sp_untiled[q]) = T.base_ext[T.sp_untiled_pos[q]];
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
    return point_record<KEYS>(T, load_point(src, pbytes, i), r, kt, pch);
  }
}

#ifndef LS_MB5
#define LS_MB5 3  // resident blocks per SM the MODE 5 kernels are compiled for (register budget)
#endif
constexpr int min_blocks(int tm, int rm, int mode) {
  return mode == 6 ? 1 : mode == 5 ? LS_MB5 : mode ? 3 : (tm * rm <= 16 ? 3 : 1);
}

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
      st = eval_space_mode<TM, MODE>(T, tab, load_point(src, pbytes, i), ev.fc, f, &s);
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
static __device__ int topk_compact(TopkState& S, int k, int cnt) {
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

static __device__ int topk_select(TopkState& S, int k) {
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
    const int left = S.sel_count;
    __syncthreads();
    if (left == 1) break;
    if (left <= 32) {  // few keys share the selected digits (ties): rank them in one warp
      Key* const few = reinterpret_cast<Key*>(S.hist);  // the histogram is free: 1 KB = 64 keys
      if (threadIdx.x == 0) S.cnt2 = 0;
      __syncthreads();
      for (int j = threadIdx.x; j < c; j += blockDim.x) {
        const Key x = B[j];
        if ((x.s & ms) == ps && ((unsigned long long)x.i & mi) == pi) few[atomicAdd(&S.cnt2, 1)] = x;
      }
      __syncthreads();
      if (threadIdx.x < left) {  // keys are unique: exactly one has rank - 1 smaller ones
        const Key x = few[threadIdx.x];
        int r = 0;
        for (int j = 0; j < left; ++j) r += kless(few[j], x) ? 1 : 0;
        if (r == rank - 1) S.thr = x;
      }
      break;
    }
  }
  // the k-th key: the only one matching the selected digits (or ranked among the few above)
  if (S.sel_count == 1)
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      const Key x = B[j];
      if ((x.s & ms) == ps && ((unsigned long long)x.i & mi) == pi) S.thr = x;
    }
  __syncthreads();
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
constexpr int TK_FIN_CTR = 1022;  // tickets[] slot of the bound merge's finish ticket
constexpr int TK_PUB_CTR = 1021;  // bound merge: blocks that published their minimum
constexpr int TK_SURV_CTR = 1020; // bound merge: survivors appended so far
constexpr int TK_T_FLAG = 1019;   // bound merge: 1 once T (mins[TK_MAXGRID]) is published
constexpr int TK_UNF_CTR = 1018;  // bound merge: blocks that ended before T was out (lists left unfiltered)
constexpr int TK_MAXGRID = 2048;  // bound-merge minima slots (grid <= topk_buf(k) <= 2048); slot TK_MAXGRID = T
constexpr unsigned TK_UNFILTERED = 0x80000000u;  // block count flag: list left unfiltered
constexpr int MERGE_TREE = 0;      // in-kernel merge tree (k large next to the grid)
constexpr int MERGE_BOUND_K2 = 1;  // bound merge, ranked by bound_merge_kernel (small batches)
constexpr int MERGE_BOUND = 2;     // bound merge, ranked by the scoring grid's last block

// Phase timestamps of the fused kernel (LS_TRACE=1, tools/ only): per block
// [start, staged, main loop done, block list written, group merged, final written].
constexpr int TR_SLOTS = 12;  // 8 timestamps, the SM id, 3 more timestamps (final-phase steps)
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
static __device__ int merge_into(TopkState& S, const Key* src, int64_t m, int k, bool sorted) {
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

static __device__ void write_keys(const TopkState& S, int kept, int k, Key* out) {
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
static __device__ void write_sorted(TopkState& S, int kept, int k, double* __restrict__ out_s, int64_t* __restrict__ out_i) {
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
static __device__ void write_block_min(const TopkState& S, int kept, Key* out) {
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
static __device__ void bitonic_sort(Key* B, int cnt) {
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

// ---- bound merge (k small next to the grid; no second launch) ---------------
#ifndef LS_BOUND_C
#define LS_BOUND_C 128  // expected survivors ~ n k / (grid TPB R0): R0 = n k / (grid TPB C) + 1
#endif
#ifndef LS_BOUND_NUM
#define LS_BOUND_NUM 3  // T from the minima present when (NUM/4) of the grid has published
#endif
// Rounds of TPB candidates per block before it publishes its minimum (within its static
// share of 3/4 of the rounds), and whether the grid's last block ranks (T is out well
// before the blocks end) or bound_merge_kernel follows.
__host__ __device__ inline int64_t bound_static_rounds(int64_t n, int grid) {
  return (n + TPB - 1) / TPB * 3 / 4 / grid;
}
__host__ __device__ inline int64_t bound_rounds(int64_t n, int k, int grid) {
  const int64_t st = bound_static_rounds(n, grid);
  int64_t r0 = n * k / ((int64_t)grid * TPB * LS_BOUND_C) + 1;
  if (r0 > st) r0 = st > 1 ? st : 1;
  return r0;
}
inline bool bound_inline_rank(int64_t n, int k, int grid) {
  const double per_block = (double)((n + TPB - 1) / TPB) / grid;
  // T comes out ~2 rounds after the (3/4 grid)-th block published (the warp scheduler's age
  // priority delays the youngest blocks); blocks must still be scoring by then
  return per_block >= 6.0 && (double)bound_rounds(n, k, grid) + 2.0 <= 0.8 * per_block;
}
// Every block publishes the minimum of the keys it has seen after its first R0
// rounds; the (3/4 grid)-th block to publish sets T = the k-th smallest of the
// minima present (a slot is +inf or a real key of its block) -- k real keys lie
// at or below T, so T bounds the global k-th key from above -- while every
// other block keeps scoring (the slowest quarter of the blocks is not waited
// for: the warp scheduler's age priority makes early progress uneven).  At its end a block appends
// the keys of its buffer at or below T (the buffer is a superset of the block's
// share of the answer: a key leaves it only below k smaller ones) to one
// survivor list, and the last block to finish ranks the survivors (about
// n * k / (grid * TPB * R0) of them) into the sorted output.  No block ever
// waits for another (a block that ends before T is out leaves its buffer for
// the last block to filter), so the grid need not be co-resident.

// Block minimum to mins[blockIdx.x]; the last publisher computes and publishes
// T (its own buffer parked in `park` while the minima use the shared buffer).
// Block-uniform call.
static __device__ __noinline__ void bound_publish(TopkState& S, int k, Key* __restrict__ mins, unsigned int* __restrict__ ctr,
                              Key* __restrict__ park, unsigned long long* __restrict__ g_trace) {
  __shared__ unsigned int s_pub;
  __syncthreads();  // this round's inserts are in
  write_block_min(S, S.cnt, mins + blockIdx.x);
  if (threadIdx.x == 0) {
    __threadfence();
    s_pub = atomicAdd(&ctr[TK_PUB_CTR], 1u);
  }
  __syncthreads();
  if (s_pub != gridDim.x * LS_BOUND_NUM / 4 - 1) return;  // the (3/4 grid)-th publisher sets T
  __threadfence();
  const int cnt = S.cnt;
  const Key thr = S.thr;
  Key* const B = S.buf();
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) park[j] = B[j];
  __syncthreads();
  if (threadIdx.x == 0) S.cnt = 0;
  __syncthreads();
  for (int j0 = 0; j0 < (int)gridDim.x; j0 += blockDim.x) {  // block-uniform trip count (warp appends)
    const int j = j0 + threadIdx.x;
    Key x;
    x.s = KEY_INF_S;
    if (j < (int)gridDim.x) x = ld_key_cg(mins + j);
    const int slot = warp_append(&S.cnt, x.s != KEY_INF_S);
    if (slot >= 0) B[slot] = x;
  }
  __syncthreads();
  Key T;
  T.s = KEY_INF_S;
  T.i = KEY_INF_I;
  if (S.cnt > k) {  // radix selection of the k-th minimum (else no bound: every list survives)
    topk_select(S, k);
    T = S.thr;
  }
  if (threadIdx.x == 0) {
    mins[TK_MAXGRID] = T;
    __threadfence();
    atomicExch(&ctr[TK_T_FLAG], 1u);
  }
  trace_mark(g_trace, 4);
  __syncthreads();  // the parked keys are visible to the whole block
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) B[j] = park[j];
  if (threadIdx.x == 0) {
    S.cnt = cnt;
    S.thr = thr;
  }
  __syncthreads();
}

// Block end of the bound merge; the last block to finish writes the answer
// and resets the workspace for the next launch.
static __device__ __noinline__ void bound_rank(TopkState& S, int k, Key* __restrict__ mins,
                                               unsigned int* __restrict__ ctr, const Key* __restrict__ block_out,
                                               int cap, Key* __restrict__ surv, double* __restrict__ out_s,
                                               int64_t* __restrict__ out_i, unsigned long long* __restrict__ n_valid,
                                               unsigned long long* __restrict__ wvalid,
                                               unsigned long long* __restrict__ g_trace, int nblk, bool lists);

// Block end of the bound merge: the keys at or below T to the survivor list, or (T not out
// yet) the list left for bound_merge_kernel / the last block.  inline_rank: the last block of
// this grid ranks (large batches, T out long before the blocks end); otherwise
// bound_merge_kernel follows (programmatic dependent launch).
static __device__ __noinline__ void bound_finish(TopkState& S, int k, Key* __restrict__ mins, unsigned int* __restrict__ ctr,
                             Key* __restrict__ block_out, int cap, Key* __restrict__ surv, double* __restrict__ out_s,
                             int64_t* __restrict__ out_i, unsigned long long* __restrict__ n_valid,
                             unsigned long long* __restrict__ wvalid, unsigned long long* __restrict__ g_trace,
                             bool inline_rank) {
  __shared__ unsigned int s_flag, s_ticket;
  __shared__ Key s_T;
  unsigned int* const cnts = reinterpret_cast<unsigned int*>(mins + TK_MAXGRID + 1);
  Key* const B = S.buf();
  if (threadIdx.x == 0) {
    s_flag = atomicAdd(&ctr[TK_T_FLAG], 0u);
    if (s_flag) {
      __threadfence();
      s_T = ld_key_cg(mins + TK_MAXGRID);
    }
  }
  __syncthreads();
  const int cnt = S.cnt;
  if (s_flag) {  // keys at or below T to the survivor list
    const Key T = s_T;
    for (int j0 = 0; j0 < cnt; j0 += blockDim.x) {  // block-uniform trip count (warp appends)
      const int j = j0 + threadIdx.x;
      Key x;
      bool keep = false;
      if (j < cnt) {
        x = B[j];
        keep = !kless(T, x);
      }
      const int slot = warp_append(&ctr[TK_SURV_CTR], keep);
      if (slot >= 0) surv[slot] = x;
    }
    if (threadIdx.x == 0) cnts[blockIdx.x] = 0;
  } else {  // T is not out yet: the block's k best (a radix selection of the buffer) are left
            // for the last block / bound_merge_kernel to filter
    const int kept = topk_select(S, k);  // block-uniform (every thread reads the same S.cnt)
    Key* dst = block_out + (int64_t)blockIdx.x * cap;
    for (int j = threadIdx.x; j < kept; j += blockDim.x) dst[j] = B[j];
    if (threadIdx.x == 0) {
      cnts[blockIdx.x] = TK_UNFILTERED | (unsigned)kept;
      atomicAdd(&ctr[TK_UNF_CTR], 1u);
    }
  }
  __syncthreads();
  trace_mark(g_trace, 3);
  if (!inline_rank) {  // bound_merge_kernel filters the lists left and ranks
    asm volatile("griddepcontrol.launch_dependents;");
    return;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(&ctr[TK_FIN_CTR], 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  bound_rank(S, k, mins, ctr, block_out, cap, surv, out_s, out_i, n_valid, wvalid, g_trace, gridDim.x, true);
}

// The last block of the bound merge: every block has published (so T is out) and filtered or
// listed its keys.  One round trip for the controls (independent loads), the lists left
// unfiltered (lists = true; bound_merge_kernel has done them otherwise), one round trip for the
// survivors, the ranking, the workspace reset.
static __device__ __noinline__ void bound_rank(TopkState& S, int k, Key* __restrict__ mins,
                                               unsigned int* __restrict__ ctr, const Key* __restrict__ block_out,
                                               int cap, Key* __restrict__ surv, double* __restrict__ out_s,
                                               int64_t* __restrict__ out_i, unsigned long long* __restrict__ n_valid,
                                               unsigned long long* __restrict__ wvalid,
                                               unsigned long long* __restrict__ g_trace, int nblk, bool lists) {
  __shared__ Key s_T;
  __shared__ int s_nl;
  const unsigned int* const cnts = reinterpret_cast<const unsigned int*>(mins + TK_MAXGRID + 1);
  Key* const B = S.buf();
  trace_mark(g_trace, 5);
  __shared__ unsigned long long s_valid;
  __shared__ int s_c;
  if (threadIdx.x == 0) {
    s_valid = __ldcg(wvalid);
    s_T = ld_key_cg(mins + TK_MAXGRID);
    s_nl = lists ? (int)__ldcg(&ctr[TK_UNF_CTR]) : 0;
    s_c = (int)__ldcg(&ctr[TK_SURV_CTR]);
  }
  __syncthreads();
  if (s_nl) {  // lists of blocks that ended before T was out (small batches): filter them now,
               // all keys of all such lists in parallel (offsets by a block scan of the counts)
    const Key T = s_T;
    int* const off = reinterpret_cast<int*>(B);  // the block's own keys are out: scratch (grid + 1 <= cap ints)
    const int G = nblk;
    constexpr int PER = TK_MAXGRID / TPB;        // counts per thread (grid <= TK_MAXGRID)
    int cntv[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = threadIdx.x * PER + q;
      const unsigned cb = b < G ? __ldcg(cnts + b) : 0u;
      cntv[q] = (cb & TK_UNFILTERED) ? (int)(cb & ~TK_UNFILTERED) : 0;
      sum += cntv[q];
    }
    __shared__ int s_wsum[TPB / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[w] = incl;
    __syncthreads();
    int base = 0;
    for (int q = 0; q < w; ++q) base += s_wsum[q];
    int run = base + incl - sum;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = threadIdx.x * PER + q;
      if (b < G) off[b] = run;
      run += cntv[q];
    }
    int total = 0;
    for (int q = 0; q < TPB / 32; ++q) total += s_wsum[q];
    if (threadIdx.x == 0) off[G] = total;
    __shared__ int s_app;  // every other block is done: appends through a shared counter
    if (threadIdx.x == 0) s_app = 0;
    __syncthreads();
    Key* const dst = surv + s_c;
    for (int j0 = 0; j0 < total; j0 += 2 * blockDim.x) {  // block-uniform trip count (warp appends)
      Key x[2];
      bool keep[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {  // two independent loads in flight per thread
        const int j = j0 + u * blockDim.x + threadIdx.x;
        keep[u] = false;
        if (j < total) {
          int lo = 0, hi = G;  // the list holding flat position j: off[lo] <= j < off[lo + 1]
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= j) lo = mid; else hi = mid;
          }
          x[u] = ld_key_cg(block_out + (int64_t)lo * cap + (j - off[lo]));
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = j0 + u * blockDim.x + threadIdx.x;
        keep[u] = j < total && !kless(T, x[u]);
        const int slot = warp_append(&s_app, keep[u]);
        if (slot >= 0) dst[slot] = x[u];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_c += s_app;
    __threadfence_block();
    __syncthreads();
  }
  const int c0 = s_c;
  trace_mark(g_trace, 9);
  if (g_trace && threadIdx.x == 0) g_trace[blockIdx.x * TR_SLOTS + 7] = (1ull << 63) | (unsigned long long)c0;
  if (c0 <= S.cap) {  // rank the survivors by counting (keys are distinct): thread t ranks keys
                     // t, t + TPB, ...; every shared load is a warp broadcast, the comparisons are
                     // branch-free with independent partial counts; the k smallest land at their rank.
                     // Many survivors (small batches): a radix selection keeps the k smallest first.
    int c = c0;
    for (int j = threadIdx.x; j < c; j += blockDim.x) B[j] = ld_key_cg(surv + j);
    if (c > 2 * TPB) {
      if (threadIdx.x == 0) S.cnt = c;
      __syncthreads();
      c = topk_select(S, k);
    }
    __syncthreads();
    trace_mark(g_trace, 10);
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
      const Key x = B[q];
      int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
      int j = 0;
      for (; j + 4 <= c; j += 4) {
        const Key y0 = B[j], y1 = B[j + 1], y2 = B[j + 2], y3 = B[j + 3];
        r0 += (int)((y0.s < x.s) | ((y0.s == x.s) & (y0.i < x.i)));
        r1 += (int)((y1.s < x.s) | ((y1.s == x.s) & (y1.i < x.i)));
        r2 += (int)((y2.s < x.s) | ((y2.s == x.s) & (y2.i < x.i)));
        r3 += (int)((y3.s < x.s) | ((y3.s == x.s) & (y3.i < x.i)));
      }
      for (; j < c; ++j) r0 += (int)((B[j].s < x.s) | ((B[j].s == x.s) & (B[j].i < x.i)));
      const int r = r0 + r1 + r2 + r3;
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
    write_sorted(S, merge_into(S, surv, c0, k, false), k, out_s, out_i);
  }
  trace_mark(g_trace, 11);
  if (threadIdx.x == 0) {  // the count out; the counters back to zero for the next launch
    if (n_valid) *n_valid = s_valid;
    *wvalid = 0ull;
    ctr[TK_DYN_CTR] = 0;
    ctr[TK_FIN_CTR] = 0;
    ctr[TK_PUB_CTR] = 0;
    ctr[TK_SURV_CTR] = 0;
    ctr[TK_T_FLAG] = 0;
    ctr[TK_UNF_CTR] = 0;
  }
  for (int j = threadIdx.x; j <= nblk; j += blockDim.x) {  // minima slots (and T) back to +inf
    Key* m = mins + (j < nblk ? j : TK_MAXGRID);
    m->s = KEY_INF_S;
    m->i = KEY_INF_I;
  }
  trace_mark(g_trace, 6);
}

#ifdef LS_MAIN_TU
// Second launch of the bound merge (batches whose blocks end before T is out): every block
// filters its share of the lists left unfiltered in parallel, the last block ranks.  Queued
// with programmatic dependent launch behind the scoring grid.
__global__ void __launch_bounds__(TPB) bound_merge_kernel(Key* __restrict__ mins, unsigned int* __restrict__ ctr,
                                                          const Key* __restrict__ block_out, int nblk, int k, int cap,
                                                          Key* __restrict__ surv, double* __restrict__ out_s,
                                                          int64_t* __restrict__ out_i,
                                                          unsigned long long* __restrict__ n_valid,
                                                          unsigned long long* __restrict__ wvalid,
                                                          unsigned long long* __restrict__ g_trace) {
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ unsigned int s_ticket;
  TopkState& S = *reinterpret_cast<TopkState*>(raw);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scoring grid is complete and visible
  const unsigned int* const cnts = reinterpret_cast<const unsigned int*>(mins + TK_MAXGRID + 1);
  const Key T = ld_key_cg(mins + TK_MAXGRID);  // out: every scoring block published
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const unsigned cb = __ldcg(cnts + b);
    if (!(cb & TK_UNFILTERED)) continue;  // block-uniform
    const int m = (int)(cb & ~TK_UNFILTERED);
    const Key* src = block_out + (int64_t)b * cap;
    for (int j0 = 0; j0 < m; j0 += blockDim.x) {  // block-uniform trip count (warp appends)
      const int j = j0 + threadIdx.x;
      Key x;
      bool keep = false;
      if (j < m) {
        x = ld_key_cg(src + j);
        keep = !kless(T, x);
      }
      const int slot = warp_append(&ctr[TK_SURV_CTR], keep);
      if (slot >= 0) surv[slot] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(&ctr[TK_FIN_CTR], 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  if (threadIdx.x == 0) S.cap = cap;
  __syncthreads();
  bound_rank(S, k, mins, ctr, block_out, cap, surv, out_s, out_i, n_valid, wvalid, g_trace, nblk, false);
}
#endif  // LS_MAIN_TU

// Fused pass: score every record, keep the block's k best, then merge the
// block lists in a two-level tree inside the same launch: the last block of
// each group of TK_GROUP merges its group, the last group merger writes the
// final k (threadfence + ticket counters; no second kernel).
template <int TM, int RM, int MODE, int SRC>
__global__ void __launch_bounds__(TPB, min_blocks(TM, RM, MODE)) score_topk_kernel(
    const DTask* __restrict__ gtask, const void* __restrict__ src, int pbytes, int64_t n, int64_t base_index, int k,
    Key* __restrict__ block_out, Key* __restrict__ group_out, unsigned int* __restrict__ tickets,
    double* __restrict__ out_s, int64_t* __restrict__ out_i, unsigned long long* __restrict__ n_valid, int cap,
    Key* __restrict__ mins, unsigned long long* __restrict__ wvalid, unsigned long long* __restrict__ g_trace,
    int merge) {
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
  // bound merge: the block minimum goes out after R0 rounds (~LS_BOUND_C expected survivors:
  // a sample of grid * TPB * R0 keys puts T near the k / sample quantile), or at the end
  const int64_t R0 = mins ? bound_rounds(n, k, gridDim.x) : 0;
  bool published = false;
  uint64_t xn = 0;  // space path: the next point, loaded one round ahead
  __shared__ __align__(16) uint4 s_pts[SRC == 2 ? 2 : 1][SRC == 2 ? PTS_STAGE_LOADS + 1 : 1];
  uint4 pv = make_uint4(0u, 0u, 0u, 0u);  // SRC 2: this thread's 16 bytes of the next round
  if constexpr (SRC == 2)
    pv = load_round_chunk(src, pbytes, base, n);
  else if constexpr (MODE == 4 || MODE == 5)
    xn = load_point_warp(src, pbytes, base, n);
  // two passes over the same loop: rounds [0, R0), the bound publication (no call inside the
  // hot loop: a call's clobbers would spill the loop state), then the rest
  int64_t r = 0;
  for (int pass = 0; pass < 2; ++pass) {
  const int64_t r_end = pass == 0 ? R0 : INT64_MAX;
  for (; base < n && r < r_end; ++r) {
    const bool dyn = r + 2 >= st_rounds;  // block-uniform: round r + 2 is dynamic
    if (dyn && threadIdx.x == 0) s_nb[r & 1] = round_base(r + 2);
    const int64_t i = base + threadIdx.x;
    bool has = false;
    Key key;
    uint64_t x = 0;
    if constexpr (SRC == 2) {  // the round's points through shared memory (block-uniform)
      if ((int)threadIdx.x < pbytes * TPB / 16) s_pts[r & 1][threadIdx.x] = pv;
      __syncthreads();
      x = staged_point(s_pts[r & 1], pbytes);
      pv = load_round_chunk(src, pbytes, nb, n);
    } else if constexpr (MODE == 4 || MODE == 5) {  // every lane (warp-cooperative load)
      x = xn;
      xn = load_point_warp(src, pbytes, nb, n);
    }
    if (i < n) {
      ls_record r_;
      uint32_t kt[4];
      double f[LS_NFEAT_GPU];
      double s;
      int st;
      if constexpr (MODE == 4 || MODE == 5) {
        st = eval_space_mode<TM, MODE>(T, tab, x, ev.fc, f, &s);
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
  if (pass == 0 && r == R0 && R0 > 0) {  // block-uniform
    bound_publish(S, k, mins, tickets, block_out + (int64_t)blockIdx.x * cap, g_trace);
    published = true;
  }
  }
  for (int off = 16; off > 0; off >>= 1) valid += __shfl_down_sync(0xffffffffu, valid, off);
  if ((threadIdx.x & 31) == 0 && valid) atomicAdd(wvalid, (unsigned long long)valid);
  __syncthreads();
  trace_mark(g_trace, 2);
  if (mins) {  // bound merge: ranked by the last block (merge == MERGE_BOUND) or bound_merge_kernel
    if (!published) bound_publish(S, k, mins, tickets, block_out + (int64_t)blockIdx.x * cap, g_trace);
    bound_finish(S, k, mins, tickets, block_out, cap, group_out, out_s, out_i, n_valid, wvalid, g_trace,
                 merge == MERGE_BOUND);
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
  trace_mark(g_trace, 4);
  if (ngroups > 1) {  // one group (grid <= TK_GROUP): its merger already holds the final k
    write_keys(S, kept, k, group_out + (int64_t)g * k);
    // ---- level 2: last group merger writes the final list
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(&tickets[ngroups], 1u);
    __syncthreads();
    if (s_ticket != (unsigned)(ngroups - 1)) return;
    __threadfence();
    kept = merge_into(S, group_out, (int64_t)ngroups * k, k, false);
  }
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
#ifdef LS_MAIN_TU
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
#endif  // LS_MAIN_TU

#ifdef LS_MAIN_TU
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
#endif  // LS_MAIN_TU

// Body-replication factor of every transformable record (U_inner, or all
// unrolled extents when no loop branches), into an open-addressing set.
#ifdef LS_MAIN_TU
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
#endif  // LS_MAIN_TU

// The cache model's inexact-footprint flag per record (CacheModel.run -> NodeCost.inexact) and the
// (loop, tensor) pairs of its diagnostic (ls/cache.py:198-202: "inexact footprint for tensor ...
// at loop ..."): at each loop of the chain, innermost first, a tensor is inexact when one of its
// dimensions' strided intervals (_si_sum / _si_union folds, ls/cache.py:47-77) lost exactness for
// the loop's single set (the variables inside it) or its full set (those and its own).  A
// dimension's interval changes only where the walk passes one of its variables, so each level
// refolds only the dimensions of that variable (the generic walk's expr_range + _si_union).
// flags: 0 exact, 1 inexact, 255 the record fails apply_schedule; masks (optional): bit
// 8 * position + tensor, two words; chains (optional): the loop slot at each chain position
// (position 0 outermost), 0xFF past the chain.
#ifdef LS_MAIN_TU
__global__ void __launch_bounds__(TPB) inexact_kernel(const DTask* __restrict__ gtask, const ls_record* __restrict__ recs,
                                                      int64_t n, uint8_t* __restrict__ out,
                                                      unsigned long long* __restrict__ masks,
                                                      uint8_t* __restrict__ chains) {
  extern __shared__ __align__(16) unsigned char dyn[];
  DTask& T = *reinterpret_cast<DTask*>(dyn);
  stage_task(T, gtask);
  Cand c = carve(dyn + T.task_bytes, T);
  auto dim_exact = [&](int t, int rr, int thr) {
    SI u = expr_range(T, T.expr[T.t_uacc[t][0]][rr], c, thr);
    for (int a = 1; a < T.t_nu[t]; ++a) u = si_union(u, expr_range(T, T.expr[T.t_uacc[t][a]][rr], c, thr));
    return u.exact != 0;
  };
  for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    const ls_record r = load_record(recs, i);
    unsigned long long m0 = 0, m1 = 0;
    if (apply_transforms(T, r, c)) {
      out[i] = 255;
    } else {
      unsigned long long ex = 0;  // bit t * MAXRANK + rr: the dimension's current interval is exact
      for (int t = 0; t < T.n_tensors; ++t)
        for (int rr = 0; rr < T.t_rank[t]; ++rr)
          if (dim_exact(t, rr, (int)NOSLOT)) ex |= 1ull << (t * MAXRANK + rr);  // nothing expanded
      for (int p = c.n - 1; p >= 0; --p) {  // innermost first
        const int v = c.C(p);
        for (int t = 0; t < T.n_tensors; ++t) {
          bool bad = false;
          for (int rr = 0; rr < T.t_rank[t]; ++rr) {
            const int D = t * T.layout_rm + rr, b = t * MAXRANK + rr;
            bool mine = false;
            for (int x = 0; x < T.dim_nv[D]; ++x) mine |= T.dim_var[D][x] == v;
            bad |= !((ex >> b) & 1ull);                       // the single set
            if (mine) {
              if (dim_exact(t, rr, p)) ex |= 1ull << b;
              else ex &= ~(1ull << b);
            }
            bad |= !((ex >> b) & 1ull);                       // the full set
          }
          if (bad) {
            const int bit = 8 * p + t;
            if (bit < 64) m0 |= 1ull << bit;
            else m1 |= 1ull << (bit - 64);
          }
        }
      }
      out[i] = (m0 | m1) ? 1 : 0;
    }
    if (masks) {
      masks[2 * i] = m0;
      masks[2 * i + 1] = m1;
    }
    if (chains)
      for (int p = 0; p < 16; ++p) chains[16 * i + p] = out[i] != 255 && p < c.n ? c.C(p) : (uint8_t)0xFF;
  }
}
#endif  // LS_MAIN_TU

// ---------------------------------------------------------------------------
// host: task construction
// ---------------------------------------------------------------------------

#include "es_dev.cuh"

// ---------------------------------------------------------------------------
// Kernel selection: the scoring / ES kernels of each path are instantiated in
// their own translation unit (k_*.cu, compiled in parallel); the host code
// reaches them through these getters.
// ---------------------------------------------------------------------------
using ScoreFn = void (*)(const DTask*, const void*, int, int64_t, double*, double*, int32_t*);
using TopkFn = void (*)(const DTask*, const void*, int, int64_t, int64_t, int, Key*, Key*, unsigned int*, double*,
                       int64_t*, unsigned long long*, int, Key*, unsigned long long*, unsigned long long*, int);
using EsGenFn = void (*)(const DTask*, EsDev*, int);
ScoreFn k_score_fn(const DTask& T, int mode, int src);  // k_generic.cu (0), k_tab.cu (1-3), k_space.cu (4, 5), k_tree.cu (6)
TopkFn k_topk_fn(const DTask& T, int mode, int src);
EsGenFn k_es_gen_fn(const DTask& T, int mode);
ScoreFn k_score_fn_generic(const DTask& T, int src);
TopkFn k_topk_fn_generic(const DTask& T, int src);
EsGenFn k_es_gen_fn_generic(const DTask& T);
ScoreFn k_score_fn_tab(const DTask& T, int mode, int src);
TopkFn k_topk_fn_tab(const DTask& T, int mode, int src);
EsGenFn k_es_gen_fn_tab(const DTask& T, int mode);
ScoreFn k_score_fn_space4(const DTask& T);
TopkFn k_topk_fn_space4(const DTask& T, int src);
EsGenFn k_es_gen_fn_space4(const DTask& T);
ScoreFn k_score_fn_space5(const DTask& T);
TopkFn k_topk_fn_space5(const DTask& T, int src);
EsGenFn k_es_gen_fn_space5(const DTask& T);
ScoreFn k_score_fn_tree(int src);
TopkFn k_topk_fn_tree(int src);
EsGenFn k_es_gen_fn_tree();
