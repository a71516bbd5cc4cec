// loopscout_b200 engine, host side: the C-ABI of include/loopscout_b200.h,
// task packing/precomputation, launches.  Device code: dev.cuh (scoring,
// top-k, merges) and es_dev.cuh (ES); the per-path kernels are instantiated
// in k_*.cu.
#define LS_MAIN_TU
#include "dev.cuh"

#include <dlfcn.h>
#include <chrono>
#include <nvtx3/nvToolsExt.h>

// NVTX range over every public scoring / merge / ES entry point (header-only NVTX3: no cost
// unless a profiler is attached): ncu / Nsight timelines show the C-ABI calls by name.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define LS_NVTX(name) NvtxRange ls_nvtx_range_(name)

ScoreFn k_score_fn(const DTask& T, int mode, int src) {
  switch (mode) {
    case 0: return k_score_fn_generic(T, src);
    case 4: return k_score_fn_space4(T);
    case 5: return k_score_fn_space5(T);
    case 6: return k_score_fn_tree(src);
    default: return k_score_fn_tab(T, mode, src);
  }
}
TopkFn k_topk_fn(const DTask& T, int mode, int src) {
  switch (mode) {
    case 0: return k_topk_fn_generic(T, src);
    case 4: return k_topk_fn_space4(T, src);
    case 5: return k_topk_fn_space5(T, src);
    case 6: return k_topk_fn_tree(src);
    default: return k_topk_fn_tab(T, mode, src);
  }
}
EsGenFn k_es_gen_fn(const DTask& T, int mode) {
  switch (mode) {
    case 0: return k_es_gen_fn_generic(T);
    case 4: return k_es_gen_fn_space4(T);
    case 5: return k_es_gen_fn_space5(T);
    case 6: return k_es_gen_fn_tree();
    default: return k_es_gen_fn_tab(T, mode);
  }
}

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
// Tile-point rows of the packed walk (MODE 5): eligible when the reorder
// axis (if any) is the last axis, there are at most 4 tile axes and 2^16 tile points, the
// space has fewer than 2^32 points and every outer extent fits 16 bits.  Row = 8 words:
// F | ceil(E/F) << 16 per tile axis (all zero when a factor is out of range), then the packed
// first-row group offsets per tensor.
bool plan_tile_points(DTask& T, const std::vector<uint64_t>& ext, std::vector<uint32_t>& rows) {
  T.sp_tp_ok = 0;
  if (!T.sp_static || !T.sp_pack) return false;
  int tile[LS_MAX_AXES], nt = 0, pax = -1;
  double total = 1;
  for (int a = 0; a < T.sp_n; ++a) {
    total *= T.sp_ax[a].n;
    if (T.sp_ax[a].kind == LS_AX_PERM) {
      if (a != T.sp_n - 1) return false;
      pax = a;
    } else if (T.sp_ax[a].kind == LS_AX_PARAM) {
      tile[nt++] = a;
    } else {
      return false;
    }
  }
  if (nt < 1 || nt > 4 || total >= 4294967296.0) return false;
  int64_t ntp = 1;
  for (int j = 0; j < nt; ++j) ntp *= T.sp_ax[tile[j]].n;
  if (ntp > 65536) return false;
  rows.assign((size_t)ntp * 8, 0u);
  for (int64_t tp = 0; tp < ntp; ++tp) {
    uint32_t* r = &rows[(size_t)tp * 8];
    int64_t rest = tp;
    uint32_t kp[4];
    for (int t = 0; t < 4; ++t) kp[t] = T.sd_offp[t];
    bool bad = false;
    for (int j = nt - 1; j >= 0; --j) {  // the last tile axis is the least significant digit
      const DAxis& ax = T.sp_ax[tile[j]];
      const uint32_t ch = (uint32_t)(rest % ax.n);
      rest /= ax.n;
      const uint64_t e = ext[ax.voff + ch];
      if (e >> 63) bad = true;
      const uint64_t outer = (e >> 16) & 0x7FFFFFFFull;
      if (!bad && outer > 0xFFFFu) return false;
      r[j] = (uint32_t)(e & 0xFFFFu) | ((uint32_t)outer << 16);
      for (int t = 0; t < 4; ++t) kp[t] += ch * T.sd_Sp[tile[j]][t];
    }
    if (bad) {
      for (int q = 0; q < 8; ++q) r[q] = 0;
      continue;
    }
    for (int t = 0; t < 4; ++t) r[4 + t] = kp[t];
  }
  for (int j = 0; j < nt; ++j) {
    T.sp_tj_new[j] = T.sp_tnew[tile[j]];
    T.sp_tj_slot[j] = T.sp_tslot[tile[j]];
  }
  T.sp_ntile = nt;
  T.sp_pax = pax;
  T.sp_total = (uint32_t)total;
  return true;
}

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
  auto collect = [&](int t, int* dims, uint32_t* pmask) {  // the tensor's dimensions whose count varies
    int nd = 0;
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
    return nd;
  };
  // entries of split `sel` (bit j: dimension j goes to group 1), -1 when a group has > 6 bits
  auto entries = [&](int nd, const int* dims, const uint32_t* pmask, int sel) -> int64_t {
    int64_t total = 0;
    for (int j = 0; j < 2; ++j) {
      uint32_t pm = 0;
      int nb = 0, members = 0;
      for (int q = 0; q < nd; ++q)
        if (((sel >> q) & 1) == j) pm |= pmask[q], nb += T.dim_nv[dims[q]], ++members;
      if (!members) continue;
      if (nb > 6) return -1;
      int64_t keys = 1;
      for (int a = 0; a < T.sp_n; ++a)
        if (T.sp_ax[a].kind == LS_AX_PARAM && ((pm >> T.sp_ax[a].param) & 1u)) keys *= T.sp_ax[a].n;
      total += keys * sd_row_len(nb);
      if (total > SD_MAX_ENTRIES) return -1;
    }
    return total;
  };
  // per tensor: the split with the fewest entries.  (LS_SD_SINGLE=1: then, while the whole table
  // stays within SD_MAX_ENTRIES, single-group splits -- one random lookup per level for that
  // tensor, the empty group reading the broadcast ones row; measured slower on the BASELINE
  // spaces: the larger tables cost more than the lookups they save.)
  int chosen[4] = {0, 0, 0, 0};
  int64_t cost[4] = {0, 0, 0, 0}, single_cost[4] = {-1, -1, -1, -1};
  for (int t = 0; t < T.n_tensors; ++t) {
    int dims[4];
    uint32_t pmask[4];
    const int nd = collect(t, dims, pmask);
    int64_t best = -1;
    for (int sel = 0; sel < (1 << nd); ++sel) {
      if (nd && (sel >> (nd - 1)) & 1) continue;  // symmetric splits: the last dimension stays in group 0
      const int64_t total = entries(nd, dims, pmask, sel);
      if (total >= 0 && (best < 0 || total < best)) best = total, chosen[t] = sel;
    }
    if (best < 0) return false;
    cost[t] = best;
    single_cost[t] = entries(nd, dims, pmask, 0);
  }
  {
    static const bool prefer_single = [] {
      const char* e = getenv("LS_SD_SINGLE");
      return e && e[0] == '1';
    }();
    int64_t total = 4;
    for (int t = 0; t < T.n_tensors; ++t) total += cost[t];
    for (int t = 0; t < T.n_tensors && prefer_single; ++t)
      if (chosen[t] && single_cost[t] >= 0 && total - cost[t] + single_cost[t] <= SD_MAX_ENTRIES) {
        total += single_cost[t] - cost[t];
        chosen[t] = 0;
      }
  }
  for (int t = 0; t < T.n_tensors; ++t) {
    int dims[4];
    uint32_t pmask[4];
    const int nd = collect(t, dims, pmask);
    const int best_sel = chosen[t];
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
        T.sd_S[a][G] = (uint32_t)(keys * sd_row_len(nb) * 4);
        keys *= ax.n;
      }
      if (off + keys * sd_row_len(nb) > SD_MAX_ENTRIES) return false;
      T.sd_off[G] = (uint32_t)(off * 4);
      rows[G] = (int32_t)keys;
      off += keys * sd_row_len(nb);
    }
  }
  T.sd_len = (int32_t)off;
  // packed walk (MODE 5): both group offsets of a tensor in one word when every offset fits 16 bits
  memset(T.sd_offp, 0, sizeof(T.sd_offp));
  memset(T.sd_Sp, 0, sizeof(T.sd_Sp));
  memset(T.sp_vbp, 0, sizeof(T.sp_vbp));
  memset(T.sp_vbp3, 0, sizeof(T.sp_vbp3));
  T.sp_pack = off * 4 <= 0xFFFF;
  for (int t = 0; t < 4; ++t) {
    T.sd_offp[t] = T.sd_off[2 * t] | (T.sd_off[2 * t + 1] << 16);
    for (int a = 0; a < T.sp_n; ++a) T.sd_Sp[a][t] = T.sd_S[a][2 * t] | (T.sd_S[a][2 * t + 1] << 16);
  }
  for (int v = 0; v < NSLOT; ++v) {
    uint32_t pk[4];
    for (int t = 0; t < 4; ++t)
      pk[t] = (uint32_t)((T.vb8[v] >> (16 * t)) & 0xFFu) | ((uint32_t)((T.vb8[v] >> (16 * t + 8)) & 0xFFu) << 16);
    T.sp_vbp[v][0] = pk[0];
    T.sp_vbp[v][1] = pk[1];
    T.sp_vbp[v][2] = pk[2];
    T.sp_vbp3[v] = pk[3];
    uint32_t use = 0;
    for (int t = 0; t < T.n_tensors; ++t) use |= ((T.t_vmask[t] >> v) & 1u) << t;
    T.sp_vbp[v][3] = use;
  }
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
    len *= tab_row_len(nv);  // rows of 2^nv stage masks + padding (bank skew, like the group tables)
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

ScoreFn score_fn(const DTask& T, int mode, int pbytes) { return k_score_fn(T, mode, pbytes ? 1 : 0); }

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
  LS_NVTX("ls_task_create");
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

int ls_inexact_footprints(ls_task* t, const ls_record* d_records, int64_t n, uint8_t* d_flags,
                          unsigned long long* d_masks, uint8_t* d_chains, void* stream) {
  LS_NVTX("ls_inexact_footprints");
  if (!t || n < 0 || (n && (!d_records || !d_flags))) return fail(LS_E_ARG, "bad argument");
  if (t->host.tree) return fail(LS_E_UNSUPPORTED, "inexact-footprint flags cover perfect chains (not general trees)");
  if (!n) return LS_E_OK;
  CUDA_TRY(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = smem_score(t->host, 0);
  BPS_TRY(bps, inexact_kernel, sm);
  inexact_kernel<<<grid_for(t, n, bps), TPB, sm, s>>>(t->d_task, d_records, n, d_flags, d_masks, d_chains);
  CUDA_TRY(cudaGetLastError());
  return LS_E_OK;
}

int ls_collect_unroll(ls_task* t, const ls_record* d_records, int64_t n, int64_t* h_values, int32_t cap,
                      int32_t* h_count, void* stream) {
  LS_NVTX("ls_collect_unroll");
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
  LS_NVTX("ls_score");
  if (!t || n < 0 || (n && !d_records)) return fail(LS_E_ARG, "bad argument");
  if (n == 0) return LS_E_OK;
  CUDA_TRY(cudaSetDevice(t->device));
  return score_device(t, d_records, 0, n, d_scores, d_features, d_status, (cudaStream_t)stream);
}

static int check_points(const ls_task* t, int32_t pbytes) {
  if (pbytes != 3 && pbytes != 4 && pbytes != 8) return fail(LS_E_ARG, "point_bytes must be 3, 4 or 8");
  if (t->host.sp_n < 1) return fail(LS_E_ARG, "no schedule space attached (ls_task_set_space)");
  return LS_E_OK;
}

int ls_score_points(ls_task* t, const void* d_points, int32_t pbytes, int64_t n, double* d_scores,
                    double* d_features, int32_t* d_status, void* stream) {
  LS_NVTX("ls_score_points");
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

// Phase timestamps of one fused launch to stderr (LS_TRACE=1, profiling aid).
static int print_trace(unsigned long long* tr, int grid, int64_t n, bool two, cudaStream_t s) {
    std::vector<unsigned long long> h((size_t)TR_SLOTS * grid);
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaMemcpy(h.data(), tr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, surv = 0;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[b * TR_SLOTS]);
    for (int b = 0; b < grid; ++b)
      if (h[b * TR_SLOTS + 7] >> 63) surv = h[b * TR_SLOTS + 7] & ~(1ull << 63), h[b * TR_SLOTS + 7] = 0;
    double avg[TR_SLOTS] = {0}, mx[TR_SLOTS] = {0};
    for (int q = 0; q < TR_SLOTS; ++q) {
      if (q == 8) continue;
      int cnt = 0;
      for (int b = 0; b < grid; ++b)
        if (h[b * TR_SLOTS + q] > t0) {
          const double v = (double)(h[b * TR_SLOTS + q] - t0) / 1e3;
          avg[q] += v, mx[q] = std::max(mx[q], v), ++cnt;
        }
      if (cnt) avg[q] /= cnt;
    }
    if (two)
      fprintf(stderr, "LS_TRACE n=%lld grid=%d us(avg/max): staged %.1f/%.1f main %.1f/%.1f | bound merge: T out %.1f "
              "filtered %.1f/%.1f last block %.1f (controls %.1f loaded %.1f ranked %.1f) final %.1f survivors %llu\n",
              (long long)n, grid, avg[1], mx[1], avg[2], mx[2], mx[4], avg[3], mx[3], mx[5], mx[9], mx[10], mx[11],
              mx[6], surv);
    else
      fprintf(stderr, "LS_TRACE n=%lld grid=%d us(avg/max): staged %.1f/%.1f main %.1f/%.1f listed %.1f/%.1f | "
              "tree group %.1f final %.1f\n", (long long)n, grid, avg[1], mx[1], avg[2], mx[2], avg[3], mx[3], mx[4],
              mx[5]);
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
    return LS_E_OK;
}

static int topk_device(ls_task* t, const void* d_src, int pbytes, int64_t n, int64_t base_index, int32_t k,
                       double* d_top_scores, int64_t* d_top_index, unsigned long long* d_valid, cudaStream_t s,
                       void* h_out = nullptr, void* h_out_dev = nullptr, bool host_points = false) {
  const int mode = mode_of(t, pbytes != 0);
  // points in mapped host memory (16-byte aligned) on the space paths: block-cooperative loads
  const bool coop = host_points && (mode == 4 || mode == 5) && (reinterpret_cast<uintptr_t>(d_src) & 15) == 0;
  const TopkFn fn = k_topk_fn(t->host, mode, coop ? 2 : pbytes ? 1 : 0);
  const size_t sm = smem_topk(t->host, k, mode);
  BPS_TRY(bps, fn, sm);
  const int grid = n > 0 ? grid_for(t, n, bps) : 1;
  const int ngroups = (grid + TK_GROUP - 1) / TK_GROUP;
  // bound merge (block-minima bound, survivors ranked by the last block) when the grid has
  // plenty of blocks per answer key; else the in-kernel merge tree
  static const int merge_env = [] {  // LS_MERGE=tree|bound forces a merge (tests / profiling aid)
    const char* e = getenv("LS_MERGE");
    return !e ? 0 : (e[0] == 't' ? 1 : e[0] == 'b' ? 2 : 0);
  }();
  bool two = 4 * k <= grid && grid <= topk_buf(k) && grid <= TK_MAXGRID;
  if (merge_env == 1) two = false;
  const int merge = !two ? MERGE_TREE
                    : (merge_env == 2 || bound_inline_rank(n, k, grid)) ? MERGE_BOUND : MERGE_BOUND_K2;
  // bound merge: [grid] buffers of topk_buf(k) keys (parked / unfiltered lists) and as many
  // survivor slots (a block appends at most its buffer)
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
  Key* group_out = block_out + (size_t)grid * (two ? topk_buf(k) : k);  // tree: group lists; bound merge: survivors
  Key* mins = two ? reinterpret_cast<Key*>(ws + WS_CTR_BYTES) : nullptr;
  unsigned char* out = ws + WS_FIXED_BYTES + keys_bytes;
  if (h_out) {  // results to a pinned host block: written by the kernel through its device
                // alias when it has one (no copy), else staged in the workspace and copied
    unsigned char* o = h_out_dev ? reinterpret_cast<unsigned char*>(h_out_dev) : out;
    d_valid = reinterpret_cast<unsigned long long*>(o);
    d_top_scores = reinterpret_cast<double*>(o + 16);
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
                           d_top_index, d_valid, topk_buf(k), mins, wvalid, tr, merge);
  CUDA_TRY(cudaGetLastError());
  if (merge == MERGE_BOUND_K2) {
    const size_t msm = topk_state_bytes(topk_buf(k));
    if (kernel_prepare(bound_merge_kernel, msm, false) < 0) return LS_E_CUDA;
    // programmatic dependent launch: queued behind the scoring grid's tail (its blocks wait in
    // griddepcontrol.wait for the grid's completion and memory), not a full kernel boundary
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min(grid, t->num_sms));
    cfg.blockDim = dim3(TPB);
    cfg.dynamicSmemBytes = msm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const Key* cbo = block_out;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, bound_merge_kernel, mins, tickets, cbo, grid, k, topk_buf(k), group_out,
                                d_top_scores, d_top_index, d_valid, wvalid, tr));
  }
  if (h_out && !h_out_dev) CUDA_TRY(cudaMemcpyAsync(h_out, out, out_bytes, cudaMemcpyDeviceToHost, s));
  L.ok = true;
  if (tr)
    if (int rc = print_trace(tr, grid, n, two, s)) return rc;
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
  LS_NVTX("ls_score_topk");
  if (!t || n < 0 || (n && !d_records) || !d_top_scores || !d_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  return score_topk_any(t, d_records, 0, n, base_index, k, d_top_scores, d_top_index, d_n_valid,
                        (cudaStream_t)stream);
}

int ls_score_topk_points(ls_task* t, const void* d_points, int32_t pbytes, int64_t n, int64_t base_index, int32_t k,
                         double* d_top_scores, int64_t* d_top_index, int64_t* d_n_valid, void* stream) {
  LS_NVTX("ls_score_topk_points");
  if (!t || n < 0 || (n && !d_points) || !d_top_scores || !d_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  if (int rc = check_points(t, pbytes)) return rc;
  return score_topk_any(t, d_points, pbytes, n, base_index, k, d_top_scores, d_top_index, d_n_valid,
                        (cudaStream_t)stream);
}

int ls_task_set_space(ls_task* t, const ls_space_desc* sp) {
  LS_NVTX("ls_task_set_space");
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
  t->host.sp_tp_ok = 0;
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
      uint64_t* drch = nullptr;
      uint4* dcrow = nullptr;
      CUDA_TRY(cudaMalloc(&dcrow, sizeof(uint4) * np));
      t->retired.push_back(dcrow);
      CUDA_TRY(cudaMalloc(&dch, sizeof(uint64_t) * np));
      t->retired.push_back(dch);
      CUDA_TRY(cudaMalloc(&drch, sizeof(uint64_t) * np));
      t->retired.push_back(drch);
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
      build_pchain_kernel<<<(np + TPB - 1) / TPB, TPB, sm>>>(t->d_task, pax, dch, dst, drch, dcrow);
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
        // (MODE 5 also packs both group offsets of a tensor into one word: every offset < 2^16)
        t->host.sp_narrow = fits && fsum < 4294967295.0 && prod * (t->host.sp_nchain + 1) < 4294967295.0 &&
                            t->host.sp_pack;
      }
      t->host.sp_chain = dch;
      t->host.sp_rchain = drch;
      t->host.sp_crow = dcrow;
      std::vector<uint32_t> tprows;
      if (t->host.sp_narrow && plan_tile_points(t->host, ext, tprows)) {
        uint4* dtp = nullptr;
        CUDA_TRY(cudaMalloc(&dtp, sizeof(uint32_t) * tprows.size()));
        t->retired.push_back(dtp);
        CUDA_TRY(cudaMemcpy(dtp, tprows.data(), sizeof(uint32_t) * tprows.size(), cudaMemcpyHostToDevice));
        t->host.sp_tp = dtp;
        t->host.sp_tp_ok = 1;
      }
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
  LS_NVTX("ls_topk_merge");
  if (!d_scores || !d_index || n_lists < 0 || k_in < 0 || k_out < 1 || k_out > TK_MAXK || !d_out_scores ||
      !d_out_index)
    return fail(LS_E_ARG, "bad argument");
  return merge_launch(nullptr, d_scores, d_index, (int64_t)n_lists * k_in, k_out, d_out_scores, d_out_index,
                      (cudaStream_t)stream);
}

int ls_topk_merge_keys(const ls_topk_key* d_keys, int64_t m, int32_t k_out, double* d_out_scores,
                       int64_t* d_out_index, void* stream) {
  LS_NVTX("ls_topk_merge_keys");
  if ((m > 0 && !d_keys) || m < 0 || k_out < 1 || k_out > TK_MAXK || !d_out_scores || !d_out_index)
    return fail(LS_E_ARG, "bad argument");
  static_assert(sizeof(ls_topk_key) == sizeof(Key), "ls_topk_key layout");
  return merge_launch(reinterpret_cast<const Key*>(d_keys), nullptr, nullptr, m, k_out, d_out_scores, d_out_index,
                      (cudaStream_t)stream);
}

// ncclAllGather, bound at run time (no link-time NCCL dependency): the process's libnccl.so.2
// (torch's, when loaded) or the system one.
using NcclAllGatherFn = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
static NcclAllGatherFn nccl_all_gather() {
  static NcclAllGatherFn fn = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<NcclAllGatherFn>(dlsym(h, "ncclAllGather")) : nullptr;
  }();
  return fn;
}

int ls_topk_allgather_merge(void* nccl_comm, int32_t rank, int32_t world, const double* d_scores,
                            const int64_t* d_index, int32_t k, ls_topk_key* d_scratch, double* d_out_scores,
                            int64_t* d_out_index, void* stream) {
  LS_NVTX("ls_topk_allgather_merge");
  if (!nccl_comm || world < 1 || rank < 0 || rank >= world || k < 1 || k > TK_MAXK || !d_scores || !d_index ||
      !d_scratch || !d_out_scores || !d_out_index)
    return fail(LS_E_ARG, "bad argument");
  const NcclAllGatherFn ag = nccl_all_gather();
  if (!ag) return fail(LS_E_UNSUPPORTED, "libnccl.so.2 (ncclAllGather) is not available");
  const cudaStream_t s = (cudaStream_t)stream;
  ls_topk_key* mine = d_scratch + (size_t)rank * k;
  if (int rc = ls_topk_to_keys(d_scores, d_index, k, mine, stream)) return rc;
  constexpr int kNcclUint8 = 1;  // ncclDataType_t
  if (int r = ag(mine, d_scratch, sizeof(ls_topk_key) * (size_t)k, kNcclUint8, nccl_comm, s))
    return fail(LS_E_CUDA, "ncclAllGather failed: ncclResult_t " + std::to_string(r));
  return ls_topk_merge_keys(d_scratch, (int64_t)world * k, k, d_out_scores, d_out_index, stream);
}

int ls_topk_to_keys(const double* d_scores, const int64_t* d_index, int64_t m, ls_topk_key* d_keys, void* stream) {
  LS_NVTX("ls_topk_to_keys");
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
  // pinned staging block: count (16 B slot) | scores | indices, written by the kernel through the
  // block's device alias (else filled by one D2H copy); the task's
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
  // cudaMallocHost memory is mapped at the same address under unified addressing (every 64-bit
  // platform CUDA supports): the kernel writes the results straight into the block
  static const bool host_trace = getenv("LS_HOST_TRACE") != nullptr;  // host-side phase times (profiling aid)
  const auto h0 = std::chrono::steady_clock::now();
  const int rc = topk_device(t, d_alias, pbytes, n, base_index, k, nullptr, nullptr, nullptr, s, S.p, S.p,
                             pbytes != 0);
  if (rc != LS_E_OK) return rc;
  const auto h1 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaStreamSynchronize(s));
  if (host_trace) {
    const auto h2 = std::chrono::steady_clock::now();
    fprintf(stderr, "LS_HOST_TRACE enqueue %.1f us, synchronize %.1f us\n",
            std::chrono::duration<double, std::micro>(h1 - h0).count(),
            std::chrono::duration<double, std::micro>(h2 - h1).count());
  }
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
  static const bool staged_env = [] {  // LS_HOST_PATH=staged forces the staged copies (tests / profiling aid)
    const char* e = getenv("LS_HOST_PATH");
    return e && e[0] == 's';
  }();
  if (n > 0 && !staged_env)
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
  LS_NVTX("ls_score_topk_host");
  if (!t || n < 0 || (n && !h_records) || !h_top_scores || !h_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  return score_topk_host_any(t, h_records, 0, n, base_index, k, h_top_scores, h_top_index, h_n_valid,
                             (cudaStream_t)stream);
}

int ls_score_topk_points_host(ls_task* t, const void* h_points, int32_t pbytes, int64_t n, int64_t base_index,
                              int32_t k, double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid,
                              void* stream) {
  LS_NVTX("ls_score_topk_points_host");
  if (!t || n < 0 || (n && !h_points) || !h_top_scores || !h_top_index) return fail(LS_E_ARG, "bad argument");
  if (k < 1 || k > TK_MAXK) return fail(LS_E_ARG, "k must be in 1..1024");
  if (int rc = check_points(t, pbytes)) return rc;
  return score_topk_host_any(t, h_points, pbytes, n, base_index, k, h_top_scores, h_top_index, h_n_valid,
                             (cudaStream_t)stream);
}

}  // extern "C"

// ES generation loop on device
#include "es.cuh"
