// Host-side per-task block-cycle table.
//
// The mock emitter (ls/ir.py:557-659) produces only a handful of distinct
// basic blocks for a perfect loop chain: a one-instruction preamble and
// loop-header blocks (counter init), three-instruction latch blocks, the
// innermost block (the access body, replicated U times by unrolled inner
// loops, followed by its own latch) and the `ret` block.  Their cycle counts
// under schedule_block (ls/ilp.py:158-204) depend only on the task (target,
// dialect, latency table, access list) and on U, never on the candidate's tile
// factors or loop order, so they are computed here once per task instead of
// once per candidate (the reference re-schedules every block of every
// candidate, ls/ilp.py:262-271).
//
// The dependence rules are those of reg_effects / build_deps
// (ls/ilp.py:53-155), applied to the operand text the emitter would print.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/loopscout_b200.h"

namespace lsb {

struct Ins {
  int shape;
  std::string mn;
  std::vector<std::string> ops;
  std::string pred;
};

static bool has_prefix(const std::string& s, const char* p) { return s.rfind(p, 0) == 0; }

static std::string root_of(const std::string& mn) { return mn.substr(0, mn.find('.')); }

// register-like tokens of one operand: [%$#]?[A-Za-z_][\w.]*, immediates dropped
static std::vector<std::string> operand_regs(const std::string& op) {
  std::vector<std::string> out;
  auto alpha = [](char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; };
  auto word = [&](char c) { return alpha(c) || (c >= '0' && c <= '9') || c == '.'; };
  size_t i = 0;
  while (i < op.size()) {
    bool sig = (op[i] == '%' || op[i] == '$' || op[i] == '#') && i + 1 < op.size() && alpha(op[i + 1]);
    if (!sig && !alpha(op[i])) {
      ++i;
      continue;
    }
    size_t j = i + (sig ? 2 : 1);
    while (j < op.size() && word(op[j])) ++j;
    if (op[i] != '$' && op[i] != '#') {
      std::string t = op.substr(i, j - i);
      t = t.substr(0, t.find('.'));
      size_t k = t.find_first_not_of('%');
      out.push_back(k == std::string::npos ? std::string() : t.substr(k));
    }
    i = j;
  }
  return out;
}

static void effects(const Ins& in, int dialect, std::set<std::string>& rd, std::set<std::string>& wr) {
  const std::string& m = in.mn;
  std::string root = root_of(m);
  if (!in.pred.empty()) {
    size_t k = in.pred.find_first_not_of('%');
    std::string p = in.pred.substr(k);
    p = p.substr(std::min(p.size(), p.find_first_not_of('!')));
    rd.insert(p);
  }
  if (in.ops.empty() || root == "ret" || root == "jmp" || root == "bra" || root == "b" || root == "br" ||
      root[0] == 'j')
    return;
  int mem = -1;
  for (size_t i = 0; i < in.ops.size(); ++i)
    if (in.ops[i].find_first_of("([") != std::string::npos) {
      mem = (int)i;
      break;
    }
  bool st_like = has_prefix(m, "st") || has_prefix(m, "vst");
  bool store = st_like || (mem >= 0 && mem == (int)in.ops.size() - 1 &&
                           (has_prefix(m, "vmov") || has_prefix(m, "mov")));
  int dest = dialect == LS_DIALECT_X86_ATT ? (int)in.ops.size() - 1 : ((st_like && mem >= 0) ? mem : 0);
  bool rmw = has_prefix(m, "vfmadd") || has_prefix(m, "fma") || has_prefix(m, "fmla") ||
             has_prefix(m, "fmls") || has_prefix(m, "add") || has_prefix(m, "sub") || root == "add" ||
             root == "addq";
  for (size_t i = 0; i < in.ops.size(); ++i) {
    std::vector<std::string> regs = operand_regs(in.ops[i]);
    if ((int)i == mem) {
      rd.insert(regs.begin(), regs.end());
      std::string res = "mem:" + (regs.empty() ? std::string("abs") : regs[0]);
      if ((int)i == dest && store)
        wr.insert(res);
      else
        rd.insert(res);
      continue;
    }
    if ((int)i == dest && root != "cmp" && root != "cmpq" && root != "test") {
      wr.insert(regs.begin(), regs.end());
      if (rmw) rd.insert(regs.begin(), regs.end());
    } else {
      rd.insert(regs.begin(), regs.end());
    }
  }
}

// schedule_block: greedy in-order issue with RAW latencies, WAR/WAW order edges
int64_t schedule_block(const std::vector<Ins>& blk, const ls_task_desc& d) {
  const int n = (int)blk.size();
  if (n == 0) return 0;
  std::map<std::string, int> rid;
  auto id = [&](const std::string& s) {
    auto it = rid.find(s);
    if (it != rid.end()) return it->second;
    int v = (int)rid.size();
    rid.emplace(s, v);
    return v;
  };
  std::vector<std::vector<int>> R(n), Wr(n);
  for (int k = 0; k < n; ++k) {
    std::set<std::string> rd, wr;
    effects(blk[k], d.dialect, rd, wr);
    for (auto& s : rd) R[k].push_back(id(s));
    for (auto& s : wr) Wr[k].push_back(id(s));
  }
  const int nres = (int)rid.size();
  std::vector<int> last_w(nres, -1);
  std::vector<std::vector<int>> last_r(nres);
  std::vector<std::vector<int>> raw(n), ord(n);
  auto add_u = [](std::vector<int>& v, int x) {
    if (std::find(v.begin(), v.end(), x) == v.end()) v.push_back(x);
  };
  for (int k = 0; k < n; ++k) {
    for (int r : R[k])
      if (last_w[r] >= 0) add_u(raw[k], last_w[r]);
    for (int w : Wr[k]) {
      if (last_w[w] >= 0) add_u(ord[k], last_w[w]);
      for (int q : last_r[w])
        if (q != k) add_u(ord[k], q);
    }
    for (int w : Wr[k]) {
      last_w[w] = k;
      last_r[w].clear();
    }
    for (int r : R[k]) last_r[r].push_back(k);
  }
  for (int k = 0; k < n; ++k) {  // false edges minus true edges
    std::vector<int> keep;
    for (int p : ord[k])
      if (std::find(raw[k].begin(), raw[k].end(), p) == raw[k].end()) keep.push_back(p);
    ord[k].swap(keep);
  }
  std::vector<int64_t> issue(n, -1), lat(n);
  std::vector<int> cls(n);
  for (int k = 0; k < n; ++k) {
    lat[k] = d.lat[blk[k].shape];
    cls[k] = d.klass[blk[k].shape];
  }
  int done = 0, first = 0;
  int64_t cycle = 0;
  while (done < n) {
    int issued = 0;
    int used[LS_I_COUNT] = {0};
    while (first < n && issue[first] >= 0) ++first;
    for (int i = first; i < n && issued < d.issue_width; ++i) {
      if (issue[i] >= 0) continue;
      int64_t ready = 0;
      bool ok = true;
      for (int p : raw[i]) {
        if (issue[p] < 0) {
          ok = false;
          break;
        }
        ready = std::max(ready, issue[p] + lat[p]);
      }
      if (ok)
        for (int p : ord[i]) {
          if (issue[p] < 0) {
            ok = false;
            break;
          }
          ready = std::max(ready, issue[p] + 1);
        }
      if (!ok || ready > cycle) continue;
      int cap = d.unit_cap[cls[i]];
      if (cap > 0 && used[cls[i]] >= cap) continue;
      issue[i] = cycle;
      ++used[cls[i]];
      ++issued;
      ++done;
    }
    ++cycle;
  }
  int64_t fin = issue[0] + lat[0];
  for (int k = 1; k < n; ++k) fin = std::max(fin, issue[k] + lat[k]);
  return fin;
}

// ---- the emitter's block shapes for one target --------------------------------

static const char* kCtrX86[8] = {"%r8", "%r9", "%r10", "%r11", "%r12", "%r13", "%r14", "%r15"};
static const char* kCtrA64[8] = {"x8", "x9", "x10", "x11", "x12", "x13", "x14", "x15"};
static const char* kBaseX86[6] = {"%rax", "%rbx", "%rcx", "%rdx", "%rsi", "%rdi"};
static const char* kBaseA64[6] = {"x0", "x1", "x2", "x3", "x4", "x5"};
static const char* kBasePtx[6] = {"%rd1", "%rd2", "%rd3", "%rd4", "%rd5", "%rd6"};

static std::string fmt(const char* f, int a) {
  char b[48];
  snprintf(b, sizeof b, f, a);
  return b;
}

struct Emitter {
  int target;
  std::vector<Ins> out;
  int vreg = 0;

  std::string ctr(int depth) const { return target == LS_TARGET_AARCH64 ? kCtrA64[depth % 8] : kCtrX86[depth % 8]; }
  std::string base(int t) const {
    return target == LS_TARGET_X86 ? kBaseX86[t % 6] : target == LS_TARGET_AARCH64 ? kBaseA64[t % 6] : kBasePtx[t % 6];
  }
  void init(int depth) {
    if (target == LS_TARGET_X86)
      out.push_back({LS_I_INIT, "movq", {"$0", ctr(depth)}, ""});
    else if (target == LS_TARGET_AARCH64)
      out.push_back({LS_I_INIT, "mov", {ctr(depth), "#0"}, ""});
    else
      out.push_back({LS_I_INIT, "mov.u32", {ctr(depth), "0"}, ""});
  }
  void latch(int depth, int64_t extent, int lid) {
    std::string c = ctr(depth), e = std::to_string(extent);
    if (target == LS_TARGET_X86) {
      out.push_back({LS_I_ADD, "addq", {"$1", c}, ""});
      out.push_back({LS_I_CMP, "cmpq", {"$" + e, c}, ""});
      out.push_back({LS_I_BRANCH, "jne", {fmt(".LBB_%d", lid)}, ""});
    } else if (target == LS_TARGET_AARCH64) {
      out.push_back({LS_I_ADD, "add", {c, c, "#1"}, ""});
      out.push_back({LS_I_CMP, "cmp", {c, "#" + e}, ""});
      out.push_back({LS_I_BRANCH, "b.ne", {fmt(".LBB_%d", lid)}, ""});
    } else {
      out.push_back({LS_I_ADD, "add.s32", {c, c, "1"}, ""});
      out.push_back({LS_I_CMP, "setp.lt.s32", {fmt("%%p%d", lid), c, e}, ""});
      out.push_back({LS_I_BRANCH, "bra", {fmt("$L_%d", lid)}, fmt("%%p%d", lid)});
    }
  }
  void ret() { out.push_back({LS_I_RET, "ret", {}, ""}); }
  // one copy of the access body: loads, then fma + store per store (ls/ir.py:584-612)
  void body(const std::vector<int>& load_t, const std::vector<int>& store_t) {
    std::vector<int> regs;
    for (int t : load_t) {
      int r = vreg++ % 16;
      regs.push_back(r);
      if (target == LS_TARGET_X86)
        out.push_back({LS_I_LOAD, "vmovups", {"(" + base(t) + ")", fmt("%%zmm%d", r)}, ""});
      else if (target == LS_TARGET_AARCH64)
        out.push_back({LS_I_LOAD, "ld1", {fmt("{v%d.4s}", r), "[" + base(t) + "]"}, ""});
      else
        out.push_back({LS_I_LOAD, "ld.global.f32", {fmt("%%f%d", r), "[" + base(t) + "]"}, ""});
    }
    const int L = (int)regs.size();
    for (size_t j = 0; j < store_t.size(); ++j) {
      int acc = 16 + (int)(j % 8);
      int s1 = L ? regs[(2 * j) % L] : 0, s2 = L ? regs[(2 * j + 1) % L] : 1;
      std::string b = base(store_t[j]);
      if (target == LS_TARGET_X86) {
        out.push_back({LS_I_FMA, "vfmadd231ps", {fmt("%%zmm%d", s1), fmt("%%zmm%d", s2), fmt("%%zmm%d", acc)}, ""});
        out.push_back({LS_I_STORE, "vmovups", {fmt("%%zmm%d", acc), "(" + b + ")"}, ""});
      } else if (target == LS_TARGET_AARCH64) {
        out.push_back({LS_I_FMA, "fmla", {fmt("v%d.4s", acc), fmt("v%d.4s", s1), fmt("v%d.4s", s2)}, ""});
        out.push_back({LS_I_STORE, "st1", {fmt("{v%d.4s}", acc), "[" + b + "]"}, ""});
      } else {
        out.push_back({LS_I_FMA, "fma.rn.f32",
                       {fmt("%%f%d", acc), fmt("%%f%d", s1), fmt("%%f%d", s2), fmt("%%f%d", acc)}, ""});
        out.push_back({LS_I_STORE, "st.global.f32", {"[" + b + "]", fmt("%%f%d", acc)}, ""});
      }
    }
  }
};

// Fixed blocks: preamble/header (one counter init), latch, ret.
void fixed_block_cycles(const ls_task_desc& d, int64_t* c_init, int64_t* c_latch, int64_t* c_ret) {
  Emitter e{d.target};
  e.init(1);
  *c_init = schedule_block(e.out, d);
  e.out.clear();
  e.latch(0, 7, 0);
  *c_latch = schedule_block(e.out, d);
  e.out.clear();
  e.ret();
  *c_ret = schedule_block(e.out, d);
}

// Innermost block with the body replicated U times and its latch (k >= 1), or
// the single top-level block of body x U followed by `ret` (all loops inlined).
int64_t body_block_cycles(const ls_task_desc& d, const std::vector<int>& load_t,
                          const std::vector<int>& store_t, int64_t U, bool with_latch) {
  Emitter e{d.target};
  for (int64_t c = 0; c < U; ++c) e.body(load_t, store_t);
  if (with_latch)
    e.latch(1, 7, 1);
  else
    e.ret();
  return schedule_block(e.out, d);
}

// A tree loop's header block: its direct accesses (loads, then fma + store per
// store) followed by the first child loop's counter init, or by its own latch
// when it has no child loop (ls/ir.py:628-654 with the block splits of
// ls/asm.py:155-167).  The counter register does not interact with the body.
int64_t group_block_cycles(const ls_task_desc& d, const std::vector<int>& load_t, const std::vector<int>& store_t,
                           bool with_latch) {
  Emitter e{d.target};
  e.body(load_t, store_t);
  if (with_latch)
    e.latch(1, 7, 1);
  else
    e.init(2);
  return schedule_block(e.out, d);
}

}  // namespace lsb
