// External code-text analysis on the device: the features `extract_features`
// takes from a user's assembly / PTX text (`analyze --code`, ls/cli.py:86; ls/cost.py:132-152),
// one CUDA block per text, a batch of texts per launch.  Per text:
//   * line split (block-wide scan over the bytes) and per-line tokenisation in parallel: comment
//     stripping, label, predicate, mnemonic, top-level operand split (parse_asm, ls/asm.py:110-151);
//   * basic blocks, label map and branch edges (ls/asm.py:153-200), then either
//   * CPU: backward-branch targets, compare immediates, the greedy IR loop pairing
//     (loop_map, ls/asm.py:250-296), significant-instruction counts (count_simd, ls/asm.py:306-337)
//     and the list-scheduled cycles of every block weighted by its execution count (reg_effects /
//     build_deps / schedule_block / ilp_feature, ls/ilp.py:82-271) -- one thread per basic block;
//   * GPU: loop trips from the setp / induction-register idiom (loop_map_ptx / _loop_trip,
//     ls/ptx.py:90-189), trip-weighted fma/ld/st counts and per-thread cycles in line order
//     (count_ptx / thread_cycles, ls/ptx.py:201-227).
// The IR-side features (cache movement; occupancy, warp slack, shared-memory ops) come from the
// scoring kernels on the program itself; code.py assembles the FeatureVector and the score.
// Everything follows the reference's string semantics for ASCII text (Python `str.split`,
// `strip`, the module's regular expressions) -- the tests pin it against the reference's own
// extract_features on emitted and mutated texts.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/loopscout_b200.h"

namespace {

constexpr int CT_TPB = 256;
constexpr int CT_MAXOPS = 8;    // operands per instruction (LS_CODE_E_LIMIT beyond)
constexpr int CT_MAXRES = 24;   // register / memory resources per instruction
constexpr int CT_MAXPRED = 96;  // dependence predecessors per instruction

struct LineRec {
  int32_t lineno;
  int32_t lab_off, lab_len;        // label (lab_len 0: none)
  int32_t has_instr;
  int32_t mn_off, mn_len;          // mnemonic
  int32_t pred_off, pred_len;      // predicate without '@' (pred_len < 0: none)
  int32_t nops;
  int32_t op_off[CT_MAXOPS], op_len[CT_MAXOPS];
};

struct Blk {
  int32_t label;  // line record holding the label, -1 none
  int32_t i0, ni; // instructions instr[i0 .. i0 + ni)
  int32_t first_line, last_line;
};

struct Edge {
  int32_t src, dst, kind;  // 0 fallthrough, 1 jump, 2 cond-jump
};

// per-text scratch, carved from one allocation sized by the text length
struct Scratch {
  LineRec* rec;       // [cap]
  int32_t* line_start;  // [cap + 1]
  int32_t* raw;       // [2 cap]: entry = rec << 1 | is_instr
  int32_t* instr;     // [cap]: line records of instructions, raw order
  Blk* blk;           // [2 cap]
  Edge* edge;         // [4 cap]
  int32_t* weight_i;  // [cap] per instruction (scratch for weights / class ids)
  int64_t* weight;    // [cap]
  uint64_t* res;      // [cap * CT_MAXRES] resource hashes (reads then writes)
  int32_t* nres;      // [cap * 2]: reads, writes
  int32_t* pred;      // [cap * 2 * CT_MAXPRED]: RAW then order predecessors
  int32_t* npred;     // [cap * 2]
  int32_t* issue;     // [cap]
  int32_t* cls;       // [cap] unit class of each instruction (-1: none)
};

__host__ __device__ inline size_t scratch_bytes(int64_t cap) {
  return (size_t)cap * sizeof(LineRec) + (size_t)(cap + 1) * 4 + (size_t)(2 * cap) * 4 + (size_t)cap * 4 +
         (size_t)(2 * cap) * sizeof(Blk) + (size_t)(4 * cap) * sizeof(Edge) + (size_t)cap * 4 + (size_t)cap * 8 +
         (size_t)cap * CT_MAXRES * 8 + (size_t)cap * 2 * 4 + (size_t)cap * 2 * CT_MAXPRED * 4 + (size_t)cap * 2 * 4 +
         (size_t)cap * 4 + (size_t)cap * 4 + 512;
}

__device__ inline Scratch carve(unsigned char* p, int64_t cap) {
  Scratch s;
  auto take = [&](size_t bytes) {
    unsigned char* q = p;
    p += (bytes + 15) & ~size_t(15);
    return q;
  };
  s.rec = reinterpret_cast<LineRec*>(take(cap * sizeof(LineRec)));
  s.line_start = reinterpret_cast<int32_t*>(take((cap + 1) * 4));
  s.raw = reinterpret_cast<int32_t*>(take(2 * cap * 4));
  s.instr = reinterpret_cast<int32_t*>(take(cap * 4));
  s.blk = reinterpret_cast<Blk*>(take(2 * cap * sizeof(Blk)));
  s.edge = reinterpret_cast<Edge*>(take(4 * cap * sizeof(Edge)));
  s.weight_i = reinterpret_cast<int32_t*>(take(cap * 4));
  s.weight = reinterpret_cast<int64_t*>(take(cap * 8));
  s.res = reinterpret_cast<uint64_t*>(take(cap * CT_MAXRES * 8));
  s.nres = reinterpret_cast<int32_t*>(take(cap * 2 * 4));
  s.pred = reinterpret_cast<int32_t*>(take(cap * 2 * CT_MAXPRED * 4));
  s.npred = reinterpret_cast<int32_t*>(take(cap * 2 * 4));
  s.issue = reinterpret_cast<int32_t*>(take(cap * 4));
  s.cls = reinterpret_cast<int32_t*>(take(cap * 4));
  return s;
}

// ---- character classes (ASCII; Python str methods / re classes) ----
__device__ inline bool is_ws(unsigned char c) {  // str.split() / strip() whitespace
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f);
}
__device__ inline bool is_linebreak(unsigned char c) {  // str.splitlines() separators
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e;
}
__device__ inline bool is_alpha_(unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }
__device__ inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }
__device__ inline bool is_word(unsigned char c) { return is_alpha_(c) || is_digit(c); }
__device__ inline unsigned char lower(unsigned char c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

struct Str {
  const unsigned char* p;
  int n;
  __device__ unsigned char operator[](int i) const { return p[i]; }
};
__device__ inline Str sub(Str s, int a, int b) { return Str{s.p + a, b - a}; }
__device__ inline Str strip(Str s) {
  int a = 0, b = s.n;
  while (a < b && is_ws(s[a])) ++a;
  while (b > a && is_ws(s[b - 1])) --b;
  return sub(s, a, b);
}
// lowercase prefix test (mnemonic.lower().startswith(x))
__device__ inline bool lstarts(Str s, const char* x) {
  int i = 0;
  for (; x[i]; ++i)
    if (i >= s.n || lower(s[i]) != (unsigned char)x[i]) return false;
  return true;
}
__device__ inline bool leq(Str s, const char* x) {  // lowercase equality
  int i = 0;
  for (; x[i]; ++i)
    if (i >= s.n || lower(s[i]) != (unsigned char)x[i]) return false;
  return i == s.n;
}
__device__ inline bool seq(Str a, Str b) {
  if (a.n != b.n) return false;
  for (int i = 0; i < a.n; ++i)
    if (a[i] != b[i]) return false;
  return true;
}
// root = mnemonic.lower().split(".", 1)[0]
__device__ inline Str root_of(Str mn) {
  int i = 0;
  while (i < mn.n && mn[i] != '.') ++i;
  return sub(mn, 0, i);
}
__device__ inline bool is_branch_root(Str root) {  // _is_branch on an already lowercased root
  if (leq(root, "jmp") || leq(root, "b") || leq(root, "br") || leq(root, "bra") || leq(root, "ret")) return true;
  if (root.n >= 1 && lower(root[0]) == 'j') return true;  // startswith("j") and != "jmp"
  return lstarts(root, "b.") || lstarts(root, "cb") || lstarts(root, "tb");
}
__device__ inline uint64_t fnv(Str s, uint64_t h = 1469598103934665603ull) {
  for (int i = 0; i < s.n; ++i) h = (h ^ s[i]) * 1099511628211ull;
  return h;
}
__device__ inline uint64_t fnv_lower(Str s, uint64_t h = 1469598103934665603ull) {
  for (int i = 0; i < s.n; ++i) h = (h ^ lower(s[i])) * 1099511628211ull;
  return h;
}
// re.fullmatch(r"-?\d+", s) -> value (false if no match or beyond int64)
__device__ inline bool parse_int(Str s, int64_t& v) {
  int i = 0;
  bool neg = false;
  if (i < s.n && s[i] == '-') neg = true, ++i;
  if (i >= s.n) return false;
  unsigned long long acc = 0;
  for (; i < s.n; ++i) {
    if (!is_digit(s[i])) return false;
    if (acc > 922337203685477580ull) return false;
    acc = acc * 10 + (s[i] - '0');
  }
  if (acc > 9223372036854775807ull) return false;
  v = neg ? -(int64_t)acc : (int64_t)acc;
  return true;
}

// ---- per-line tokenisation (parse_asm's loop body, ls/asm.py:122-149) ----
__device__ int parse_line(Str text, int a, int b, int lineno, LineRec& r) {
  r.lineno = lineno;
  r.lab_len = 0;
  r.has_instr = 0;
  r.pred_len = -1;
  r.nops = 0;
  Str line = sub(text, a, b);
  // re.split(r"#(?![0-9-])", line, 1)[0]
  for (int i = 0; i < line.n; ++i)
    if (line[i] == '#' && !(i + 1 < line.n && (is_digit(line[i + 1]) || line[i + 1] == '-'))) {
      line.n = i;
      break;
    }
  for (int i = 0; i + 1 < line.n; ++i)  // line.split("//", 1)[0]
    if (line[i] == '/' && line[i + 1] == '/') {
      line.n = i;
      break;
    }
  line = strip(line);
  while (line.n && line[line.n - 1] == ';') --line.n;  // rstrip(";")
  line = strip(line);
  if (!line.n) return 0;
  // label: ^([.$A-Za-z_][\w.$]*):\s*(.*)$
  if (line[0] == '.' || line[0] == '$' || is_alpha_(line[0])) {
    int i = 1;
    while (i < line.n && (is_word(line[i]) || line[i] == '.' || line[i] == '$')) ++i;
    if (i < line.n && line[i] == ':') {
      r.lab_off = (int)(line.p - text.p);
      r.lab_len = i;
      line = strip(sub(line, i + 1, line.n));
      if (!line.n) return 1;
    }
  }
  if (line[0] == '@') {  // predicate, line = line.split(None, 1)
    int i = 0;
    while (i < line.n && !is_ws(line[i])) ++i;
    int j = i;
    while (j < line.n && is_ws(line[j])) ++j;
    if (j >= line.n) return -LS_CODE_E_VALUE;  // a lone predicate: not enough values to unpack
    r.pred_off = (int)(line.p - text.p) + 1;
    r.pred_len = i - 1;
    line = sub(line, j, line.n);
  }
  int i = 0;  // parts = line.split(None, 1)
  while (i < line.n && !is_ws(line[i])) ++i;
  r.mn_off = (int)(line.p - text.p);
  r.mn_len = i;
  r.has_instr = 1;
  while (i < line.n && is_ws(line[i])) ++i;
  if (i < line.n) {  // _split_operands (ls/asm.py:62-77)
    Str rest = sub(line, i, line.n);
    int depth = 0, start = 0;
    for (int q = 0; q <= rest.n; ++q) {
      const bool end = q == rest.n;
      const unsigned char ch = end ? 0 : rest[q];
      if (!end) {
        if (ch == '(' || ch == '[' || ch == '{') ++depth;
        else if (ch == ')' || ch == ']' || ch == '}') --depth;
      }
      if (end || (ch == ',' && depth == 0)) {
        Str op = strip(sub(rest, start, q));
        if (!end || op.n) {
          if (r.nops >= CT_MAXOPS) return -LS_CODE_E_LIMIT;
          r.op_off[r.nops] = (int)(op.p - text.p);
          r.op_len[r.nops] = op.n;
          ++r.nops;
        }
        start = q + 1;
      }
    }
  }
  return 1;
}

__device__ inline Str mn_of(Str text, const LineRec& r) { return Str{text.p + r.mn_off, r.mn_len}; }
__device__ inline Str op_of(Str text, const LineRec& r, int i) { return Str{text.p + r.op_off[i], r.op_len[i]}; }
__device__ inline Str lab_of(Str text, const LineRec& r) { return Str{text.p + r.lab_off, r.lab_len}; }

// _immediate of loop_bound_immediate: strip, one leading '$' / '#', -?\d+
__device__ inline bool cmp_immediate(Str op, int64_t& v) {
  op = strip(op);
  if (op.n && (op[0] == '$' || op[0] == '#')) op = sub(op, 1, op.n);
  return parse_int(op, v);
}

// ---- reg_effects (ls/ilp.py:82-121) ----
__device__ inline int mem_operand(Str text, const LineRec& r) {
  for (int i = 0; i < r.nops; ++i) {
    Str op = op_of(text, r, i);
    for (int q = 0; q < op.n; ++q)
      if (op[q] == '(' || op[q] == '[') return i;
  }
  return -1;
}

// re.findall(r"[%$#]?[A-Za-z_][\w.]*", op), minus $/# tokens, split(".")[0].lstrip("%")
template <typename F>
__device__ inline void regs_in(Str op, F&& emit) {
  int i = 0;
  while (i < op.n) {
    int j = i;
    const bool pre = op[j] == '%' || op[j] == '$' || op[j] == '#';
    if (pre) ++j;
    if (j < op.n && is_alpha_(op[j])) {
      int k = j + 1;
      while (k < op.n && (is_word(op[k]) || op[k] == '.')) ++k;
      if (!(pre && (op[i] == '$' || op[i] == '#'))) {
        int a = i, b = k;
        for (int q = a; q < b; ++q)
          if (op[q] == '.') {
            b = q;
            break;
          }
        while (a < b && op[a] == '%') ++a;
        emit(Str{op.p + a, b - a});
      }
      i = k;
    } else {
      ++i;
    }
  }
}

constexpr uint64_t MEM_SALT = 0x9E3779B97F4A7C15ull;

// latency class (ls/ilp.py:38-47): 0 fma, 1 load, 2 move, 3 store, else the root's hash
__device__ uint64_t latency_class(Str text, const LineRec& r) {
  Str mn = mn_of(text, r), root = root_of(mn);
  if (lstarts(mn, "vfmadd") || lstarts(mn, "vfnmadd") || lstarts(mn, "vfmsub") || leq(root, "fma") ||
      leq(root, "fmla") || leq(root, "fmls"))
    return fnv(Str{reinterpret_cast<const unsigned char*>("fma"), 3});
  if (lstarts(mn, "vmov") || lstarts(mn, "ld") || lstarts(mn, "vld"))
    return mem_operand(text, r) >= 0 ? fnv(Str{reinterpret_cast<const unsigned char*>("load"), 4})
                                     : fnv(Str{reinterpret_cast<const unsigned char*>("move"), 4});
  if (lstarts(mn, "st") || lstarts(mn, "vst")) return fnv(Str{reinterpret_cast<const unsigned char*>("store"), 5});
  return fnv_lower(root);
}

}  // namespace

// ---------------------------------------------------------------------------
// the kernel: one block per text
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CT_TPB) code_kernel(const unsigned char* __restrict__ texts,
                                                      const int64_t* __restrict__ offs, int32_t n_texts,
                                                      const ls_code_desc* __restrict__ gd,
                                                      unsigned char* __restrict__ scratch,
                                                      const int64_t* __restrict__ scratch_off,
                                                      double* __restrict__ feats, int32_t* __restrict__ status,
                                                      int64_t* __restrict__ err_info, int64_t* __restrict__ diag,
                                                      const int64_t* __restrict__ diag_off,
                                                      int32_t* __restrict__ ndiag) {
  const int t = blockIdx.x;
  if (t >= n_texts) return;
  const ls_code_desc& D = *gd;
  const int64_t a0 = offs[t], a1 = offs[t + 1];
  const Str text{texts + a0, (int)(a1 - a0)};
  const int64_t cap = text.n + 2;
  Scratch S = carve(scratch + scratch_off[t], cap);
  // diagnostics (thread 0 only): events in the reference's order, rendered by the host
  int32_t n_note = 0;
  int64_t* my_diag = diag ? diag + diag_off[t] * LS_CODE_DIAG_WORDS : nullptr;
  auto note = [&](int kind, int blk, int64_t a, int64_t b, int64_t c, int64_t aux_off, int64_t aux_len) {
    if (my_diag && n_note < cap) {  // cap = ls_code_diag_cap(text bytes) >= blocks, back edges + 1
      int64_t* e = my_diag + (size_t)n_note * LS_CODE_DIAG_WORDS;
      int64_t lo = -1, ll = 0;
      if (blk >= 0 && S.blk[blk].label >= 0) {
        const LineRec& r = S.rec[S.blk[blk].label];
        lo = r.lab_off;
        ll = r.lab_len;
      }
      e[0] = kind, e[1] = blk, e[2] = lo, e[3] = ll, e[4] = a, e[5] = b, e[6] = c, e[7] = aux_off, e[8] = aux_len;
      e[9] = 0;
    }
    ++n_note;
  };
  __shared__ int s_cnt[CT_TPB + 1];
  __shared__ int s_err, s_nlines, s_ninstr, s_nblk, s_nedge;
  if (threadIdx.x == 0) s_err = 0;
  // ---- 1. line starts (str.splitlines: \r\n is one break), block-wide scan over byte chunks
  const int chunk = (text.n + CT_TPB - 1) / CT_TPB;
  const int c0 = min(text.n, (int)threadIdx.x * chunk), c1 = min(text.n, c0 + chunk);
  auto brk = [&](int i) {  // a line break ends at byte i (\r followed by \n breaks at the \n)
    const unsigned char c = text[i];
    if (!is_linebreak(c)) return false;
    return !(c == '\r' && i + 1 < text.n && text[i + 1] == '\n');
  };
  int mine = 0;
  for (int i = c0; i < c1; ++i) mine += brk(i);
  s_cnt[threadIdx.x] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int q = 0; q < CT_TPB; ++q) {
      const int v = s_cnt[q];
      s_cnt[q] = run;
      run += v;
    }
    s_cnt[CT_TPB] = run;
  }
  __syncthreads();
  {
    int w = s_cnt[threadIdx.x];
    for (int i = c0; i < c1; ++i)
      if (brk(i)) S.line_start[++w] = i + 1;  // line w + 1 starts after break w
  }
  if (threadIdx.x == 0) {
    S.line_start[0] = 0;
    const int nb = s_cnt[CT_TPB];
    // splitlines drops a final empty line after a trailing break
    s_nlines = (nb && S.line_start[nb] == text.n) ? nb : nb + 1;
    S.line_start[s_nlines] = text.n + 1;  // sentinel: end of the last line is text.n
  }
  __syncthreads();
  const int nlines = text.n ? s_nlines : 0;
  // ---- 2. tokenise every line
  for (int l = threadIdx.x; l < nlines; l += CT_TPB) {
    int a = S.line_start[l], b = l + 1 < nlines ? S.line_start[l + 1] : text.n;
    while (b > a && is_linebreak(text[b - 1])) --b;  // drop the break itself
    const int rc = parse_line(text, a, b, l + 1, S.rec[l]);
    if (rc < 0) atomicMin(&s_err, rc), S.rec[l].has_instr = 0, S.rec[l].lab_len = 0;
    if (rc == 0) S.rec[l].has_instr = 0, S.rec[l].lab_len = 0;
  }
  __syncthreads();
  {
    const int e = s_err;
    __syncthreads();  // every thread has read it before thread 0 reuses it below
    if (e) {
      if (threadIdx.x == 0) status[t] = -e;
      return;
    }
  }
  // ---- 3. raw entries, blocks, edges (thread 0; ls/asm.py:150-200)
  if (threadIdx.x == 0) {
    int nraw = 0, ninstr = 0;
    for (int l = 0; l < nlines; ++l) {
      const LineRec& r = S.rec[l];
      if (r.lab_len) S.raw[nraw++] = l << 1;
      if (r.has_instr) {
        S.raw[nraw++] = (l << 1) | 1;
        S.instr[ninstr++] = l;
      }
    }
    int err = 0;
    if (!ninstr) err = LS_CODE_E_EMPTY;
    int nblk = 0, nedge = 0;
    if (!err) {
      int cur_label = -1, cur_first = -1, cur_i0 = 0, cur_n = 0;
      auto flush = [&](int last_line) {
        if (cur_n || cur_label >= 0)
          S.blk[nblk++] = Blk{cur_label, cur_i0, cur_n, cur_first >= 0 ? cur_first : last_line, last_line};
        cur_label = -1;
        cur_first = -1;
        cur_n = 0;
      };
      int ii = 0;  // instruction cursor (raw order == S.instr order)
      for (int q = 0; q < nraw; ++q) {
        const int l = S.raw[q] >> 1;
        const int lineno = S.rec[l].lineno;
        if (!(S.raw[q] & 1)) {
          flush(lineno - 1);
          cur_label = l;
          cur_first = lineno;
          continue;
        }
        if (cur_first < 0) cur_first = lineno;
        if (!cur_n) cur_i0 = ii;
        ++cur_n;
        ++ii;
        Str mn = mn_of(text, S.rec[l]);
        if (is_branch_root(root_of(mn)) || lstarts(mn, "b.")) flush(lineno);
      }
      flush(S.rec[S.raw[nraw - 1] >> 1].lineno);
      // blocks keep their order (every flushed block has instructions or a label)
      for (int b = 0; b < nblk && !err; ++b) {
        const Blk& B = S.blk[b];
        bool fall = true;
        if (B.ni) {
          const LineRec& term = S.rec[S.instr[B.i0 + B.ni - 1]];
          Str mn = mn_of(text, term), root = root_of(mn);
          if (is_branch_root(root)) {
            int target = -1;
            for (int o = 0; o < term.nops && target < 0; ++o) {
              Str op = op_of(text, term, o);
              for (int c = nblk - 1; c >= 0; --c)  // labels dict: the last block with the label wins
                if (S.blk[c].label >= 0 && seq(lab_of(text, S.rec[S.blk[c].label]), op)) {
                  target = c;
                  break;
                }
            }
            if (leq(root, "ret")) {
              fall = false;
            } else {
              if (target < 0) {
                err = LS_CODE_E_LABEL;
                err_info[3 * t] = term.lineno;
                err_info[3 * t + 1] = term.nops ? term.op_off[0] : -1;
                err_info[3 * t + 2] = term.nops ? term.op_len[0] : 0;
                break;
              }
              const bool uncond = leq(mn, "jmp") || leq(mn, "b") || leq(mn, "br") ||
                                  (leq(root, "bra") && term.pred_len < 0);
              S.edge[nedge++] = Edge{b, target, uncond ? 1 : 2};
              fall = !uncond;
            }
          }
        }
        if (fall && b + 1 < nblk) S.edge[nedge++] = Edge{b, b + 1, 0};
      }
    }
    s_err = err;
    s_ninstr = ninstr;
    s_nblk = nblk;
    s_nedge = nedge;
  }
  __syncthreads();
  {
    const int e = s_err;
    __syncthreads();  // read by every thread before the scheduling phase may set it again
    if (e) {
      if (threadIdx.x == 0) status[t] = e;
      return;
    }
  }
  const int ninstr = s_ninstr, nblk = s_nblk, nedge = s_nedge;
  double* F = feats + 4 * (size_t)t;
  if (D.family == LS_FAMILY_CPU) {
    // ---- 4a. loop_map + count_simd (thread 0): execution count per block
    if (threadIdx.x == 0) {
      for (int b = 0; b < nblk; ++b) S.weight[b] = 1;
      int matched = 0;
      double nfma = 0, nvl = 0, nvs = 0;
      for (int b = 0; b < nblk; ++b) {  // identify_loop_lbbs: targets of backward jumps, textual order
        bool is_t = false;
        for (int e = 0; e < nedge && !is_t; ++e)
          is_t = S.edge[e].kind && S.edge[e].dst == b && S.edge[e].dst <= S.edge[e].src;
        if (!is_t) continue;
        if (matched >= D.n_loops) {
          note(LS_CODE_D_UNMATCHED_BLOCK, b, 0, 0, 0, -1, 0);
          continue;
        }
        // loop_bound_immediate: the first back edge's source block with a cmp/setp immediate
        bool have = false;
        int64_t bound = 0;
        for (int e = 0; e < nedge && !have; ++e) {
          const Edge& E = S.edge[e];
          if (E.dst != b || !E.kind || E.dst > E.src) continue;
          const Blk& src = S.blk[E.src];
          for (int q = src.ni - 1; q >= 0 && !have; --q) {
            const LineRec& r = S.rec[S.instr[src.i0 + q]];
            Str mn = mn_of(text, r);
            if (!(lstarts(mn, "cmp") || lstarts(mn, "setp"))) continue;
            for (int o = 0; o < r.nops && !have; ++o) have = cmp_immediate(op_of(text, r, o), bound);
          }
        }
        const int64_t ext = D.loop_extent[matched], stp = D.loop_step[matched];
        if (have && (bound == ext || bound == ext * stp)) {
          const int64_t w = D.loop_weight[matched];
          S.weight[b] = w;
          const Blk& B = S.blk[b];
          for (int q = 0; q < B.ni; ++q) {  // count_simd over the matched block
            const LineRec& r = S.rec[S.instr[B.i0 + q]];
            Str mn = mn_of(text, r);
            if (D.target == LS_CODE_TARGET_X86) {
              if (lstarts(mn, "vfmadd") || lstarts(mn, "vfnmadd") || lstarts(mn, "vfmsub")) {
                nfma += (double)w;
              } else if (lstarts(mn, "vmov")) {
                bool paren = false;
                if (r.nops) {
                  Str o0 = op_of(text, r, 0);
                  for (int c = 0; c < o0.n; ++c) paren |= o0[c] == '(';
                }
                if (paren) nvl += (double)w;
                else nvs += (double)w;
              }
            } else {
              if (lstarts(mn, "fmla") || lstarts(mn, "fmls")) nfma += (double)w;
              else if (lstarts(mn, "ld")) nvl += (double)w;
              else if (lstarts(mn, "st")) nvs += (double)w;
            }
          }
          ++matched;
        } else {
          note(LS_CODE_D_BOUND_MISMATCH, b, have, bound, matched, -1, 0);
        }
      }
      note(LS_CODE_D_LOOPS_MATCHED, -1, matched, 0, 0, -1, 0);
      F[0] = nfma;
      F[1] = nvl;
      F[2] = nvs;
    }
    __syncthreads();
    // ---- 4b. schedule every block (one thread per block; build_deps / schedule_block)
    for (int b = threadIdx.x; b < nblk; b += CT_TPB) {
      const Blk& B = S.blk[b];
      if (!B.ni) continue;
      int err = 0;
      // resources of every instruction of the block
      for (int q = 0; q < B.ni && !err; ++q) {
        const int ix = B.i0 + q;
        const LineRec& r = S.rec[S.instr[ix]];
        uint64_t* rd = S.res + (size_t)ix * CT_MAXRES;
        int nr = 0, nw = 0;
        uint64_t wr[CT_MAXRES];
        auto add = [&](uint64_t* set, int& n, uint64_t h) {
          for (int c = 0; c < n; ++c)
            if (set[c] == h) return;
          if (n >= CT_MAXRES / 2) {
            err = LS_CODE_E_LIMIT;
            return;
          }
          set[n++] = h;
        };
        Str mn = mn_of(text, r), root = root_of(mn);
        if (r.pred_len >= 0) {  // predicate.lstrip("%").lstrip("!")
          Str pr{text.p + r.pred_off, r.pred_len};
          int a = 0;
          while (a < pr.n && pr[a] == '%') ++a;
          while (a < pr.n && pr[a] == '!') ++a;
          add(rd, nr, fnv(sub(pr, a, pr.n)));
        }
        const bool noops = !r.nops || leq(root, "ret") || leq(root, "jmp") || leq(root, "bra") || leq(root, "b") ||
                           leq(root, "br") || (root.n && lower(root[0]) == 'j');
        if (!noops) {
          const int mem = mem_operand(text, r);
          bool store = lstarts(mn, "st") || lstarts(mn, "vst");
          if (!store && mem >= 0) store = mem == r.nops - 1 && (lstarts(mn, "vmov") || lstarts(mn, "mov"));
          int dest;
          if (D.dialect == LS_CODE_DIALECT_ATT) {
            dest = r.nops - 1;
          } else {
            dest = 0;
            if ((lstarts(mn, "st") || lstarts(mn, "vst")) && mem >= 0) dest = mem;
          }
          const bool cmp_like = leq(root, "cmp") || leq(root, "cmpq") || leq(root, "test");
          const bool rmw = lstarts(mn, "vfmadd") || lstarts(mn, "fma") || lstarts(mn, "fmla") || lstarts(mn, "fmls") ||
                           lstarts(mn, "add") || lstarts(mn, "sub") || leq(root, "add") || leq(root, "addq");
          for (int o = 0; o < r.nops; ++o) {
            Str op = op_of(text, r, o);
            if (o == mem) {
              uint64_t base = 0;
              bool have = false;
              regs_in(op, [&](Str g) {
                const uint64_t h = fnv(g);
                if (!have) base = h, have = true;
                add(rd, nr, h);
              });
              if (!have) base = fnv(Str{reinterpret_cast<const unsigned char*>("abs"), 3});
              const uint64_t mh = base ^ MEM_SALT;
              if (o == dest && store) add(wr, nw, mh);
              else add(rd, nr, mh);
              continue;
            }
            if (o == dest && !cmp_like) {
              regs_in(op, [&](Str g) {
                add(wr, nw, fnv(g));
                if (rmw) add(rd, nr, fnv(g));
              });
            } else {
              regs_in(op, [&](Str g) { add(rd, nr, fnv(g)); });
            }
          }
        }
        for (int c = 0; c < nw; ++c) rd[CT_MAXRES / 2 + c] = wr[c];
        S.nres[2 * ix] = nr;
        S.nres[2 * ix + 1] = nw;
        // latency and unit class of the instruction
        const uint64_t cls = latency_class(text, r);
        int lat = D.default_latency, klass = -1;
        for (int c = 0; c < D.n_classes; ++c)
          if (D.cls_hash[c] == cls) {
            if (D.cls_latency[c] > 0) lat = D.cls_latency[c];
            klass = c;
          }
        S.weight_i[ix] = lat;  // latency
        S.cls[ix] = klass;
      }
      if (err) {
        atomicMin(&s_err, -err);
        continue;
      }
      // build_deps: RAW from the last writer, WAW, WAR from the reads since the last write
      for (int q = 0; q < B.ni && !err; ++q) {
        const int ix = B.i0 + q;
        const uint64_t* rd = S.res + (size_t)ix * CT_MAXRES;
        const uint64_t* wr = rd + CT_MAXRES / 2;
        const int nr = S.nres[2 * ix], nw = S.nres[2 * ix + 1];
        int* raw = S.pred + (size_t)ix * 2 * CT_MAXPRED;
        int* ord = raw + CT_MAXPRED;
        int nraw = 0, nord = 0;
        auto push = [&](int* lst, int& n, int p) {
          for (int c = 0; c < n; ++c)
            if (lst[c] == p) return;
          if (n >= CT_MAXPRED) {
            err = LS_CODE_E_LIMIT;
            return;
          }
          lst[n++] = p;
        };
        auto writes = [&](int j, uint64_t h) {
          const uint64_t* w = S.res + (size_t)j * CT_MAXRES + CT_MAXRES / 2;
          for (int c = 0; c < S.nres[2 * j + 1]; ++c)
            if (w[c] == h) return true;
          return false;
        };
        auto reads = [&](int j, uint64_t h) {
          const uint64_t* w = S.res + (size_t)j * CT_MAXRES;
          for (int c = 0; c < S.nres[2 * j]; ++c)
            if (w[c] == h) return true;
          return false;
        };
        for (int c = 0; c < nr; ++c)
          for (int j = ix - 1; j >= B.i0; --j)
            if (writes(j, rd[c])) {
              push(raw, nraw, j - B.i0);
              break;
            }
        for (int c = 0; c < nw; ++c)
          for (int j = ix - 1; j >= B.i0; --j) {
            if (reads(j, wr[c])) push(ord, nord, j - B.i0);  // WAR (reads since the last write)
            if (writes(j, wr[c])) {
              push(ord, nord, j - B.i0);  // WAW
              break;
            }
          }
        // false_edges -= true_edges
        int k2 = 0;
        for (int c = 0; c < nord; ++c) {
          bool dup = false;
          for (int d = 0; d < nraw; ++d) dup |= raw[d] == ord[c];
          if (!dup) ord[k2++] = ord[c];
        }
        nord = k2;
        S.npred[2 * ix] = nraw;
        S.npred[2 * ix + 1] = nord;
      }
      if (err) {
        atomicMin(&s_err, -err);
        continue;
      }
      // schedule_block: greedy cycle-by-cycle issue in program order (ls/ilp.py:158-204)
      int32_t* iss = S.issue;  // per instruction, indexed ix
      for (int q = 0; q < B.ni; ++q) iss[B.i0 + q] = -1;
      int done = 0, cycle = 0;
      while (done < B.ni) {
        if (cycle > (1 << 24)) {  // a zero unit cap never issues (the reference loops forever)
          err = LS_CODE_E_LIMIT;
          break;
        }
        int issued = 0;
        int unit_used[LS_CODE_MAX_CLASSES];
        for (int c = 0; c < D.n_classes; ++c) unit_used[c] = 0;
        for (int q = 0; q < B.ni; ++q) {
          const int ix = B.i0 + q;
          if (iss[ix] >= 0 || issued >= D.issue_width) continue;
          int ready = 0;
          bool ok = true;
          const int* raw = S.pred + (size_t)ix * 2 * CT_MAXPRED;
          const int* ord = raw + CT_MAXPRED;
          for (int c = 0; c < S.npred[2 * ix] && ok; ++c) {
            const int p = B.i0 + raw[c];
            if (iss[p] < 0) ok = false;
            else ready = max(ready, iss[p] + S.weight_i[p]);
          }
          for (int c = 0; c < S.npred[2 * ix + 1] && ok; ++c) {
            const int p = B.i0 + ord[c];
            if (iss[p] < 0) ok = false;
            else ready = max(ready, iss[p] + 1);
          }
          if (!ok || ready > cycle) continue;
          const int kc = S.cls[ix];
          if (kc >= 0 && D.cls_units[kc] > 0 && unit_used[kc] >= D.cls_units[kc]) continue;
          iss[ix] = cycle;
          if (kc >= 0) ++unit_used[kc];
          ++issued;
          ++done;
        }
        ++cycle;
      }
      if (err) {
        atomicMin(&s_err, -err);
        continue;
      }
      int fin = 0;
      for (int q = 0; q < B.ni; ++q) fin = max(fin, iss[B.i0 + q] + S.weight_i[B.i0 + q]);
      S.weight_i[B.i0] = fin;  // the block's cycles (first instruction's slot; latencies no longer needed)
    }
    __syncthreads();
    if (s_err) {
      if (threadIdx.x == 0) status[t] = -s_err;
      return;
    }
    if (threadIdx.x == 0) {  // ilp_feature: block order, cycles x execution count
      double total = 0.0;
      for (int b = 0; b < nblk; ++b)
        if (S.blk[b].ni) total = __dadd_rn(total, (double)((int64_t)S.weight_i[S.blk[b].i0] * S.weight[b]));
      F[3] = total;
      status[t] = 0;
      if (ndiag) ndiag[t] = n_note;
    }
    return;
  }
  // ---- 5. PTX: loop trips, trip-weighted counts and per-thread cycles (thread 0; ls/ptx.py)
  if (threadIdx.x == 0) {
    // back edges sorted by target block (stable)
    int nl = 0;
    int32_t* lst = S.npred;      // loop start lines
    int32_t* lend = S.npred + nedge + 1;
    int64_t* ltrip = S.weight;   // trip, or -1
    for (int b = 0; b < nblk; ++b)
      for (int e = 0; e < nedge; ++e) {
        const Edge& E = S.edge[e];
        if (!E.kind || E.dst > E.src || E.dst != b) continue;
        const Blk& tgt = S.blk[E.dst];
        const Blk& src = S.blk[E.src];
        const int start_line = tgt.first_line, end_line = src.last_line;
        int64_t trip = -1;
        // _loop_trip
        const LineRec& term = S.rec[S.instr[src.i0 + src.ni - 1]];
        int setp = -1;
        for (int q = src.ni - 1; q >= 0 && setp < 0; --q) {
          const LineRec& r = S.rec[S.instr[src.i0 + q]];
          if (!lstarts(mn_of(text, r), "setp")) continue;
          bool take = r.nops == 2 || term.pred_len < 0;
          if (!take && r.nops) {
            Str o0 = op_of(text, r, 0), pr{text.p + term.pred_off, term.pred_len};
            int a = 0, c = 0;
            while (a < o0.n && (o0[a] == '%' || o0[a] == '!')) ++a;
            while (c < pr.n && (pr[c] == '%' || pr[c] == '!')) ++c;
            take = seq(sub(o0, a, o0.n), sub(pr, c, pr.n));
          }
          if (take) setp = S.instr[src.i0 + q];
        }
        if (setp >= 0 && S.rec[setp].nops >= 2) {
          const LineRec& sp = S.rec[setp];
          Str mn = mn_of(text, sp);  // setp.mnemonic.split(".")[1] (original case)
          Str op{reinterpret_cast<const unsigned char*>("ne"), 2};
          for (int c = 0; c < mn.n; ++c)
            if (mn[c] == '.') {
              int d = c + 1;
              while (d < mn.n && mn[d] != '.') ++d;
              op = sub(mn, c + 1, d);
              break;
            }
          Str reg = strip(op_of(text, sp, sp.nops >= 3 ? 1 : 0));
          // the comparison's span in the text; -1: the implicit "ne" of a setp without a suffix
          const int64_t reg_off = reg.p - text.p, op_off = op.p >= text.p && op.p <= text.p + text.n ? op.p - text.p : -1;
          int64_t bound;
          if (!parse_int(strip(op_of(text, sp, sp.nops >= 3 ? 2 : 1)), bound)) {
            note(LS_CODE_D_NON_IMM_BOUND, E.dst, 0, 0, 0, -1, 0);
          } else {
            bool have_init = false, nonlinear = false;
            int64_t init = 0, delta = 0;
            for (int q = 0; q < ninstr; ++q) {  // every instruction, block order == raw order
              const LineRec& r = S.rec[S.instr[q]];
              if (!r.nops || !seq(strip(op_of(text, r, 0)), reg)) continue;
              Str root = root_of(mn_of(text, r));
              if (r.lineno < start_line) {
                int64_t v;
                if (leq(root, "mov") && r.nops > 1 && parse_int(strip(op_of(text, r, 1)), v)) init = v, have_init = true;
              } else if (r.lineno <= end_line) {
                if ((leq(root, "add") || leq(root, "sub")) && r.nops >= 3 && seq(strip(op_of(text, r, 1)), reg)) {
                  int64_t d;
                  if (!parse_int(strip(op_of(text, r, 2)), d)) nonlinear = true;
                  else delta += leq(root, "add") ? d : -d;
                } else if (leq(root, "mul") || leq(root, "shl") || leq(root, "mad") || leq(root, "mov")) {
                  nonlinear = true;
                }
              }
            }
            if (nonlinear) {
              note(LS_CODE_D_NONLINEAR, E.dst, 0, 0, 0, reg_off, reg.n);
            } else if (!have_init || delta == 0) {
              note(LS_CODE_D_NOT_DERIVABLE, E.dst, 0, 0, 0, reg_off, reg.n);
            } else {
              const double span = (double)(bound - init), dl = (double)delta;
              bool known = true;
              if (seq(op, Str{reinterpret_cast<const unsigned char*>("lt"), 2}) ||
                  seq(op, Str{reinterpret_cast<const unsigned char*>("gt"), 2})) {
                trip = (int64_t)ceil(span / dl);
              } else if (seq(op, Str{reinterpret_cast<const unsigned char*>("le"), 2}) ||
                         seq(op, Str{reinterpret_cast<const unsigned char*>("ge"), 2})) {
                trip = (int64_t)floor(span / dl) + 1;
              } else if (seq(op, Str{reinterpret_cast<const unsigned char*>("ne"), 2})) {
                const double q = span / dl;
                trip = q == floor(q) ? (int64_t)q : -1;
              } else {
                known = false;
                note(LS_CODE_D_UNSUPPORTED_CMP, E.dst, 0, 0, 0, op_off, op.n);
              }
              if (trip <= 0) {
                trip = -1;
                if (known) note(LS_CODE_D_INCONSISTENT, E.dst, init, delta, bound, op_off, op.n);
              }
            }
          }
        } else {
          note(LS_CODE_D_NO_SETP, E.dst, 0, 0, 0, -1, 0);
        }
        lst[nl] = start_line;
        lend[nl] = end_line;
        ltrip[nl] = trip;
        ++nl;
      }
    double nfma = 0, nld = 0, nst = 0, work = 0;
    bool ovf = false;
    for (int b = 0; b < nblk; ++b) {  // blocks, then instructions: the reference's line order
      const Blk& B = S.blk[b];
      for (int q = 0; q < B.ni; ++q) {
        const LineRec& r = S.rec[S.instr[B.i0 + q]];
        int64_t w = 1;
        for (int c = 0; c < nl; ++c)
          if (ltrip[c] > 0 && lst[c] <= r.lineno && r.lineno <= lend[c]) {
            if (w > INT64_MAX / ltrip[c]) ovf = true;
            w *= ltrip[c];
          }
        Str mn = mn_of(text, r), root = root_of(mn);
        if (leq(root, "fma") || leq(root, "mad")) nfma += (double)w;
        else if (lstarts(mn, "ld")) nld += (double)w;
        else if (lstarts(mn, "st")) nst += (double)w;
        double cost = 1.0;
        const uint64_t h = fnv_lower(root);
        for (int c = 0; c < D.n_costs; ++c)
          if (D.cost_hash[c] == h) cost = D.cost[c];
        work = __dadd_rn(work, __dmul_rn(cost, (double)w));
      }
    }
    F[0] = work;
    F[1] = nfma;
    F[2] = nld;
    F[3] = nst;
    status[t] = ovf ? LS_CODE_E_LIMIT : 0;
    if (ndiag) ndiag[t] = n_note;
  }
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
static thread_local std::string g_code_err;

extern "C" {

uint64_t ls_code_hash(const char* s, int32_t n) {  // the class / cost table keys (lowercase roots)
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < n; ++i) h = (h ^ (unsigned char)s[i]) * 1099511628211ull;
  return h;
}

int64_t ls_code_scratch_bytes(int64_t text_bytes) { return (int64_t)scratch_bytes(text_bytes + 2); }

int64_t ls_code_diag_cap(int64_t text_bytes) { return text_bytes + 2; }

int ls_code_features(const ls_code_desc* desc, const char* d_texts, const int64_t* h_offsets, int32_t n_texts,
                     void* d_scratch, int64_t scratch_bytes_total, double* d_features, int32_t* d_status,
                     int64_t* d_err_info, void* stream) {
  return ls_code_features_diag(desc, d_texts, h_offsets, n_texts, d_scratch, scratch_bytes_total, d_features, d_status,
                               d_err_info, nullptr, nullptr, stream);
}

int ls_code_features_diag(const ls_code_desc* desc, const char* d_texts, const int64_t* h_offsets, int32_t n_texts,
                          void* d_scratch, int64_t scratch_bytes_total, double* d_features, int32_t* d_status,
                          int64_t* d_err_info, int64_t* d_diag, int32_t* d_ndiag, void* stream) {
  if ((d_diag == nullptr) != (d_ndiag == nullptr)) return LS_E_ARG;
  if (!desc || n_texts < 0 || (n_texts && (!d_texts || !h_offsets || !d_features || !d_status || !d_err_info)))
    return LS_E_ARG;
  if (desc->n_classes > LS_CODE_MAX_CLASSES || desc->n_costs > LS_CODE_MAX_CLASSES || desc->n_loops > LS_CODE_MAX_LOOPS ||
      desc->issue_width < 1)
    return LS_E_ARG;
  if (!n_texts) return LS_E_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // per-text scratch offsets (host) + the descriptor and offsets on the device
  std::string buf;
  int64_t need = 0;
  std::vector<int64_t> soff((size_t)n_texts * 2);  // scratch offsets, then diagnostic event offsets
  int64_t ev = 0;
  for (int i = 0; i < n_texts; ++i) {
    const int64_t len = h_offsets[i + 1] - h_offsets[i];
    if (len < 0 || len > (1 << 26)) return LS_E_ARG;
    soff[i] = need;
    need += ((int64_t)scratch_bytes(len + 2) + 255) & ~(int64_t)255;
    soff[n_texts + i] = ev;
    ev += ls_code_diag_cap(len);
  }
  const size_t meta = sizeof(ls_code_desc) + sizeof(int64_t) * (size_t)(n_texts + 1) + sizeof(int64_t) * 2 * n_texts;
  if (!d_scratch || scratch_bytes_total < need + (int64_t)meta + 256) return LS_E_ARG;
  unsigned char* sc = reinterpret_cast<unsigned char*>(d_scratch);
  unsigned char* md = sc + need;
  md = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(md) + 255) & ~uintptr_t(255));
  ls_code_desc* dd = reinterpret_cast<ls_code_desc*>(md);
  int64_t* doffs = reinterpret_cast<int64_t*>(md + sizeof(ls_code_desc));
  int64_t* dsoff = doffs + n_texts + 1;
  std::vector<unsigned char> hm(meta);
  memcpy(hm.data(), desc, sizeof(ls_code_desc));
  memcpy(hm.data() + sizeof(ls_code_desc), h_offsets, sizeof(int64_t) * (n_texts + 1));
  memcpy(hm.data() + sizeof(ls_code_desc) + sizeof(int64_t) * (n_texts + 1), soff.data(), sizeof(int64_t) * 2 * n_texts);
  cudaError_t e = cudaMemcpyAsync(md, hm.data(), meta, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // hm is a temporary
  if (e != cudaSuccess) return g_code_err = cudaGetErrorString(e), LS_E_CUDA;
  code_kernel<<<n_texts, CT_TPB, 0, s>>>(reinterpret_cast<const unsigned char*>(d_texts), doffs, n_texts, dd, sc, dsoff,
                                         d_features, d_status, d_err_info, d_diag, dsoff + n_texts, d_ndiag);
  e = cudaGetLastError();
  if (e != cudaSuccess) return g_code_err = cudaGetErrorString(e), LS_E_CUDA;
  return LS_E_OK;
}

}  // extern "C"
