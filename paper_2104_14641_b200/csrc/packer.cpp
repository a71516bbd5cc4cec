// Host packer of explicit schedule lists (the rank path, ls/cli.py:106-141) into
// ls_record fields, as a CPython extension: one pass over the Schedule objects
// (ours or the reference's own ir.Schedule / Tile / Reorder / Unroll /
// Vectorize / Parallel, ls/ir.py:214-343 -- matched by class name and
// attributes), grouping by shape exactly like pack.shape_key and encoding like
// pack.pack_schedules:
//   shape     per transform: (kind, loop) or ("Reorder", sorted(order))
//   param[8]  Tile factors / Vectorize widths in transform order (uint16;
//             _encode_factor's rules, status 16 when unencodable)
//   perm      nibble j of reorder r = rank of order[j] in sorted(order),
//             shifted past the nibbles of the earlier reorders
// A schedule the fast path cannot read (unknown transform class, non-int
// factor, missing attribute) makes pack() return None so the caller falls
// back to the Python packer, which raises the reference's exception.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace {

enum Kind { K_TILE = 0, K_REORDER = 1, K_UNROLL = 2, K_VECTORIZE = 3, K_PARALLEL = 4, K_BAD = -1 };

Kind kind_by_name(PyTypeObject* tp) {
  const char* n = tp->tp_name;
  const char* dot = strrchr(n, '.');
  if (dot) n = dot + 1;
  if (!strcmp(n, "Tile")) return K_TILE;
  if (!strcmp(n, "Reorder")) return K_REORDER;
  if (!strcmp(n, "Unroll")) return K_UNROLL;
  if (!strcmp(n, "Vectorize")) return K_VECTORIZE;
  if (!strcmp(n, "Parallel")) return K_PARALLEL;
  return K_BAD;
}

// transform class -> kind, cached by type object (a handful of classes per process)
Kind kind_of(PyObject* t) {
  static PyTypeObject* seen[8];
  static Kind kinds[8];
  static int n_seen = 0;
  PyTypeObject* tp = Py_TYPE(t);
  for (int q = 0; q < n_seen; ++q)
    if (seen[q] == tp) return kinds[q];
  const Kind k = kind_by_name(tp);
  if (n_seen < 8 && k != K_BAD) {  // transform classes are never freed while schedules use them
    Py_INCREF(tp);
    seen[n_seen] = tp;
    kinds[n_seen++] = k;
  }
  return k;
}

struct Attr {  // interned attribute names
  PyObject *transforms, *loop, *factor, *order, *width;
  bool init() {
    transforms = PyUnicode_InternFromString("transforms");
    loop = PyUnicode_InternFromString("loop");
    factor = PyUnicode_InternFromString("factor");
    order = PyUnicode_InternFromString("order");
    width = PyUnicode_InternFromString("width");
    return transforms && loop && factor && order && width;
  }
} A;

// UTF-8 of a str, a view of the object's cached UTF-8 (valid while the object lives; code-point
// order == byte order of UTF-8, as Python's sorted())
bool utf8(PyObject* s, std::string_view& out) {
  if (!PyUnicode_Check(s)) return false;
  Py_ssize_t n = 0;
  const char* p = PyUnicode_AsUTF8AndSize(s, &n);
  if (!p) {
    PyErr_Clear();
    return false;
  }
  out = std::string_view(p, (size_t)n);
  return true;
}

bool get_int(PyObject* o, long long& v) {
  if (!PyLong_Check(o)) return false;
  int ovf = 0;
  v = PyLong_AsLongLongAndOverflow(o, &ovf);
  if (ovf || (v == -1 && PyErr_Occurred())) {
    PyErr_Clear();
    v = ovf > 0 ? LLONG_MAX : LLONG_MIN;
  }
  return true;
}

bool writable(PyObject* o, Py_buffer& b, Py_ssize_t need) {
  if (PyObject_GetBuffer(o, &b, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) < 0) return false;
  if (b.len < need) {
    PyBuffer_Release(&b);
    PyErr_SetString(PyExc_ValueError, "output buffer too small");
    return false;
  }
  return true;
}

// pack(schedules, max_extent, shape_out i32[n], param_out u16[n*8], perm_out u64[n], status_out i32[n])
//   -> list of shape keys (first-appearance order) or None (fall back)
PyObject* pack(PyObject*, PyObject* args) {
  PyObject *seq, *o_shape, *o_param, *o_perm, *o_status;
  long long max_extent;
  if (!PyArg_ParseTuple(args, "OLOOOO", &seq, &max_extent, &o_shape, &o_param, &o_perm, &o_status)) return nullptr;
  PyObject* fast = PySequence_Fast(seq, "schedules must be a sequence");
  if (!fast) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  Py_buffer bs, bp, bq, bt;
  if (!writable(o_shape, bs, n * 4)) return Py_DECREF(fast), nullptr;
  if (!writable(o_param, bp, n * 16)) return PyBuffer_Release(&bs), Py_DECREF(fast), nullptr;
  if (!writable(o_perm, bq, n * 8)) return PyBuffer_Release(&bs), PyBuffer_Release(&bp), Py_DECREF(fast), nullptr;
  if (!writable(o_status, bt, n * 4))
    return PyBuffer_Release(&bs), PyBuffer_Release(&bp), PyBuffer_Release(&bq), Py_DECREF(fast), nullptr;
  int32_t* shape_out = static_cast<int32_t*>(bs.buf);
  uint16_t* param_out = static_cast<uint16_t*>(bp.buf);
  uint64_t* perm_out = static_cast<uint64_t*>(bq.buf);
  int32_t* status_out = static_cast<int32_t*>(bt.buf);

  std::unordered_map<std::string, int32_t> shapes;
  std::vector<PyObject*> keys;  // owned shape-key tuples
  std::string sig, last_sig;
  int32_t last_id = -1;
  std::string_view name;
  std::vector<std::string_view> names;
  std::vector<int> ordr;
  bool ok = true;
  // the canonical shape signature: kind byte + loop name(s), NUL-separated
  for (Py_ssize_t i = 0; i < n && ok; ++i) {
    PyObject* s = PySequence_Fast_GET_ITEM(fast, i);
    PyObject* tr = PyObject_GetAttr(s, A.transforms);
    if (!tr) {
      PyErr_Clear();
      ok = false;
      break;
    }
    PyObject* tf = PySequence_Fast(tr, "");
    Py_DECREF(tr);
    if (!tf) {
      PyErr_Clear();
      ok = false;
      break;
    }
    const Py_ssize_t m = PySequence_Fast_GET_SIZE(tf);
    sig.clear();
    uint16_t prm[8] = {0};
    int slot = 0, shift = 0;
    uint64_t perm = 0;
    int32_t status = 0;
    for (Py_ssize_t j = 0; j < m && ok; ++j) {
      PyObject* t = PySequence_Fast_GET_ITEM(tf, j);
      const Kind k = kind_of(t);
      if (k == K_BAD) {
        ok = false;
        break;
      }
      sig.push_back((char)('0' + k));
      if (k == K_REORDER) {
        PyObject* od = PyObject_GetAttr(t, A.order);
        PyObject* of = od ? PySequence_Fast(od, "") : nullptr;
        Py_XDECREF(od);
        if (!of) {
          PyErr_Clear();
          ok = false;
          break;
        }
        const Py_ssize_t q = PySequence_Fast_GET_SIZE(of);
        names.resize((size_t)q);
        for (Py_ssize_t a = 0; a < q && ok; ++a) ok = utf8(PySequence_Fast_GET_ITEM(of, a), names[a]);
        if (!ok) {
          Py_DECREF(of);
          break;
        }
        ordr.resize((size_t)q);
        for (Py_ssize_t a = 0; a < q; ++a) ordr[a] = (int)a;
        std::stable_sort(ordr.begin(), ordr.end(), [&](int x, int y) { return names[x] < names[y]; });
        for (int a : ordr) {  // sorted names into the signature
          sig += names[a];
          sig.push_back('\0');
        }
        sig.push_back('\1');
        // nibble of position a = index of names[a] in sorted(order) (first match, as list.index)
        for (Py_ssize_t a = 0; a < q; ++a) {
          int r = 0;
          for (Py_ssize_t b = 0; b < q; ++b)
            if (names[ordr[b]] == names[a]) {
              r = (int)b;
              break;
            }
          if (shift + a < 16) perm |= (uint64_t)r << (4 * (shift + a));
        }
        Py_DECREF(of);  // the name views stay valid until here
        shift += (int)q;
        continue;
      }
      PyObject* lp = PyObject_GetAttr(t, A.loop);
      if (!lp || !utf8(lp, name)) {
        Py_XDECREF(lp);
        PyErr_Clear();
        ok = false;
        break;
      }
      sig += name;
      sig.push_back('\0');
      Py_DECREF(lp);
      if (k == K_TILE || k == K_VECTORIZE) {
        PyObject* fv = PyObject_GetAttr(t, k == K_TILE ? A.factor : A.width);
        long long v = 0;
        if (!fv || !get_int(fv, v)) {
          Py_XDECREF(fv);
          PyErr_Clear();
          ok = false;
          break;
        }
        Py_DECREF(fv);
        // pack._encode_factor
        long long e;
        if (v <= 0) {
          e = v == 0 ? 0 : -1;
        } else if (v <= 0xFFFF) {
          e = v;
        } else {
          e = max_extent < 0xFFFF ? 0xFFFF : -1;
        }
        if (e < 0) {
          status = 16;  // LS_ST_UNSUPPORTED
          e = 0;
        }
        if (slot < 8) prm[slot] = (uint16_t)e;
        ++slot;
      }
    }
    Py_DECREF(tf);
    if (!ok) break;
    int32_t id;
    if (i > 0 && sig == last_sig) {  // consecutive schedules of one shape: no hashing
      id = last_id;
      shape_out[i] = id;
      memcpy(param_out + 8 * i, prm, sizeof(prm));
      perm_out[i] = perm;
      status_out[i] = status;
      continue;
    }
    auto it = shapes.find(sig);
    if (it == shapes.end()) {
      id = (int32_t)keys.size();
      shapes.emplace(sig, id);
      keys.push_back(nullptr);  // built below from the first schedule of the shape
      PyObject* key = nullptr;
      // build the Python shape key like pack.shape_key
      PyObject* tr2 = PyObject_GetAttr(s, A.transforms);
      PyObject* tf2 = tr2 ? PySequence_Fast(tr2, "") : nullptr;
      Py_XDECREF(tr2);
      if (tf2) {
        const Py_ssize_t m2 = PySequence_Fast_GET_SIZE(tf2);
        key = PyTuple_New(m2);
        for (Py_ssize_t j = 0; key && j < m2; ++j) {
          PyObject* t = PySequence_Fast_GET_ITEM(tf2, j);
          const Kind k = kind_of(t);
          static const char* kn[] = {"Tile", "Reorder", "Unroll", "Vectorize", "Parallel"};
          PyObject* arg;
          if (k == K_REORDER) {
            PyObject* od = PyObject_GetAttr(t, A.order);
            PyObject* lst = od ? PySequence_List(od) : nullptr;
            Py_XDECREF(od);
            if (lst && PyList_Sort(lst) == 0) {
              arg = PyList_AsTuple(lst);
            } else {
              arg = nullptr;
            }
            Py_XDECREF(lst);
          } else {
            arg = PyObject_GetAttr(t, A.loop);
          }
          PyObject* pair = arg ? Py_BuildValue("(sN)", kn[k], arg) : nullptr;
          if (!pair) {
            Py_CLEAR(key);
            break;
          }
          PyTuple_SET_ITEM(key, j, pair);
        }
        Py_DECREF(tf2);
      }
      if (!key) {
        PyErr_Clear();
        ok = false;
        break;
      }
      keys[id] = key;
    } else {
      id = it->second;
    }
    last_sig = sig;
    last_id = id;
    shape_out[i] = id;
    memcpy(param_out + 8 * i, prm, sizeof(prm));
    perm_out[i] = perm;
    status_out[i] = status;
  }
  PyBuffer_Release(&bs);
  PyBuffer_Release(&bp);
  PyBuffer_Release(&bq);
  PyBuffer_Release(&bt);
  Py_DECREF(fast);
  if (!ok) {
    for (PyObject* k : keys) Py_XDECREF(k);
    Py_RETURN_NONE;
  }
  PyObject* out = PyList_New((Py_ssize_t)keys.size());
  if (!out) {
    for (PyObject* k : keys) Py_XDECREF(k);
    return nullptr;
  }
  for (size_t q = 0; q < keys.size(); ++q) PyList_SET_ITEM(out, (Py_ssize_t)q, keys[q]);
  return out;
}

// call(fn, task, points, point_bytes, n, base_index, k, scores, index, n_valid, stream): the
// host-buffer points call (ls_score_topk_points_host) through its address -- the thinnest
// binding (one vectorcall, no ctypes argument conversion), used by Task.score_topk_points_host.
using HostPointsFn = int (*)(void*, const void*, int32_t, int64_t, int64_t, int32_t, double*, int64_t*, int64_t*,
                             void*);
PyObject* call_points_host(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 11) {
    PyErr_SetString(PyExc_TypeError, "call_points_host takes 11 arguments");
    return nullptr;
  }
  unsigned long long v[11];
  for (int i = 0; i < 11; ++i) {
    v[i] = PyLong_AsUnsignedLongLongMask(args[i]);
    if (PyErr_Occurred()) return nullptr;
  }
  const auto fn = reinterpret_cast<HostPointsFn>(v[0]);
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = fn(reinterpret_cast<void*>(v[1]), reinterpret_cast<const void*>(v[2]), (int32_t)v[3], (int64_t)v[4],
          (int64_t)v[5], (int32_t)v[6], reinterpret_cast<double*>(v[7]), reinterpret_cast<int64_t*>(v[8]),
          reinterpret_cast<int64_t*>(v[9]), reinterpret_cast<void*>(v[10]));
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

PyMethodDef methods[] = {
    {"pack", pack, METH_VARARGS, "pack(schedules, max_extent, shape_out, param_out, perm_out, status_out)"},
    {"call_points_host", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)()>(call_points_host)), METH_FASTCALL,
     "call_points_host(fn, task, points, point_bytes, n, base_index, k, scores, index, n_valid, stream) -> rc"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_packer", "Fast packer of schedule lists into ls_record fields",
                      -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__packer(void) {
  if (!A.init()) return nullptr;
  return PyModule_Create(&module);
}
