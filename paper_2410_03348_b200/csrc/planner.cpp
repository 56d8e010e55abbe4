// Native host planner: the map/shuffle stage of apply_if (distribution.py:244-260) as a
// CPython extension, so the only interpreted work per combination is the user's own
// black-box symbol function.
//
//   map_shuffle(f, cond, symbol_lists, undefined)
//       -> (out_symbols: tuple, kept: bytes[int64 ordinals], out_idx: bytes[int32], calls)
//   or ("error", syms_tuple, exception) when f / cond raised (the Python side re-raises it
//   as SymbolFunctionError(symbols), distribution.py:179-185).
//
// Semantics restated from the reference, bit for bit:
//  * enumeration = itertools.product(*symbol_lists): a mixed-radix counter, last list
//    fastest (distribution.py:246);
//  * cond is called before f, and combinations it rejects are skipped (:248-249);
//  * f's result `is UNDEFINED` drops the combination (:251);
//  * output symbols are numbered by first derivation through a real Python dict keyed by
//    the result object, so hashing/equality (1 == 1.0 == True) is exactly the
//    reference's (:258-260).
// Calls use the vectorcall protocol on a stack array of borrowed symbol references: no
// argument tuple is built unless an error has to be reported.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cstdint>
#include <vector>

namespace {

struct Ref {  // owned reference
  PyObject* p = nullptr;
  explicit Ref(PyObject* o = nullptr) : p(o) {}
  ~Ref() { Py_XDECREF(p); }
  Ref(Ref&& o) noexcept : p(o.p) { o.p = nullptr; }
  Ref(const Ref&) = delete;
  Ref& operator=(const Ref&) = delete;
  PyObject* release() {
    PyObject* o = p;
    p = nullptr;
    return o;
  }
};

PyObject* error_result(PyObject* const* args, Py_ssize_t n) {
  // ("error", syms, exc) with the pending exception taken out of the thread state
  PyObject* exc = PyErr_GetRaisedException();
  Ref syms(PyTuple_New(n));
  if (!syms.p) {
    Py_XDECREF(exc);
    return nullptr;
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    Py_INCREF(args[i]);
    PyTuple_SET_ITEM(syms.p, i, args[i]);
  }
  PyObject* r = Py_BuildValue("(sOO)", "error", syms.p, exc ? exc : Py_None);
  Py_XDECREF(exc);
  return r;
}

PyObject* map_shuffle(PyObject*, PyObject* args) {
  PyObject *f, *cond, *lists_obj, *undefined;
  if (!PyArg_ParseTuple(args, "OOOO", &f, &cond, &lists_obj, &undefined)) return nullptr;
  Ref lists(PySequence_Fast(lists_obj, "symbol_lists must be a sequence"));
  if (!lists.p) return nullptr;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(lists.p);
  std::vector<Ref> seqs;
  std::vector<PyObject**> items(n);
  std::vector<Py_ssize_t> sizes(n);
  seqs.reserve(n);
  for (Py_ssize_t i = 0; i < n; ++i) {
    seqs.emplace_back(PySequence_Fast(PySequence_Fast_GET_ITEM(lists.p, i), "each symbol list must be a sequence"));
    if (!seqs.back().p) return nullptr;
    items[i] = PySequence_Fast_ITEMS(seqs.back().p);
    sizes[i] = PySequence_Fast_GET_SIZE(seqs.back().p);
  }
  const bool use_cond = cond != Py_None;
  Ref buckets(PyDict_New());
  if (!buckets.p) return nullptr;
  std::vector<int64_t> kept;
  std::vector<int32_t> out_idx;
  long long calls = 0;
  bool empty = false;  // itertools.product() of no lists yields one empty combination
  for (Py_ssize_t i = 0; i < n; ++i) empty = empty || sizes[i] == 0;
  if (!empty) {
    std::vector<Py_ssize_t> pos(n, 0);
    std::vector<PyObject*> argv(n);
    for (Py_ssize_t i = 0; i < n; ++i) argv[i] = items[i][0];
    int64_t ordinal = 0;
    for (;;) {
      bool keep = true;
      if (use_cond) {
        ++calls;
        Ref c(PyObject_Vectorcall(cond, argv.data(), (size_t)n, nullptr));
        if (!c.p) return error_result(argv.data(), n);
        const int t = PyObject_IsTrue(c.p);
        if (t < 0) return error_result(argv.data(), n);
        keep = t != 0;
      }
      if (keep) {
        ++calls;
        Ref v(PyObject_Vectorcall(f, argv.data(), (size_t)n, nullptr));
        if (!v.p) return error_result(argv.data(), n);
        if (v.p != undefined) {
          PyObject* idx = PyDict_GetItemWithError(buckets.p, v.p);  // borrowed
          int32_t k;
          if (idx) {
            k = (int32_t)PyLong_AsLong(idx);
          } else {
            if (PyErr_Occurred()) return nullptr;  // unhashable result: raised as-is, like the reference dict
            k = (int32_t)PyDict_GET_SIZE(buckets.p);
            Ref key(PyLong_FromLong(k));
            if (!key.p || PyDict_SetItem(buckets.p, v.p, key.p) < 0) return nullptr;
          }
          kept.push_back(ordinal);
          out_idx.push_back(k);
        }
      }
      ++ordinal;
      // mixed-radix increment, last list fastest (itertools.product order)
      Py_ssize_t d = n - 1;
      for (; d >= 0; --d) {
        if (++pos[d] < sizes[d]) {
          argv[d] = items[d][pos[d]];
          break;
        }
        pos[d] = 0;
        argv[d] = items[d][0];
      }
      if (d < 0) break;
    }
  }
  Ref keys(PyDict_Keys(buckets.p));
  if (!keys.p) return nullptr;
  Ref out_symbols(PyList_AsTuple(keys.p));
  if (!out_symbols.p) return nullptr;
  Ref kept_b(PyBytes_FromStringAndSize(reinterpret_cast<const char*>(kept.data()),
                                       (Py_ssize_t)(kept.size() * sizeof(int64_t))));
  Ref idx_b(PyBytes_FromStringAndSize(reinterpret_cast<const char*>(out_idx.data()),
                                      (Py_ssize_t)(out_idx.size() * sizeof(int32_t))));
  if (!kept_b.p || !idx_b.p) return nullptr;
  return Py_BuildValue("(OOOL)", out_symbols.p, kept_b.p, idx_b.p, calls);
}

PyMethodDef methods[] = {
    {"map_shuffle", map_shuffle, METH_VARARGS,
     "map_shuffle(f, cond, symbol_lists, undefined) -> (out_symbols, kept, out_idx, calls) | ('error', syms, exc)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_planner", "Native host map/shuffle for apply_if", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__planner(void) { return PyModule_Create(&module); }
