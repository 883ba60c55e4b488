// hostpath.cpp — CPython binding of the host-buffer entry point tb_bleu_host
// (include/tensorbleu.h) for the package's host path.
//
// The reference's entry points (`sentence_bleu` / `corpus_bleu` /
// `compute_stats`, pkg/src/batchbleu/bleu.py:173-305) take host arrays and
// return numpy results; its kernels release the GIL
// (pkg/src/batchbleu/_kernels.pyx:63,113,164).  This module is the thin
// native layer between the Python mirror (bleu.py) and the C ABI: it takes
// the cached row views of the TokenBatch objects, allocates the numpy
// outputs, releases the GIL for the blocking device call, and returns the
// status so that Python raises the reference's exception types.
//
//   run(mode, views, batch, max_order, smoothing, eps, k, weights_addr, stream)
//     mode    0 = stats, 1 = sentence, 2 = corpus
//     views   tuple of (ids_ptr, ld, width, lengths_ptr, token_bytes), candidate first
//   -> (rc, flags, *outputs)
//     stats:    num (B,N) i64, den (B,N) i64, cand_len (B,) i64, eff_ref (B,) i64
//     sentence: scores (B,) f64, precisions (B,N) f64, bp (B,) f64
//     corpus:   totals (2N+2,) i64, corpus (N+2,) f64 = [score, bp, precisions]
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>

#include <cstdint>

#include "../../include/tensorbleu.h"

namespace {

bool view_of(PyObject* t, const void** ids, int64_t* ld, int64_t* width, const int64_t** len, int* tb) {
  if (!PyTuple_Check(t) || PyTuple_GET_SIZE(t) != 5) {
    PyErr_SetString(PyExc_TypeError, "row view must be a 5-tuple");
    return false;
  }
  *ids = reinterpret_cast<const void*>(PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(t, 0)));
  *ld = PyLong_AsLongLong(PyTuple_GET_ITEM(t, 1));
  *width = PyLong_AsLongLong(PyTuple_GET_ITEM(t, 2));
  *len = reinterpret_cast<const int64_t*>(PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(t, 3)));
  *tb = static_cast<int>(PyLong_AsLong(PyTuple_GET_ITEM(t, 4)));
  return !PyErr_Occurred();
}

PyObject* new_array(int nd, npy_intp d0, npy_intp d1, int type) {
  npy_intp dims[2] = {d0, d1};
  return PyArray_SimpleNew(nd, dims, type);
}

void* data(PyObject* a) { return PyArray_DATA(reinterpret_cast<PyArrayObject*>(a)); }

PyObject* run(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 9) {
    PyErr_SetString(PyExc_TypeError, "run() takes 9 arguments");
    return nullptr;
  }
  const long mode = PyLong_AsLong(args[0]);
  PyObject* views = args[1];
  const int64_t B = PyLong_AsLongLong(args[2]);
  const int N = static_cast<int>(PyLong_AsLong(args[3]));
  const int smoothing = static_cast<int>(PyLong_AsLong(args[4]));
  const double eps = PyFloat_AsDouble(args[5]);
  const double k = PyFloat_AsDouble(args[6]);
  const double* weights = reinterpret_cast<const double*>(PyLong_AsUnsignedLongLong(args[7]));
  void* stream = reinterpret_cast<void*>(PyLong_AsUnsignedLongLong(args[8]));
  if (PyErr_Occurred()) return nullptr;
  if (!PyTuple_Check(views) || PyTuple_GET_SIZE(views) < 2 || PyTuple_GET_SIZE(views) > TB_MAX_REFS + 1) {
    PyErr_SetString(PyExc_ValueError, "views must hold the candidate and 1..TB_MAX_REFS references");
    return nullptr;
  }
  if (B < 0 || N < 1 || N > TB_MAX_ORDER) {
    PyErr_SetString(PyExc_ValueError, "bad batch size or max_order");
    return nullptr;
  }
  const int R = static_cast<int>(PyTuple_GET_SIZE(views)) - 1;
  const void* ids[TB_MAX_REFS + 1];
  const int64_t* lens[TB_MAX_REFS + 1];
  int64_t lds[TB_MAX_REFS + 1], widths[TB_MAX_REFS + 1];
  int tb = 0;
  for (int s = 0; s <= R; ++s) {
    int tbs = 0;
    if (!view_of(PyTuple_GET_ITEM(views, s), &ids[s], &lds[s], &widths[s], &lens[s], &tbs)) return nullptr;
    if (s == 0) tb = tbs;
    if (tbs != tb) {
      PyErr_SetString(PyExc_ValueError, "all row views must share one token width");
      return nullptr;
    }
  }
  PyObject* o[4] = {nullptr, nullptr, nullptr, nullptr};
  int nout = 0;
  if (mode == 0) {
    o[0] = new_array(2, B, N, NPY_INT64);
    o[1] = new_array(2, B, N, NPY_INT64);
    o[2] = new_array(1, B, 0, NPY_INT64);
    o[3] = new_array(1, B, 0, NPY_INT64);
    nout = 4;
  } else if (mode == 1) {
    o[0] = new_array(1, B, 0, NPY_FLOAT64);
    o[1] = new_array(2, B, N, NPY_FLOAT64);
    o[2] = new_array(1, B, 0, NPY_FLOAT64);
    nout = 3;
  } else {
    o[0] = new_array(1, 2 * N + 2, 0, NPY_INT64);
    o[1] = new_array(1, N + 2, 0, NPY_FLOAT64);
    nout = 2;
  }
  for (int i = 0; i < nout; ++i)
    if (!o[i]) {
      for (int j = 0; j < nout; ++j) Py_XDECREF(o[j]);
      return nullptr;
    }
  int64_t *num = nullptr, *den = nullptr, *cl = nullptr, *er = nullptr, *tot = nullptr;
  double *sc = nullptr, *prec = nullptr, *bp = nullptr, *cor = nullptr;
  if (mode == 0) {
    num = static_cast<int64_t*>(data(o[0]));
    den = static_cast<int64_t*>(data(o[1]));
    cl = static_cast<int64_t*>(data(o[2]));
    er = static_cast<int64_t*>(data(o[3]));
  } else if (mode == 1) {
    sc = static_cast<double*>(data(o[0]));
    prec = static_cast<double*>(data(o[1]));
    bp = static_cast<double*>(data(o[2]));
  } else {
    tot = static_cast<int64_t*>(data(o[0]));
    cor = static_cast<double*>(data(o[1]));
  }
  int32_t flags = 0;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = tb_bleu_host(tb, ids[0], lds[0], widths[0], lens[0], R, ids + 1, lds + 1, widths + 1, lens + 1, B, N,
                    smoothing, eps, k, weights, num, den, cl, er, sc, prec, bp, tot, cor, &flags, stream);
  Py_END_ALLOW_THREADS
  PyObject* res = PyTuple_New(2 + nout);
  if (!res) {
    for (int j = 0; j < nout; ++j) Py_DECREF(o[j]);
    return nullptr;
  }
  PyTuple_SET_ITEM(res, 0, PyLong_FromLong(rc));
  PyTuple_SET_ITEM(res, 1, PyLong_FromLong(flags));
  for (int i = 0; i < nout; ++i) PyTuple_SET_ITEM(res, 2 + i, o[i]);
  return res;
}

// launch(views, batch, max_order, smoothing, eps, k, weights_addr, outs, err_addr, ws_addr, ws_bytes, stream)
//   -> rc.  Asynchronous tb_bleu_stats on device rows; `outs` is a 9-tuple of
//   device addresses or None: num, den, cand_len, eff_ref, scores,
//   precisions, bp, totals, corpus.
PyObject* launch(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 12) {
    PyErr_SetString(PyExc_TypeError, "launch() takes 12 arguments");
    return nullptr;
  }
  PyObject* views = args[0];
  const int64_t B = PyLong_AsLongLong(args[1]);
  const int N = static_cast<int>(PyLong_AsLong(args[2]));
  const int smoothing = static_cast<int>(PyLong_AsLong(args[3]));
  const double eps = PyFloat_AsDouble(args[4]);
  const double k = PyFloat_AsDouble(args[5]);
  const double* weights = reinterpret_cast<const double*>(PyLong_AsUnsignedLongLong(args[6]));
  PyObject* outs = args[7];
  int32_t* err = reinterpret_cast<int32_t*>(PyLong_AsUnsignedLongLong(args[8]));
  void* ws = reinterpret_cast<void*>(PyLong_AsUnsignedLongLong(args[9]));
  const size_t ws_bytes = static_cast<size_t>(PyLong_AsUnsignedLongLong(args[10]));
  void* stream = reinterpret_cast<void*>(PyLong_AsUnsignedLongLong(args[11]));
  if (PyErr_Occurred()) return nullptr;
  if (!PyTuple_Check(views) || PyTuple_GET_SIZE(views) < 2 || PyTuple_GET_SIZE(views) > TB_MAX_REFS + 1 ||
      !PyTuple_Check(outs) || PyTuple_GET_SIZE(outs) != 9) {
    PyErr_SetString(PyExc_ValueError, "bad views / outs");
    return nullptr;
  }
  const int R = static_cast<int>(PyTuple_GET_SIZE(views)) - 1;
  const void* ids[TB_MAX_REFS + 1];
  const int64_t* lens[TB_MAX_REFS + 1];
  int64_t lds[TB_MAX_REFS + 1], widths[TB_MAX_REFS + 1];
  int tb = 0;
  for (int s = 0; s <= R; ++s) {
    int tbs = 0;
    if (!view_of(PyTuple_GET_ITEM(views, s), &ids[s], &lds[s], &widths[s], &lens[s], &tbs)) return nullptr;
    if (s == 0) tb = tbs;
    if (tbs != tb) {
      PyErr_SetString(PyExc_ValueError, "all row views must share one token width");
      return nullptr;
    }
  }
  void* o[9];
  for (int i = 0; i < 9; ++i) {
    PyObject* x = PyTuple_GET_ITEM(outs, i);
    o[i] = x == Py_None ? nullptr : reinterpret_cast<void*>(PyLong_AsUnsignedLongLong(x));
  }
  if (PyErr_Occurred()) return nullptr;
  const int rc = tb_bleu_stats(tb, ids[0], lds[0], widths[0], lens[0], R, ids + 1, lds + 1, widths + 1, lens + 1, B,
                               N, smoothing, eps, k, weights, static_cast<int64_t*>(o[0]),
                               static_cast<int64_t*>(o[1]), static_cast<int64_t*>(o[2]), static_cast<int64_t*>(o[3]),
                               static_cast<double*>(o[4]), static_cast<double*>(o[5]), static_cast<double*>(o[6]),
                               static_cast<int64_t*>(o[7]), static_cast<double*>(o[8]), err, ws, ws_bytes, stream);
  return PyLong_FromLong(rc);
}

PyMethodDef kMethods[] = {
    {"launch", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(launch)), METH_FASTCALL,
     "launch(views, batch, max_order, smoothing, eps, k, weights_addr, outs, err_addr, ws_addr, ws_bytes, "
     "stream) -> rc"},
    {"run", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(run)), METH_FASTCALL,
     "run(mode, views, batch, max_order, smoothing, eps, k, weights_addr, stream) -> (rc, flags, *outputs)"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_hostpath",
                       "Native host-buffer path of paper_2510_05485_b200 (tb_bleu_host).", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__hostpath(void) {
  import_array();
  return PyModule_Create(&kModule);
}
