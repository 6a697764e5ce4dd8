/*
 * jsv_decode.c -- CPython extension `_jsvdecode`: turns a batch of
 * jsv_plan_out records (include/jsv.h) into the drop-in's PlanResult objects.
 *
 * Same objects and the same insertion orders as planner._results_from (the
 * pure-Python decoder kept as the reference for this one, and used when this
 * module is not built): the per-result work is ~60 Python objects, so doing it
 * from C removes the interpreter loop around them.  Frozen dataclasses are
 * instantiated with object.__new__ and filled with object.__setattr__ (what
 * their generated __init__ does), so ==, repr and dataclasses.* are unchanged.
 * Record field offsets come from the ctypes structure (no layout hard-coded).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  Py_ssize_t size, feasible, has_config, binding, objective, a_obj, nodes, pool_size,
      pool_present, truncated, n_items, items, hput, latency, capacity, demand, accuracy, slices,
      fanout, path_acc, total_slices, uncovered_mask, lat_margin, thr_margin, res_margin,
      acc_margin;
  Py_ssize_t max_items;
} Layout;

static int get_off(PyObject* d, const char* k, Py_ssize_t* out) {
  PyObject* v = PyDict_GetItemString(d, k);
  if (!v) {
    PyErr_Format(PyExc_KeyError, "layout field %s", k);
    return -1;
  }
  *out = PyLong_AsSsize_t(v);
  return PyErr_Occurred() ? -1 : 0;
}

static int32_t rd_i32(const char* b, Py_ssize_t off, Py_ssize_t i) {
  int32_t v;
  memcpy(&v, b + off + 4 * i, 4);
  return v;
}
static uint32_t rd_u32(const char* b, Py_ssize_t off, Py_ssize_t i) {
  uint32_t v;
  memcpy(&v, b + off + 4 * i, 4);
  return v;
}
static double rd_f64(const char* b, Py_ssize_t off, Py_ssize_t i) {
  double v;
  memcpy(&v, b + off + 8 * i, 8);
  return v;
}
static int64_t rd_i64(const char* b, Py_ssize_t off) {
  int64_t v;
  memcpy(&v, b + off, 8);
  return v;
}

static PyObject* s_empty;  /* () */
static PyObject *a_name, *a_subject, *a_passed, *a_margin, *a_nodes, *a_wall, *a_pool, *a_trunc,
    *a_feasible, *a_config, *a_objective, *a_amax, *a_binding, *a_verdicts, *a_stats, *a_m,
    *a_entry, *a_lat, *a_cap, *a_dem, *a_sl, *a_acc, *a_fan, *a_hput, *a_pacc, *a_tot, *a_aobj,
    *a_struct, *k_latency, *k_throughput, *k_resources, *k_accuracy, *k_coverage, *k_blank,
    *k_comma;

/* object.__new__(cls) */
static PyObject* new_of(PyObject* cls) {
  return PyBaseObject_Type.tp_new((PyTypeObject*)cls, s_empty, NULL);
}
/* object.__setattr__(o, name, v); steals v */
static int put(PyObject* o, PyObject* name, PyObject* v) {
  if (!v) return -1;
  int rc = PyObject_GenericSetAttr(o, name, v);
  Py_DECREF(v);
  return rc;
}
static PyObject* pfloat(double x) { return PyFloat_FromDouble(x); }
static PyObject* pint(long long x) { return PyLong_FromLongLong(x); }
static PyObject* pbool(int x) { return Py_NewRef(x ? Py_True : Py_False); }

#define CHK(x) \
  do {         \
    if ((x) < 0) goto fail; \
  } while (0)
#define NN(x) \
  do {        \
    if (!(x)) goto fail; \
  } while (0)

/* The cyclic GC only needs to see objects that can be part of a reference
 * cycle.  Immutable objects built here whose referents are all untracked
 * (strings, numbers, or objects untracked by this rule) cannot be, so they are
 * untracked as soon as they are complete -- the rule CPython applies to tuples
 * lazily during a collection, applied eagerly (and to the frozen dataclasses
 * filled here) so that the ~20 short-lived objects per result stay out of
 * every gen-0 traversal and never get promoted. */
static void untrack_tuple(PyObject* t) {
  for (Py_ssize_t k = 0; k < PyTuple_GET_SIZE(t); ++k)
    if (PyObject_GC_IsTracked(PyTuple_GET_ITEM(t, k))) return;
  PyObject_GC_UnTrack(t);
}

/* ConstraintVerdict(name: str, subject: str, passed: bool, margin: float) */
static PyObject* verdict(PyObject* cls, PyObject* name, PyObject* subject, int passed,
                         double margin) {
  PyObject* o = new_of(cls);
  if (!o) return NULL;
  if (put(o, a_name, Py_NewRef(name)) < 0 || put(o, a_subject, Py_NewRef(subject)) < 0 ||
      put(o, a_passed, pbool(passed)) < 0 || put(o, a_margin, pfloat(margin)) < 0) {
    Py_DECREF(o);
    return NULL;
  }
  if (!PyObject_GC_IsTracked(name) && !PyObject_GC_IsTracked(subject)) PyObject_GC_UnTrack(o);
  return o;
}

/* decode(buf, n, layout, meta, demands, wall_ms) -> list[PlanResult]
 * meta = (ids, keys_full, topo_t, topo_i, task_t, task_i, edge_names, edge_idx,
 *         paths, path_names, a_max, binding_names,
 *         PlanResult, Configuration, ConstraintVerdict, SolverStats, key_hashes)
 * key_hashes[ti][k] = hash(keys_full[ti][k]), computed once per lowering */
static PyObject* decode(PyObject* self, PyObject* args) {
  (void)self;
  Py_buffer view;
  Py_ssize_t n;
  PyObject *layout, *meta, *demands;
  double wall_ms;
  if (!PyArg_ParseTuple(args, "y*nO!O!O!d", &view, &n, &PyDict_Type, &layout, &PyTuple_Type, &meta,
                        &PyList_Type, &demands, &wall_ms))
    return NULL;
  PyObject* res = NULL;
  Layout L;
  memset(&L, 0, sizeof(L));
  if (get_off(layout, "size", &L.size) || get_off(layout, "feasible", &L.feasible) ||
      get_off(layout, "has_config", &L.has_config) || get_off(layout, "binding", &L.binding) ||
      get_off(layout, "objective", &L.objective) || get_off(layout, "a_obj", &L.a_obj) ||
      get_off(layout, "nodes", &L.nodes) || get_off(layout, "pool_size", &L.pool_size) ||
      get_off(layout, "pool_present", &L.pool_present) ||
      get_off(layout, "truncated", &L.truncated) || get_off(layout, "n_items", &L.n_items) ||
      get_off(layout, "items", &L.items) || get_off(layout, "hput", &L.hput) ||
      get_off(layout, "latency", &L.latency) || get_off(layout, "capacity", &L.capacity) ||
      get_off(layout, "demand", &L.demand) || get_off(layout, "accuracy", &L.accuracy) ||
      get_off(layout, "slices", &L.slices) || get_off(layout, "fanout", &L.fanout) ||
      get_off(layout, "path_acc", &L.path_acc) || get_off(layout, "total_slices", &L.total_slices) ||
      get_off(layout, "uncovered_mask", &L.uncovered_mask) ||
      get_off(layout, "lat_margin", &L.lat_margin) || get_off(layout, "thr_margin", &L.thr_margin) ||
      get_off(layout, "res_margin", &L.res_margin) || get_off(layout, "acc_margin", &L.acc_margin) ||
      get_off(layout, "max_items", &L.max_items)) {
    PyBuffer_Release(&view);
    return NULL;
  }
  if (PyTuple_GET_SIZE(meta) != 17 || view.len < n * L.size || PyList_GET_SIZE(demands) < n) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "decode: bad arguments");
    return NULL;
  }
  PyObject* ids = PyTuple_GET_ITEM(meta, 0);
  PyObject* keys_full = PyTuple_GET_ITEM(meta, 1);
  PyObject* key_hashes = PyTuple_GET_ITEM(meta, 16);
  if (!PyTuple_Check(key_hashes) || !PyTuple_Check(keys_full) ||
      PyTuple_GET_SIZE(key_hashes) != PyTuple_GET_SIZE(keys_full)) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "decode: bad key hashes");
    return NULL;
  }
  PyObject* topo_t = PyTuple_GET_ITEM(meta, 2);
  PyObject* topo_i = PyTuple_GET_ITEM(meta, 3);
  PyObject* task_t = PyTuple_GET_ITEM(meta, 4);
  PyObject* task_i = PyTuple_GET_ITEM(meta, 5);
  PyObject* edge_names = PyTuple_GET_ITEM(meta, 6);
  PyObject* edge_idx = PyTuple_GET_ITEM(meta, 7);
  PyObject* paths = PyTuple_GET_ITEM(meta, 8);
  PyObject* path_names = PyTuple_GET_ITEM(meta, 9);
  PyObject* a_max_o = PyTuple_GET_ITEM(meta, 10);
  PyObject* bnames = PyTuple_GET_ITEM(meta, 11);
  PyObject* C_res = PyTuple_GET_ITEM(meta, 12);
  PyObject* C_cfg = PyTuple_GET_ITEM(meta, 13);
  PyObject* C_ver = PyTuple_GET_ITEM(meta, 14);
  PyObject* C_st = PyTuple_GET_ITEM(meta, 15);
  const Py_ssize_t T = PyTuple_GET_SIZE(ids), NT = PyTuple_GET_SIZE(topo_t);
  const Py_ssize_t NTASK = PyTuple_GET_SIZE(task_t), E = PyTuple_GET_SIZE(edge_names);
  const Py_ssize_t P = PyTuple_GET_SIZE(paths);
  long ti_topo[64], ti_task[64], eidx[64];
  if (T > 64 || NT > 64 || NTASK > 64 || E > 64) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "decode: graph too large");
    return NULL;
  }
  for (Py_ssize_t k = 0; k < NT; ++k) ti_topo[k] = PyLong_AsLong(PyTuple_GET_ITEM(topo_i, k));
  for (Py_ssize_t k = 0; k < NTASK; ++k) ti_task[k] = PyLong_AsLong(PyTuple_GET_ITEM(task_i, k));
  for (Py_ssize_t k = 0; k < E; ++k) eidx[k] = PyLong_AsLong(PyTuple_GET_ITEM(edge_idx, k));
  const double a_max = PyFloat_AsDouble(a_max_o);
  res = PyList_New(n);
  if (!res) goto fail_nores;
  for (Py_ssize_t i = 0; i < n; ++i) {
    const char* b = (const char*)view.buf + i * L.size;
    PyObject *stats = NULL, *sizes = NULL, *cut = NULL, *r = NULL, *cfg = NULL, *vs = NULL;
    PyObject *m = NULL, *hput = NULL, *bad = NULL, *d = NULL;
    /* stats */
    NN(sizes = PyDict_New());
    NN(cut = PyList_New(0));
    for (Py_ssize_t k = 0; k < NT; ++k) {
      const long ti = ti_topo[k];
      if (rd_i32(b, L.pool_present, ti)) {
        PyObject* v = pint(rd_i32(b, L.pool_size, ti));
        NN(v);
        int rc = PyDict_SetItem(sizes, PyTuple_GET_ITEM(topo_t, k), v);
        Py_DECREF(v);
        CHK(rc);
        if (rd_i32(b, L.truncated, ti)) CHK(PyList_Append(cut, PyTuple_GET_ITEM(topo_t, k)));
      }
    }
    NN(stats = new_of(C_st));
    CHK(put(stats, a_nodes, pint(rd_i64(b, L.nodes))));
    CHK(put(stats, a_wall, pfloat(wall_ms)));
    {
      /* SolverStats(nodes, wall_ms, pool_sizes: {str: int}, truncated_tasks: (str, ...)) */
      PyObject* tt = PyList_AsTuple(cut);
      NN(tt);
      untrack_tuple(tt);
      const int leaf = !PyObject_GC_IsTracked(sizes) && !PyObject_GC_IsTracked(tt);
      CHK(put(stats, a_pool, sizes)); sizes = NULL;
      CHK(put(stats, a_trunc, tt));
      if (leaf) PyObject_GC_UnTrack(stats);
    }
    Py_CLEAR(cut);
    const int code = rd_i32(b, L.binding, 0);
    PyObject* bind = code < 0 ? Py_None : PyTuple_GET_ITEM(bnames, code);
    NN(r = new_of(C_res));
    if (!rd_i32(b, L.has_config, 0)) {
      CHK(put(r, a_feasible, pbool(0)));
      CHK(put(r, a_config, Py_NewRef(Py_None)));
      CHK(put(r, a_objective, Py_NewRef(Py_None)));
      CHK(put(r, a_amax, Py_NewRef(a_max_o)));
      CHK(put(r, a_binding, Py_NewRef(bind)));
      CHK(put(r, a_verdicts, Py_NewRef(s_empty)));
      CHK(put(r, a_stats, stats)); stats = NULL;
      PyList_SET_ITEM(res, i, r);
      continue;
    }
    /* m (task-id order) and hput (topological order) */
    NN(m = PyList_New(0));
    for (Py_ssize_t ti = 0; ti < T; ++ti) {
      PyObject* kt = PyTuple_GET_ITEM(keys_full, ti);
      const int ni = rd_i32(b, L.n_items, ti);
      for (int k = 0; k < ni; ++k) {
        const uint32_t w = rd_u32(b, L.items, ti * L.max_items + k);
        PyObject* e = Py_BuildValue("(On)", PyTuple_GET_ITEM(kt, w >> 16), (Py_ssize_t)(w & 0xFFFFu));
        NN(e);
        untrack_tuple(e);
        int rc = PyList_Append(m, e);
        Py_DECREF(e);
        CHK(rc);
      }
    }
    NN(hput = PyDict_New());
    for (Py_ssize_t k = 0; k < NT; ++k) {
      const long ti = ti_topo[k];
      PyObject* kt = PyTuple_GET_ITEM(keys_full, ti);
      PyObject* kh = PyTuple_GET_ITEM(key_hashes, ti);
      const int ni = rd_i32(b, L.n_items, ti);
      for (int j = 0; j < ni; ++j) {
        const uint32_t w = rd_u32(b, L.items, ti * L.max_items + j);
        const Py_hash_t h = (Py_hash_t)PyLong_AsSsize_t(PyTuple_GET_ITEM(kh, w >> 16));
        if (h == -1 && PyErr_Occurred()) goto fail;
        PyObject* v = pfloat(rd_f64(b, L.hput, ti * L.max_items + j));
        NN(v);
        int rc = _PyDict_SetItem_KnownHash(hput, PyTuple_GET_ITEM(kt, w >> 16), v, h);
        Py_DECREF(v);
        CHK(rc);
      }
    }
    const uint32_t unc = rd_u32(b, L.uncovered_mask, 0);
    {
      PyObject* bl = PyList_New(0);
      NN(bl);
      for (Py_ssize_t k = 0; k < NT && unc; ++k)
        if ((unc >> ti_topo[k]) & 1u)
          if (PyList_Append(bl, PyTuple_GET_ITEM(topo_t, k)) < 0) {
            Py_DECREF(bl);
            goto fail;
          }
      bad = PyList_AsTuple(bl);
      Py_DECREF(bl);
      NN(bad);
      untrack_tuple(bad);
    }
    NN(cfg = new_of(C_cfg));
    {
      PyObject* mt = PyList_AsTuple(m);
      Py_CLEAR(m);
      NN(mt);
      untrack_tuple(mt);
      CHK(put(cfg, a_m, mt));
    }
    CHK(put(cfg, a_entry, PyNumber_Float(PyList_GET_ITEM(demands, i))));
#define TASKDICT(ATTR, FIELD, ORDER_T, ORDER_I, CNT, CONV)                         \
  do {                                                                             \
    NN(d = PyDict_New());                                                          \
    for (Py_ssize_t k = 0; k < (CNT); ++k) {                                       \
      PyObject* v = CONV;                                                          \
      NN(v);                                                                       \
      int rc = PyDict_SetItem(d, PyTuple_GET_ITEM(ORDER_T, k), v);                 \
      Py_DECREF(v);                                                                \
      CHK(rc);                                                                     \
    }                                                                              \
    CHK(put(cfg, ATTR, d));                                                        \
    d = NULL;                                                                      \
  } while (0)
    TASKDICT(a_lat, latency, task_t, ti_task, NTASK, pfloat(rd_f64(b, L.latency, ti_task[k])));
    TASKDICT(a_cap, capacity, task_t, ti_task, NTASK, pfloat(rd_f64(b, L.capacity, ti_task[k])));
    TASKDICT(a_dem, demand, topo_t, ti_topo, NT, pfloat(rd_f64(b, L.demand, ti_topo[k])));
    TASKDICT(a_sl, slices, task_t, ti_task, NTASK, pint(rd_i32(b, L.slices, ti_task[k])));
    TASKDICT(a_acc, accuracy, task_t, ti_task, NTASK, pfloat(rd_f64(b, L.accuracy, ti_task[k])));
    TASKDICT(a_fan, fanout, edge_names, eidx, E, pfloat(rd_f64(b, L.fanout, eidx[k])));
    CHK(put(cfg, a_hput, hput)); hput = NULL;
    TASKDICT(a_pacc, path_acc, paths, , P, pfloat(rd_f64(b, L.path_acc, k)));
#undef TASKDICT
    CHK(put(cfg, a_tot, pint(rd_i32(b, L.total_slices, 0))));
    CHK(put(cfg, a_aobj, pfloat(rd_f64(b, L.a_obj, 0))));
    CHK(put(cfg, a_amax, Py_NewRef(a_max_o)));
    PyObject* objv = pfloat(rd_f64(b, L.objective, 0));
    NN(objv);
    if (PyObject_GenericSetAttr(cfg, a_objective, objv) < 0) {
      Py_DECREF(objv);
      goto fail;
    }
    CHK(put(cfg, a_struct, Py_NewRef(bad)));
    /* verdicts */
    {
      const Py_ssize_t nv = P + NT + 3;
      NN(vs = PyTuple_New(nv));
      Py_ssize_t q = 0;
      for (Py_ssize_t k = 0; k < P; ++k) {
        const double mg = rd_f64(b, L.lat_margin, k);
        PyObject* v = verdict(C_ver, k_latency, PyTuple_GET_ITEM(path_names, k), mg >= 0, mg);
        if (!v) { Py_DECREF(objv); goto fail; }
        PyTuple_SET_ITEM(vs, q++, v);
      }
      for (Py_ssize_t k = 0; k < NT; ++k) {
        const double mg = rd_f64(b, L.thr_margin, ti_topo[k]);
        PyObject* v = verdict(C_ver, k_throughput, PyTuple_GET_ITEM(topo_t, k), mg >= 0, mg);
        if (!v) { Py_DECREF(objv); goto fail; }
        PyTuple_SET_ITEM(vs, q++, v);
      }
      double mg = rd_f64(b, L.res_margin, 0);
      PyObject* v = verdict(C_ver, k_resources, k_blank, mg >= 0, mg);
      if (!v) { Py_DECREF(objv); goto fail; }
      PyTuple_SET_ITEM(vs, q++, v);
      mg = rd_f64(b, L.acc_margin, 0);
      v = verdict(C_ver, k_accuracy, k_blank, mg >= 0, mg);
      if (!v) { Py_DECREF(objv); goto fail; }
      PyTuple_SET_ITEM(vs, q++, v);
      PyObject* subj = PyUnicode_Join(k_comma, bad);
      if (!subj) { Py_DECREF(objv); goto fail; }
      const Py_ssize_t nb = PyTuple_GET_SIZE(bad);
      v = verdict(C_ver, k_coverage, subj, nb == 0, nb == 0 ? 0.0 : -(double)nb);
      Py_DECREF(subj);
      if (!v) { Py_DECREF(objv); goto fail; }
      PyTuple_SET_ITEM(vs, q++, v);
      untrack_tuple(vs);
    }
    {
      const int feas = rd_i32(b, L.feasible, 0) != 0;
      int ok = put(r, a_feasible, pbool(feas)) >= 0 &&
               PyObject_GenericSetAttr(r, a_config, cfg) >= 0 &&
               put(r, a_objective, feas ? Py_NewRef(objv) : Py_NewRef(Py_None)) >= 0 &&
               put(r, a_amax, Py_NewRef(a_max_o)) >= 0 &&
               put(r, a_binding, Py_NewRef(feas ? Py_None : bind)) >= 0 &&
               PyObject_GenericSetAttr(r, a_verdicts, vs) >= 0 && put(r, a_stats, stats) >= 0;
      stats = NULL;
      Py_DECREF(objv);
      if (!ok) goto fail;
    }
    Py_CLEAR(cfg);
    Py_CLEAR(vs);
    Py_CLEAR(bad);
    PyList_SET_ITEM(res, i, r);
    continue;
  fail:
    Py_XDECREF(stats); Py_XDECREF(sizes); Py_XDECREF(cut); Py_XDECREF(r); Py_XDECREF(cfg);
    Py_XDECREF(vs); Py_XDECREF(m); Py_XDECREF(hput); Py_XDECREF(bad); Py_XDECREF(d);
    Py_DECREF(res);
    res = NULL;
    break;
  }
fail_nores:
  PyBuffer_Release(&view);
  (void)a_max;
  return res;
}

static PyMethodDef methods[] = {
    {"decode", decode, METH_VARARGS, "decode(buf, n, layout, meta, demands, wall_ms)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_jsvdecode", NULL, -1, methods,
                                 NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__jsvdecode(void) {
  s_empty = PyTuple_New(0);
#define I(v, s) v = PyUnicode_InternFromString(s)
  I(a_name, "name"); I(a_subject, "subject"); I(a_passed, "passed"); I(a_margin, "margin");
  I(a_nodes, "nodes"); I(a_wall, "wall_ms"); I(a_pool, "pool_sizes"); I(a_trunc, "truncated_tasks");
  I(a_feasible, "feasible"); I(a_config, "config"); I(a_objective, "objective");
  I(a_amax, "a_max"); I(a_binding, "binding_constraint"); I(a_verdicts, "verdicts");
  I(a_stats, "stats"); I(a_m, "m"); I(a_entry, "entry_demand_rps"); I(a_lat, "latency_ms");
  I(a_cap, "capacity_rps"); I(a_dem, "demand_rps"); I(a_sl, "slices"); I(a_acc, "accuracy");
  I(a_fan, "fanout"); I(a_hput, "hput"); I(a_pacc, "path_accuracy"); I(a_tot, "total_slices");
  I(a_aobj, "a_obj"); I(a_struct, "structurally_infeasible");
  I(k_latency, "latency"); I(k_throughput, "throughput"); I(k_resources, "resources");
  I(k_accuracy, "accuracy"); I(k_coverage, "coverage"); I(k_blank, ""); I(k_comma, ",");
#undef I
  return PyModule_Create(&mod);
}
