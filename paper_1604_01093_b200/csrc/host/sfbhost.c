/*
 * _sfbhost: the host-side stacking of correspondence sets (build_sparse_term,
 * reference solver.py:89-111) in C.  A global problem has tens of thousands
 * of CorrespondenceSet objects; walking them from Python costs ~1 us each,
 * here one pass reads every set's frame ids and points (numpy C API) and
 * memcpy's the (k, 3) float64 blocks into place.
 *
 * stack_sets_into: see below.  Raises KeyError for a frame outside the problem
 * (as build_sparse_term) and ValueError when points_i / points_j differ in rows.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

/* one set's two point blocks: data pointers into arrays kept alive by refs */
typedef struct {
  PyObject *ai, *aj;
  const char *pi, *pj;
} SetBufs;

/* (k, 3) C-contiguous aligned native float64 ndarray -> its data and rows
 * (the numpy C API: no buffer-export cost per set) */
static int get_f64_rows(PyObject* arr, const char** data, Py_ssize_t* rows) {
  if (!PyArray_Check(arr)) return 0;
  PyArrayObject* a = (PyArrayObject*)arr;
  if (PyArray_TYPE(a) != NPY_DOUBLE || PyArray_NDIM(a) != 2 || PyArray_DIM(a, 1) != 3 ||
      !PyArray_ISCARRAY_RO(a) || !PyArray_ISNOTSWAPPED(a))
    return 0;
  *data = (const char*)PyArray_DATA(a);
  *rows = PyArray_DIM(a, 0);
  return 1;
}

/* set range [s0, s1) of the stacked copy */
#define COPY_THREADS 6
typedef struct {
  const SetBufs* b;
  const int64_t* of;
  char *di, *dj;
  Py_ssize_t s0, s1;
} CopyTask;

static void* copy_task(void* arg) {
  const CopyTask* t = (const CopyTask*)arg;
  for (Py_ssize_t s = t->s0; s < t->s1; ++s) {
    const size_t nb = (size_t)(t->of[s + 1] - t->of[s]) * 24;
    if (nb) {
      memcpy(t->di + t->of[s] * 24, t->b[s].pi, nb);
      memcpy(t->dj + t->of[s] * 24, t->b[s].pj, nb);
    }
  }
  return NULL;
}

/* interned attribute names (PyObject_GetAttrString would build a str per call) */
static PyObject *s_frame_i, *s_frame_j, *s_points_i, *s_points_j;

static int frame_of(PyObject* set, PyObject* attr, PyObject* index, int32_t* out) {
  PyObject* f = PyObject_GetAttr(set, attr);
  if (!f) return -1;
  PyObject* v = PyDict_GetItemWithError(index, f);  /* borrowed */
  if (!v) {
    if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, f);
    Py_DECREF(f);
    return -1;
  }
  Py_DECREF(f);
  const long k = PyLong_AsLong(v);
  if (k == -1 && PyErr_Occurred()) return -1;
  *out = (int32_t)k;
  return 0;
}

static int writable(PyObject* o, Py_buffer* v, Py_ssize_t need) {
  if (PyObject_GetBuffer(o, v, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) != 0) return 0;
  if (v->len < need) {
    PyBuffer_Release(v);
    return -1;
  }
  return 1;
}

/* stack_sets_into(sets, frame_index, frames, offsets, points_i, points_j) ->
 *   total rows N (>= 0) when written, -N - 1 when points_i / points_j are too
 *   small for N rows (frames / offsets must hold n and n + 1 entries), or None
 *   when a set's points are not C-contiguous float64 (k, 3) ndarrays.
 * Outputs are caller-owned (reused, pinned) buffers: no allocation, no page
 * faults per call. */
static PyObject* stack_sets_into(PyObject* self, PyObject* args) {
  PyObject *seq_in, *index, *o_fr, *o_of, *o_pi, *o_pj;
  (void)self;
  if (!PyArg_ParseTuple(args, "OO!OOOO", &seq_in, &PyDict_Type, &index, &o_fr, &o_of, &o_pi,
                        &o_pj))
    return NULL;
  PyObject* seq = PySequence_Fast(seq_in, "sets must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyObject** items = PySequence_Fast_ITEMS(seq);
  SetBufs* b = (SetBufs*)PyMem_Calloc((size_t)(n > 0 ? n : 1), sizeof(SetBufs));
  Py_buffer vf, vo, vi, vj;
  int hf = 0, ho = 0, hi = 0, hj = 0;
  PyObject* res = NULL;
  if (!b) {
    PyErr_NoMemory();
    goto done;
  }
  if ((hf = writable(o_fr, &vf, 8 * n)) <= 0 || (ho = writable(o_of, &vo, 8 * (n + 1))) <= 0) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "frames / offsets buffer too small");
    hf = hf > 0;
    ho = ho > 0;
    goto done;
  }
  int32_t* fr = (int32_t*)vf.buf;
  int64_t* of = (int64_t*)vo.buf;
  int64_t total = 0;
  int fast = 1;
  of[0] = 0;
  for (Py_ssize_t s = 0; s < n; ++s) {
    PyObject* cs = items[s];
    if (frame_of(cs, s_frame_i, index, &fr[2 * s]) < 0) goto done;
    if (frame_of(cs, s_frame_j, index, &fr[2 * s + 1]) < 0) goto done;
    if (fast) {
      PyObject* ai = PyObject_GetAttr(cs, s_points_i);
      PyObject* aj = ai ? PyObject_GetAttr(cs, s_points_j) : NULL;
      if (!ai || !aj) {
        Py_XDECREF(ai);
        goto done;
      }
      Py_ssize_t ri = 0, rj = 0;
      b[s].ai = ai;  /* references released at the end */
      b[s].aj = aj;
      const int ok = get_f64_rows(ai, &b[s].pi, &ri) && get_f64_rows(aj, &b[s].pj, &rj);
      if (!ok) {
        fast = 0;  /* keep validating frames; the caller takes the NumPy path */
      } else if (ri != rj) {
        PyErr_SetString(PyExc_ValueError,
                        "points_i and points_j of a correspondence set differ in shape");
        goto done;
      } else {
        total += ri;
      }
    }
    of[s + 1] = total;
  }
  if (!fast) {
    res = Py_NewRef(Py_None);
    goto done;
  }
  hi = writable(o_pi, &vi, 24 * total);
  hj = hi > 0 ? writable(o_pj, &vj, 24 * total) : 0;
  if (hi < 0 || hj < 0 || (hi > 0 && hj == 0 && !PyErr_Occurred())) {
    hi = hi > 0;
    hj = hj > 0;
    res = PyLong_FromLongLong(-(long long)total - 1);
    goto done;
  }
  if (hi == 0 || hj == 0) goto done;
  {
    /* the copies need no Python objects (b[] holds the references): release
     * the GIL - the frames-upload thread can finish meanwhile - and split
     * large stacks over a few threads by set range */
    CopyTask t[COPY_THREADS];
    const int64_t bytes = total * 48;
    int nt = bytes >= ((int64_t)4 << 20) ? COPY_THREADS : 1;
    if (nt > n) nt = n > 0 ? (int)n : 1;
    Py_BEGIN_ALLOW_THREADS
    pthread_t th[COPY_THREADS];
    int started[COPY_THREADS] = {0};
    for (int k = 0; k < nt; ++k) {
      /* balance by rows: task k copies the sets whose first row lies in its share */
      t[k] = (CopyTask){b, of, (char*)vi.buf, (char*)vj.buf, 0, 0};
      const int64_t lo = total * k / nt, hi = total * (k + 1) / nt;
      Py_ssize_t s0 = 0, s1 = n;
      { Py_ssize_t a = 0, z = n; while (a < z) { Py_ssize_t m = (a + z) / 2; if (of[m] < lo) a = m + 1; else z = m; } s0 = a; }
      { Py_ssize_t a = 0, z = n; while (a < z) { Py_ssize_t m = (a + z) / 2; if (of[m] < hi) a = m + 1; else z = m; } s1 = a; }
      if (k == nt - 1) s1 = n;
      if (k == 0) s0 = 0;
      t[k].s0 = s0;
      t[k].s1 = s1;
    }
    for (int k = 1; k < nt; ++k) started[k] = pthread_create(&th[k], NULL, copy_task, &t[k]) == 0;
    copy_task(&t[0]);
    for (int k = 1; k < nt; ++k) {
      if (started[k]) pthread_join(th[k], NULL);
      else copy_task(&t[k]);
    }
    Py_END_ALLOW_THREADS
  }
  res = PyLong_FromLongLong((long long)total);
done:
  if (b) {
    for (Py_ssize_t s = 0; s < n; ++s) {
      Py_XDECREF(b[s].ai);
      Py_XDECREF(b[s].aj);
    }
    PyMem_Free(b);
  }
  if (hf > 0) PyBuffer_Release(&vf);
  if (ho > 0) PyBuffer_Release(&vo);
  if (hi > 0) PyBuffer_Release(&vi);
  if (hj > 0) PyBuffer_Release(&vj);
  Py_DECREF(seq);
  return res;
}

/* sfb_frame_desc (include/sfb.h) */
typedef struct {
  int32_t width, height;
  double fx, fy, cx, cy;
  const void *valid_depth, *valid_normal, *points, *normals, *grad;
} FrameDesc;

static PyObject *s_vd, *s_vn, *s_pts, *s_nrm, *s_grad, *s_k, *s_fx, *s_fy, *s_cx, *s_cy, *s_w,
    *s_h;

/* plane -> data pointer when it is an aligned C-contiguous ndarray of the
 * given type and shape (h, w[, c]) */
static const void* plane(PyObject* o, int type, npy_intp h, npy_intp w, int c) {
  if (!o || !PyArray_Check(o)) return NULL;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_TYPE(a) != type || !PyArray_ISCARRAY_RO(a) || !PyArray_ISNOTSWAPPED(a)) return NULL;
  if (PyArray_NDIM(a) != (c ? 3 : 2) || PyArray_DIM(a, 0) != h || PyArray_DIM(a, 1) != w ||
      (c && PyArray_DIM(a, 2) != c))
    return NULL;
  return PyArray_DATA(a);
}

static int attr_double(PyObject* o, PyObject* name, double* out) {
  PyObject* v = PyObject_GetAttr(o, name);
  if (!v) return -1;
  *out = PyFloat_AsDouble(v);
  Py_DECREF(v);
  return (*out == -1.0 && PyErr_Occurred()) ? -1 : 0;
}

/* fill_frame_descs(caches, descs) -> True, or None when some plane is not in
 * the library's layout (bool / float32, C-contiguous, (h, w[, c])).  descs is
 * a writable buffer of len(caches) sfb_frame_desc; the planes stay owned by
 * the caches (borrowed for the upload call). */
static PyObject* fill_frame_descs(PyObject* self, PyObject* args) {
  PyObject *seq_in, *out;
  (void)self;
  if (!PyArg_ParseTuple(args, "OO", &seq_in, &out)) return NULL;
  PyObject* seq = PySequence_Fast(seq_in, "caches must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyObject** items = PySequence_Fast_ITEMS(seq);
  Py_buffer v;
  PyObject* res = NULL;
  if (PyObject_GetBuffer(out, &v, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) != 0) {
    Py_DECREF(seq);
    return NULL;
  }
  if (v.len < (Py_ssize_t)sizeof(FrameDesc) * n) {
    PyErr_SetString(PyExc_ValueError, "descriptor buffer too small");
    goto done;
  }
  FrameDesc* d = (FrameDesc*)v.buf;
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* c = items[k];
    PyObject* o[5] = {PyObject_GetAttr(c, s_vd), PyObject_GetAttr(c, s_vn),
                      PyObject_GetAttr(c, s_pts), PyObject_GetAttr(c, s_nrm),
                      PyObject_GetAttr(c, s_grad)};
    PyObject* kk = PyObject_GetAttr(c, s_k);
    int ok = o[0] && o[1] && o[2] && o[3] && o[4] && kk;
    if (ok && PyArray_Check(o[0]) && PyArray_NDIM((PyArrayObject*)o[0]) == 2) {
      const npy_intp h = PyArray_DIM((PyArrayObject*)o[0], 0), w = PyArray_DIM((PyArrayObject*)o[0], 1);
      d[k].valid_depth = plane(o[0], NPY_BOOL, h, w, 0);
      d[k].valid_normal = plane(o[1], NPY_BOOL, h, w, 0);
      d[k].points = plane(o[2], NPY_FLOAT32, h, w, 3);
      d[k].normals = plane(o[3], NPY_FLOAT32, h, w, 3);
      d[k].grad = plane(o[4], NPY_FLOAT32, h, w, 2);
      d[k].width = (int32_t)w;
      d[k].height = (int32_t)h;
      ok = d[k].valid_depth && d[k].valid_normal && d[k].points && d[k].normals && d[k].grad;
      if (ok) {
        double kw = 0, kh = 0;
        if (attr_double(kk, s_fx, &d[k].fx) || attr_double(kk, s_fy, &d[k].fy) ||
            attr_double(kk, s_cx, &d[k].cx) || attr_double(kk, s_cy, &d[k].cy) ||
            attr_double(kk, s_w, &kw) || attr_double(kk, s_h, &kh)) {
          PyErr_Clear();
          ok = 0;
        } else if ((npy_intp)kw != w || (npy_intp)kh != h) {
          ok = 0;  /* the NumPy path raises the size mismatch */
        }
      }
    } else {
      PyErr_Clear();
      ok = 0;
    }
    for (int q = 0; q < 5; ++q) Py_XDECREF(o[q]);
    Py_XDECREF(kk);
    if (!ok) {
      res = Py_NewRef(Py_None);
      goto done;
    }
  }
  res = Py_NewRef(Py_True);
done:
  PyBuffer_Release(&v);
  Py_DECREF(seq);
  return res;
}

/* ---- poses (solver._push_poses / _pull_poses) ---------------------------- */
static PyObject *s_rotation, *s_translation;

/* float64 ndarray of `n` elements in any layout -> out (C order) */
static int copy_f64(PyObject* o, int nd, const npy_intp* dims, double* out) {
  if (!PyArray_Check(o)) return 0;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_TYPE(a) != NPY_DOUBLE || !PyArray_ISNOTSWAPPED(a)) return 0;
  if (nd == 2) {
    if (PyArray_NDIM(a) != 2 || PyArray_DIM(a, 0) != dims[0] || PyArray_DIM(a, 1) != dims[1]) return 0;
    for (npy_intp r = 0; r < dims[0]; ++r)
      for (npy_intp c = 0; c < dims[1]; ++c) memcpy(out++, PyArray_GETPTR2(a, r, c), 8);
    return 1;
  }
  /* translation: any shape holding dims[0] elements (np.reshape(3)) */
  if (PyArray_SIZE(a) != dims[0]) return 0;
  if (PyArray_NDIM(a) == 1) {
    for (npy_intp k = 0; k < dims[0]; ++k) memcpy(out++, PyArray_GETPTR1(a, k), 8);
    return 1;
  }
  if (!PyArray_ISCARRAY_RO(a)) return 0;
  memcpy(out, PyArray_DATA(a), 8 * (size_t)dims[0]);
  return 1;
}

static int out_array(PyObject* o, int typenum, npy_intp n, char** data) {
  if (!PyArray_Check(o)) return 0;
  PyArrayObject* a = (PyArrayObject*)o;
  if (PyArray_TYPE(a) != typenum || !PyArray_ISCARRAY(a) || PyArray_SIZE(a) != n) return 0;
  *data = (char*)PyArray_DATA(a);
  return 1;
}

/* pack_poses(poses, R, t, fl) -> True | None.  R (n,3,3), t (n,3) float64 and
 * fl (n,) uint8 C arrays; fl[k] = rotation F-ordered (not C), the BLAS
 * operand-order flag of device_problem._pose_arrays.  None: an entry is not a
 * float64 ndarray pair (the caller takes the NumPy path). */
static PyObject* pack_poses(PyObject* self, PyObject* args) {
  PyObject *poses, *Ro, *to, *flo;
  if (!PyArg_ParseTuple(args, "OOOO", &poses, &Ro, &to, &flo)) return NULL;
  PyObject* seq = PySequence_Fast(poses, "poses must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  char *R, *t, *fl;
  PyObject* res = NULL;
  if (!out_array(Ro, NPY_DOUBLE, 9 * n, &R) || !out_array(to, NPY_DOUBLE, 3 * n, &t) ||
      !out_array(flo, NPY_UINT8, n, &fl)) {
    PyErr_SetString(PyExc_ValueError, "pack_poses: bad output arrays");
    goto done;
  }
  static const npy_intp d33[2] = {3, 3}, d3[1] = {3};
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* p = PySequence_Fast_GET_ITEM(seq, k);
    PyObject* rot = PyObject_GetAttr(p, s_rotation);
    if (!rot) goto done;
    PyObject* tr = PyObject_GetAttr(p, s_translation);
    if (!tr) {
      Py_DECREF(rot);
      goto done;
    }
    const int ok = copy_f64(rot, 2, d33, (double*)R + 9 * k) && copy_f64(tr, 1, d3, (double*)t + 3 * k);
    if (ok) {
      PyArrayObject* a = (PyArrayObject*)rot;
      fl[k] = (PyArray_IS_F_CONTIGUOUS(a) && !PyArray_IS_C_CONTIGUOUS(a)) ? 1 : 0;
    }
    Py_DECREF(rot);
    Py_DECREF(tr);
    if (!ok) {
      res = Py_NewRef(Py_None);
      goto done;
    }
  }
  res = Py_NewRef(Py_True);
done:
  Py_DECREF(seq);
  return res;
}

/* make_poses(poses, frame_ids, R, t, cls, first) -> None: for k >= first,
 * poses[frame_ids[k]] = cls(R[k].copy(), t[k].copy()). */
static PyObject* make_poses(PyObject* self, PyObject* args) {
  PyObject *poses, *ids, *Ro, *to, *cls;
  Py_ssize_t first;
  if (!PyArg_ParseTuple(args, "O!OOOOn", &PyDict_Type, &poses, &ids, &Ro, &to, &cls, &first))
    return NULL;
  PyObject* seq = PySequence_Fast(ids, "frame_ids must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  char *R, *t;
  PyObject* res = NULL;
  if (!out_array(Ro, NPY_DOUBLE, 9 * n, &R) || !out_array(to, NPY_DOUBLE, 3 * n, &t)) {
    PyErr_SetString(PyExc_ValueError, "make_poses: bad input arrays");
    goto done;
  }
  for (Py_ssize_t k = first; k < n; ++k) {
    npy_intp d33[2] = {3, 3}, d3[1] = {3};
    PyObject* rk = PyArray_SimpleNew(2, d33, NPY_DOUBLE);
    PyObject* tk = rk ? PyArray_SimpleNew(1, d3, NPY_DOUBLE) : NULL;
    if (!tk) {
      Py_XDECREF(rk);
      goto done;
    }
    memcpy(PyArray_DATA((PyArrayObject*)rk), R + 72 * k, 72);
    memcpy(PyArray_DATA((PyArrayObject*)tk), t + 24 * k, 24);
    PyObject* obj = PyObject_CallFunctionObjArgs(cls, rk, tk, NULL);
    Py_DECREF(rk);
    Py_DECREF(tk);
    if (!obj) goto done;
    const int rc = PyDict_SetItem(poses, PySequence_Fast_GET_ITEM(seq, k), obj);
    Py_DECREF(obj);
    if (rc) goto done;
  }
  res = Py_NewRef(Py_None);
done:
  Py_DECREF(seq);
  return res;
}

static PyMethodDef methods[] = {
    {"pack_poses", pack_poses, METH_VARARGS, "pack_poses(poses, R, t, fl) -> True | None"},
    {"make_poses", make_poses, METH_VARARGS,
     "make_poses(poses, frame_ids, R, t, cls, first) -> None"},
    {"fill_frame_descs", fill_frame_descs, METH_VARARGS,
     "fill_frame_descs(caches, descs) -> True | None"},
    {"stack_sets_into", stack_sets_into, METH_VARARGS,
     "stack_sets_into(sets, frame_index, frames, offsets, points_i, points_j) -> N | -N-1 | None"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sfbhost",
                                    "host-side helpers of the B200 solver", -1, methods};

PyMODINIT_FUNC PyInit__sfbhost(void) {
  import_array();
  s_frame_i = PyUnicode_InternFromString("frame_i");
  s_frame_j = PyUnicode_InternFromString("frame_j");
  s_points_i = PyUnicode_InternFromString("points_i");
  s_points_j = PyUnicode_InternFromString("points_j");
  if (!s_frame_i || !s_frame_j || !s_points_i || !s_points_j) return NULL;
  s_rotation = PyUnicode_InternFromString("rotation");
  s_translation = PyUnicode_InternFromString("translation");
  if (!s_rotation || !s_translation) return NULL;
  s_vd = PyUnicode_InternFromString("valid_depth");
  s_vn = PyUnicode_InternFromString("valid_normal");
  s_pts = PyUnicode_InternFromString("points_low");
  s_nrm = PyUnicode_InternFromString("normals_low");
  s_grad = PyUnicode_InternFromString("grad_low");
  s_k = PyUnicode_InternFromString("intrinsics_low");
  s_fx = PyUnicode_InternFromString("fx");
  s_fy = PyUnicode_InternFromString("fy");
  s_cx = PyUnicode_InternFromString("cx");
  s_cy = PyUnicode_InternFromString("cy");
  s_w = PyUnicode_InternFromString("width");
  s_h = PyUnicode_InternFromString("height");
  return PyModule_Create(&module);
}
