/* packer.c — native host-side packing of rollouts into pinned per-token arrays.
 *
 * Replaces the per-token Python loop of build_train_batch
 * (/root/reference/pkg/src/asyncrl/trainer.py:83-111): trajectories, in formation
 * order (controller.form_batch, controller.py:184-202), are flattened into
 *   tokens int64 [T], behaviour log-probs float64 [T], per-token versions int32 [T]
 *   (rollout.py:50-53, 159 — the reference drops them; the staleness mask needs
 *   them), traj_bounds int64 [n+1] (= cu_seqlens, trainer.py:101) and rewards
 *   float64 [n] (trainer.py:116-118 reads traj.reward.reward).
 * An unrewarded trajectory raises ValueError with the reference's message
 * (trainer.py:93-94); a behaviour / version list whose length differs from the
 * token list is an error too (the reference would silently misalign them).
 *
 * The destination buffers are caller-owned (pinned torch tensors) and passed as
 * integer addresses, so the packed arrays go host -> device in one DMA each.
 * CPython C API, no torch / numpy dependency.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

static PyObject* get_list(PyObject* traj, const char* name) {
  PyObject* o = PyObject_GetAttrString(traj, name);
  if (!o) return NULL;
  if (o == Py_None) return o;
  PyObject* f = PySequence_Fast(o, "expected a sequence");
  Py_DECREF(o);
  return f;
}

/* count(trajectories) -> (n_tokens, n_traj) */
static PyObject* packer_count(PyObject* self, PyObject* args) {
  PyObject* trajs;
  if (!PyArg_ParseTuple(args, "O", &trajs)) return NULL;
  PyObject* seq = PySequence_Fast(trajs, "trajectories must be a sequence");
  if (!seq) return NULL;
  Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  long long total = 0;
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* toks = get_list(PySequence_Fast_GET_ITEM(seq, k), "tokens");
    if (!toks) {
      Py_DECREF(seq);
      return NULL;
    }
    if (toks != Py_None) total += PySequence_Fast_GET_SIZE(toks);
    Py_DECREF(toks);
  }
  Py_DECREF(seq);
  return Py_BuildValue("(Ln)", total, n);
}

static int fill_i64(PyObject* lst, int64_t* dst) {
  Py_ssize_t m = PySequence_Fast_GET_SIZE(lst);
  PyObject** it = PySequence_Fast_ITEMS(lst);
  for (Py_ssize_t i = 0; i < m; ++i) {
    long long v = PyLong_AsLongLong(it[i]);
    if (v == -1 && PyErr_Occurred()) return -1;
    dst[i] = (int64_t)v;
  }
  return 0;
}
static int fill_i32(PyObject* lst, int32_t* dst) {
  Py_ssize_t m = PySequence_Fast_GET_SIZE(lst);
  PyObject** it = PySequence_Fast_ITEMS(lst);
  for (Py_ssize_t i = 0; i < m; ++i) {
    long v = PyLong_AsLong(it[i]);
    if (v == -1 && PyErr_Occurred()) return -1;
    dst[i] = (int32_t)v;
  }
  return 0;
}
static int fill_f64(PyObject* lst, double* dst) {
  Py_ssize_t m = PySequence_Fast_GET_SIZE(lst);
  PyObject** it = PySequence_Fast_ITEMS(lst);
  for (Py_ssize_t i = 0; i < m; ++i) {
    PyObject* o = it[i];
    double v = PyFloat_CheckExact(o) ? PyFloat_AS_DOUBLE(o) : PyFloat_AsDouble(o);
    if (v == -1.0 && PyErr_Occurred()) return -1;
    dst[i] = v;
  }
  return 0;
}

/* fill(trajectories, tokens_addr, behav_addr, versions_addr (0 = skip), bounds_addr,
 *      rewards_addr, capacity) -> have_versions (bool) */
static PyObject* packer_fill(PyObject* self, PyObject* args) {
  PyObject* trajs;
  unsigned long long a_tok, a_beh, a_ver, a_bnd, a_rew;
  long long capacity;
  if (!PyArg_ParseTuple(args, "OKKKKKL", &trajs, &a_tok, &a_beh, &a_ver, &a_bnd, &a_rew, &capacity))
    return NULL;
  int64_t* tok = (int64_t*)(uintptr_t)a_tok;
  double* beh = (double*)(uintptr_t)a_beh;
  int32_t* ver = (int32_t*)(uintptr_t)a_ver;
  int64_t* bnd = (int64_t*)(uintptr_t)a_bnd;
  double* rew = (double*)(uintptr_t)a_rew;
  PyObject* seq = PySequence_Fast(trajs, "trajectories must be a sequence");
  if (!seq) return NULL;
  Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  int64_t pos = 0;
  int have_versions = 1;
  bnd[0] = 0;
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* traj = PySequence_Fast_GET_ITEM(seq, k);
    PyObject *r = NULL, *toks = NULL, *beh_l = NULL, *ver_l = NULL;
    r = PyObject_GetAttrString(traj, "reward");
    if (!r) goto fail;
    if (r == Py_None) {  /* trainer.py:93-94 */
      PyObject* tid = PyObject_GetAttrString(traj, "trajectory_id");
      if (tid) {
        PyErr_Format(PyExc_ValueError, "trajectory %S is unrewarded", tid);
        Py_DECREF(tid);
      }
      goto fail;
    }
    {
      PyObject* rv = PyObject_GetAttrString(r, "reward");  /* RewardResult.reward */
      if (!rv) goto fail;
      rew[k] = PyFloat_AsDouble(rv);
      Py_DECREF(rv);
      if (rew[k] == -1.0 && PyErr_Occurred()) goto fail;
    }
    toks = get_list(traj, "tokens");
    if (!toks) goto fail;
    beh_l = get_list(traj, "behavior_logprobs");
    if (!beh_l) goto fail;
    {
      const Py_ssize_t m = toks == Py_None ? 0 : PySequence_Fast_GET_SIZE(toks);
      if (pos + m > capacity) {
        PyErr_SetString(PyExc_ValueError, "packed tokens exceed the destination capacity");
        goto fail;
      }
      if (m > 0) {
        if (beh_l == Py_None || PySequence_Fast_GET_SIZE(beh_l) != m) {
          PyErr_Format(PyExc_ValueError,
                       "trajectory %zd: behavior_logprobs length differs from tokens", k);
          goto fail;
        }
        if (fill_i64(toks, tok + pos) || fill_f64(beh_l, beh + pos)) goto fail;
      }
      if (ver && have_versions) {
        ver_l = PyObject_HasAttrString(traj, "versions") ? get_list(traj, "versions") : (Py_INCREF(Py_None), Py_None);
        if (!ver_l) goto fail;
        if (ver_l == Py_None || PySequence_Fast_GET_SIZE(ver_l) != m) have_versions = 0;
        else if (m > 0 && fill_i32(ver_l, ver + pos)) goto fail;
      }
      pos += m;
      bnd[k + 1] = pos;
    }
    Py_XDECREF(r);
    Py_XDECREF(toks);
    Py_XDECREF(beh_l);
    Py_XDECREF(ver_l);
    continue;
  fail:
    Py_XDECREF(r);
    Py_XDECREF(toks);
    Py_XDECREF(beh_l);
    Py_XDECREF(ver_l);
    Py_DECREF(seq);
    return NULL;
  }
  Py_DECREF(seq);
  return PyBool_FromLong(ver ? have_versions : 0);
}

static PyMethodDef methods[] = {
    {"count", packer_count, METH_VARARGS, "count(trajectories) -> (n_tokens, n_traj)"},
    {"fill", packer_fill, METH_VARARGS,
     "fill(trajectories, tokens_addr, behav_addr, versions_addr, bounds_addr, rewards_addr, "
     "capacity) -> have_versions"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_packer",
                                    "Native rollout packer (build_train_batch, trainer.py:83-111)",
                                    -1, methods};

PyMODINIT_FUNC PyInit__packer(void) { return PyModule_Create(&moddef); }
