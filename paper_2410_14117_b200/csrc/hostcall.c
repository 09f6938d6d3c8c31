/* hostcall.c -- CPython fast path for the host-ABI step (B200EnvBatch.step).
 *
 * The per-step cost of the ctypes call (11 argument conversions, a ctypes
 * object for the action pointer, the error check) is ~2.5 us of a ~27 us C2
 * step; this METH_FASTCALL function reads the action array through the buffer
 * protocol and calls uuvsim_step_ex (include/uuvsim.h) through a function
 * pointer handed over once by bind().  Binding glue only: the compute path is
 * the same C ABI call.  Like ctypes, it releases the GIL for the call.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

typedef int32_t (*step_ex_fn)(uint64_t, const double*, uint64_t, double*, uint64_t, double*,
                              uint64_t, uint8_t*, uint64_t, int8_t*, uint64_t);

static step_ex_fn g_step_ex = NULL;

/* bind(address of uuvsim_step_ex) */
static PyObject* hc_bind(PyObject* self, PyObject* arg) {
    void* p = PyLong_AsVoidPtr(arg);
    if (!p && PyErr_Occurred()) return NULL;
    g_step_ex = (step_ex_fn)p;
    Py_RETURN_NONE;
}

/* step_ex(handle, actions, n_env, act_dim, ptrs) -> C ABI return code, or -100 when
 * the actions are not a C-contiguous float64 [n_env, act_dim] buffer (the caller
 * then takes the general path).  ptrs = (obs, obs_len, rew, rew_len, done,
 * done_len, reason, reason_len) as integers. */
static PyObject* hc_step_ex(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
    if (nargs != 5 || !g_step_ex) {
        PyErr_SetString(PyExc_TypeError, "step_ex(handle, actions, n_env, act_dim, ptrs)");
        return NULL;
    }
    const unsigned long long h = PyLong_AsUnsignedLongLong(args[0]);
    const Py_ssize_t n = PyLong_AsSsize_t(args[2]);
    const Py_ssize_t a = PyLong_AsSsize_t(args[3]);
    if (PyErr_Occurred()) return NULL;
    PyObject* ptrs = args[4];
    if (!PyTuple_Check(ptrs) || PyTuple_GET_SIZE(ptrs) != 8) {
        PyErr_SetString(PyExc_TypeError, "ptrs must be an 8-tuple");
        return NULL;
    }
    unsigned long long p[8];
    for (int i = 0; i < 8; ++i) {
        p[i] = PyLong_AsUnsignedLongLong(PyTuple_GET_ITEM(ptrs, i));
        if (PyErr_Occurred()) return NULL;
    }
    Py_buffer v;
    if (PyObject_GetBuffer(args[1], &v, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT | PyBUF_ND) != 0) {
        PyErr_Clear();
        return PyLong_FromLong(-100);
    }
    const char* f = v.format ? v.format : "B";
    if (f[0] == '<' || f[0] == '=' || f[0] == '@') ++f;
    if (strcmp(f, "d") != 0 || v.itemsize != 8 || v.ndim != 2 || v.shape[0] != n ||
        v.shape[1] != a) {
        PyBuffer_Release(&v);
        return PyLong_FromLong(-100);
    }
    int32_t rc;
    Py_BEGIN_ALLOW_THREADS
    rc = g_step_ex((uint64_t)h, (const double*)v.buf, (uint64_t)(n * a), (double*)(uintptr_t)p[0],
                   (uint64_t)p[1], (double*)(uintptr_t)p[2], (uint64_t)p[3],
                   (uint8_t*)(uintptr_t)p[4], (uint64_t)p[5], (int8_t*)(uintptr_t)p[6],
                   (uint64_t)p[7]);
    Py_END_ALLOW_THREADS
    PyBuffer_Release(&v);
    return PyLong_FromLong(rc);
}

static PyMethodDef hc_methods[] = {
    {"bind", (PyCFunction)hc_bind, METH_O, "bind(address of uuvsim_step_ex)"},
    {"step_ex", (PyCFunction)(void (*)(void))hc_step_ex, METH_FASTCALL,
     "step_ex(handle, actions, n_env, act_dim, ptrs) -> code (-100: use the general path)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef hc_module = {PyModuleDef_HEAD_INIT, "_hostcall", NULL, -1, hc_methods};

PyMODINIT_FUNC PyInit__hostcall(void) { return PyModule_Create(&hc_module); }
