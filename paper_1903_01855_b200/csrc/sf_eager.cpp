// sf_eager.cpp — _sfeager, the native eager front-end (CPython extension).
//
// The reference's eager path is Python from the operator to the numpy call:
// wrapper -> dispatch (registry lookup, attr canonicalisation) ->
// _dispatch_eager (input checks, placement, KernelEnv, kernel, stats, tape
// notification), stageflow/ops.py:294-362 and :370-485 — about 13 us per op.
// This module does the same work in C for the cases that dominate eager
// programs: built-in / plugin elementwise ops, tiny matmuls, transposes,
// identity, reshape and broadcast_to on tensors of a single-device runtime
// outside any trace.  It checks dtypes and shapes, computes the broadcast
// geometry, hands one compact descriptor to the device's launch queue
// (sf_queue_push, csrc/sf_queue.cu), builds the output Tensor directly, and
// counts the dispatch.  Everything else — traces, device scopes, several
// devices, Variables, user kernels, and every error — goes to the Python
// dispatcher (ops._dispatch_py), which is the reference semantics verbatim;
// an op taking the fast path is bit-identical to the same op through Python
// because both end in the same native launch.  Active tapes are notified
// through the Python tape code (ops._notify_tapes) with the same arguments.
//
// It also defines the storage types the front-end builds on:
//   DeviceBuffer — one caching-allocator block (freed with sf_free on
//                  dealloc, no ctypes round trip);
//   TensorBase   — the slot layout of paper_1903_01855_b200.tensor.Tensor
//                  and its arithmetic operators (reference: ops.py:456-485).
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

#include <cstdint>
#include <cstring>

#include "../../include/sfb200.h"

namespace {

// ---------------------------------------------------------------- strings
PyObject* s_owner;
PyObject* s_context;
PyObject* s_runtime;
PyObject* s_device_buffer;
PyObject* s_ptr;
PyObject* s_reshape;
PyObject* s_shape;

// ------------------------------------------------------------ DeviceBuffer

struct DevBuf {
  PyObject_HEAD
  int dev;
  unsigned long long ptr;
  Py_ssize_t nbytes;
  PyObject* weakreflist;
};

void DevBuf_dealloc(PyObject* o) {
  DevBuf* self = (DevBuf*)o;
  if (self->weakreflist) PyObject_ClearWeakRefs(o);
  if (self->ptr) {
    sf_free(self->dev, (void*)(uintptr_t)self->ptr);
    self->ptr = 0;
  }
  Py_TYPE(o)->tp_free(o);
}

int DevBuf_init(PyObject* o, PyObject* args, PyObject* kw) {
  DevBuf* self = (DevBuf*)o;
  static const char* kwl[] = {"dev", "ptr", "nbytes", nullptr};
  int dev = 0;
  PyObject* pobj = nullptr;
  Py_ssize_t nbytes = 0;
  if (!PyArg_ParseTupleAndKeywords(args, kw, "iOn", (char**)kwl, &dev, &pobj, &nbytes)) return -1;
  unsigned long long ptr = 0;
  if (pobj != Py_None) {
    ptr = PyLong_AsUnsignedLongLong(pobj);
    if (PyErr_Occurred()) return -1;
  }
  self->dev = dev;
  self->ptr = ptr;
  self->nbytes = nbytes;
  return 0;
}

PyMemberDef DevBuf_members[] = {
    {"dev", T_INT, offsetof(DevBuf, dev), 0, "device ordinal"},
    {"ptr", T_ULONGLONG, offsetof(DevBuf, ptr), 0, "device address (0 once released)"},
    {"nbytes", T_PYSSIZET, offsetof(DevBuf, nbytes), 0, "requested size in bytes"},
    {nullptr}};

PyTypeObject DevBufType = {PyVarObject_HEAD_INIT(nullptr, 0)};

PyObject* new_devbuf(int dev, void* ptr, Py_ssize_t nbytes) {
  DevBuf* b = PyObject_New(DevBuf, &DevBufType);
  if (!b) {
    sf_free(dev, ptr);
    return nullptr;
  }
  b->dev = dev;
  b->ptr = (unsigned long long)(uintptr_t)ptr;
  b->nbytes = nbytes;
  b->weakreflist = nullptr;
  return (PyObject*)b;
}

// -------------------------------------------------------------- TensorBase

struct TensorObj {
  PyObject_HEAD
  PyObject* dtype;
  PyObject* shape;
  PyObject* device;
  PyObject* buf;
  PyObject* host;
  PyObject* symbolic;
  PyObject* born_trace;
  PyObject* sib;
  PyObject* pend;
  PyObject* weakreflist;
};

int Tensor_traverse(PyObject* o, visitproc visit, void* arg) {
  TensorObj* t = (TensorObj*)o;
  Py_VISIT(Py_TYPE(o));
  Py_VISIT(t->dtype);
  Py_VISIT(t->shape);
  Py_VISIT(t->device);
  Py_VISIT(t->buf);
  Py_VISIT(t->host);
  Py_VISIT(t->symbolic);
  Py_VISIT(t->born_trace);
  Py_VISIT(t->sib);
  Py_VISIT(t->pend);
  return 0;
}

int Tensor_clear(PyObject* o) {
  TensorObj* t = (TensorObj*)o;
  Py_CLEAR(t->dtype);
  Py_CLEAR(t->shape);
  Py_CLEAR(t->device);
  Py_CLEAR(t->buf);
  Py_CLEAR(t->host);
  Py_CLEAR(t->symbolic);
  Py_CLEAR(t->born_trace);
  Py_CLEAR(t->sib);
  Py_CLEAR(t->pend);
  return 0;
}

void Tensor_dealloc(PyObject* o) {
  PyObject_GC_UnTrack(o);
  TensorObj* t = (TensorObj*)o;
  if (t->weakreflist) PyObject_ClearWeakRefs(o);
  Tensor_clear(o);
  // (a heap subtype's reference is dropped by subtype_dealloc)
  Py_TYPE(o)->tp_free(o);
}

PyMemberDef Tensor_members[] = {
    {"dtype", T_OBJECT, offsetof(TensorObj, dtype), 0, nullptr},
    {"shape", T_OBJECT, offsetof(TensorObj, shape), 0, nullptr},
    {"device", T_OBJECT, offsetof(TensorObj, device), 0, nullptr},
    {"_buf", T_OBJECT, offsetof(TensorObj, buf), 0, nullptr},
    {"_host", T_OBJECT, offsetof(TensorObj, host), 0, nullptr},
    {"_symbolic", T_OBJECT, offsetof(TensorObj, symbolic), 0, nullptr},
    {"_born_trace", T_OBJECT, offsetof(TensorObj, born_trace), 0, nullptr},
    {"_sib", T_OBJECT, offsetof(TensorObj, sib), 0, nullptr},
    {"_pend", T_OBJECT, offsetof(TensorObj, pend), 0, nullptr},
    {nullptr}};

PyTypeObject TensorBaseType = {PyVarObject_HEAD_INIT(nullptr, 0)};

inline bool is_tensor(PyObject* o) { return PyObject_TypeCheck(o, &TensorBaseType); }

// ------------------------------------------------------------ configuration

enum Kind { K_EW1 = 1, K_EW2 = 2, K_MATMUL = 3, K_TRANSPOSE = 4, K_IDENTITY = 5,
            K_RESHAPE = 6, K_BROADCAST_TO = 7 };
enum Flags { F_FLOATS_ONLY = 1, F_OUT_BOOL = 2 };

struct FastOp {
  PyObject* opdef = nullptr;  // the registered OpDef (strong)
  PyObject* name = nullptr;
  int kind = 0, opcode = 0, flags = 0;
  unsigned long long count = 0;
};

constexpr int kMaxFast = 128;
FastOp g_ops[kMaxFast];
int g_nops = 0;
PyObject* g_table = nullptr;  // name -> index

// runtime the table was built for (strong ref); the module dict of
// paper_1903_01855_b200.runtime (to read `_runtime`) and its thread-local
PyObject* g_rt = nullptr;
PyObject* g_registry = nullptr;
PyObject* g_rt_dict = nullptr;
PyObject* g_local = nullptr;
bool g_single = false;      // runtime has one device
int g_ordinal = 0;
PyObject* g_device = nullptr;  // that device's DeviceName
PyTypeObject* g_tensor_type = nullptr;  // paper_1903_01855_b200.tensor.Tensor
PyObject* g_dtypes[5] = {};  // DType members by wire tag (1..4)
int g_width[5] = {0, 4, 8, 4, 1};
Py_ssize_t off_traces = -1, off_tapes = -1, off_scopes = -1;

// Python callables
PyObject* g_slow_dispatch = nullptr;  // ops._dispatch_py(op, inputs, attrs)
PyObject* g_notify = nullptr;         // ops._notify_tapes(op_def, inputs, outputs, attrs, ctx)
PyObject* g_configure = nullptr;      // _fastpath.configure(runtime)
PyObject* g_kernel_error = nullptr;   // errors.KernelError

bool g_enabled = true;

int tag_of(PyObject* dtype) {
  for (int i = 1; i <= 4; ++i)
    if (g_dtypes[i] == dtype) return i;
  return 0;
}

Py_ssize_t slot_offset(PyObject* type, const char* name) {
  PyObject* d = PyObject_GetAttrString(type, name);
  if (!d) return -1;
  Py_ssize_t off = -1;
  if (Py_IS_TYPE(d, &PyMemberDescr_Type)) off = ((PyMemberDescrObject*)d)->d_member->offset;
  Py_DECREF(d);
  if (off < 0) PyErr_Format(PyExc_TypeError, "%s is not a slot", name);
  return off;
}

// The live ExecutionContext if the fast path may run (borrowed pointer in
// *ctx, kept alive by the thread-local), else nullptr with no error set.
// Fast: the runtime the table was built for, a context of that runtime,
// no open trace, no device scope, one device.
PyObject* fast_context() {
  if (!g_enabled || !g_rt_dict) return nullptr;
  PyObject* rt = PyDict_GetItemWithError(g_rt_dict, s_runtime);  // borrowed
  if (!rt) {
    PyErr_Clear();
    return nullptr;
  }
  if (rt != g_rt) {
    if (rt == Py_None || !g_configure) return nullptr;
    PyObject* r = PyObject_CallOneArg(g_configure, rt);
    if (!r) {
      PyErr_Clear();
      return nullptr;
    }
    Py_DECREF(r);
    if (rt != g_rt) return nullptr;
  }
  if (!g_single || !g_table) return nullptr;
  PyObject* owner = PyObject_GetAttr(g_local, s_owner);
  if (!owner) {
    PyErr_Clear();
    return nullptr;
  }
  Py_DECREF(owner);  // the thread-local keeps it alive
  if (owner != rt) return nullptr;
  PyObject* ctx = PyObject_GetAttr(g_local, s_context);
  if (!ctx) {
    PyErr_Clear();
    return nullptr;
  }
  Py_DECREF(ctx);
  PyObject* traces = *(PyObject**)((char*)ctx + off_traces);
  PyObject* scopes = *(PyObject**)((char*)ctx + off_scopes);
  if (!traces || !scopes || !PyList_CheckExact(traces) || !PyList_CheckExact(scopes)) return nullptr;
  if (PyList_GET_SIZE(traces) || PyList_GET_SIZE(scopes)) return nullptr;
  return ctx;
}

bool tapes_active(PyObject* ctx) {
  PyObject* tapes = *(PyObject**)((char*)ctx + off_tapes);
  return tapes && (!PyList_CheckExact(tapes) || PyList_GET_SIZE(tapes) > 0);
}

// ---------------------------------------------------------------- operands

struct Operand {
  const void* ptr = nullptr;
  double imm = 0.0;
};

bool shape_dims(PyObject* shape, long long* dims, int* nd, long long* numel) {
  if (!PyTuple_CheckExact(shape)) return false;
  const Py_ssize_t n = PyTuple_GET_SIZE(shape);
  if (n > SF_MAX_DIMS) return false;
  long long c = 1;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* v = PyTuple_GET_ITEM(shape, i);
    if (!PyLong_CheckExact(v)) return false;
    const long long d = PyLong_AsLongLong(v);
    if (d < 0) {
      PyErr_Clear();
      return false;
    }
    dims[i] = d;
    c *= d;
  }
  *nd = (int)n;
  *numel = c;
  return true;
}

// Read a one-element host array through the buffer protocol.
bool host_scalar(PyObject* host, int tag, double* out) {
  Py_buffer view;
  if (PyObject_GetBuffer(host, &view, PyBUF_SIMPLE) != 0) {
    PyErr_Clear();
    return false;
  }
  bool ok = view.len == g_width[tag];
  if (ok) {
    switch (tag) {
      case SF_DTYPE_F32: { float v; std::memcpy(&v, view.buf, 4); *out = v; break; }
      case SF_DTYPE_F64: { double v; std::memcpy(&v, view.buf, 8); *out = v; break; }
      case SF_DTYPE_I32: { int32_t v; std::memcpy(&v, view.buf, 4); *out = v; break; }
      default: { unsigned char v; std::memcpy(&v, view.buf, 1); *out = v ? 1.0 : 0.0; break; }
    }
  }
  PyBuffer_Release(&view);
  return ok;
}

// Device pointer of a concrete tensor (uploading host bytes on demand).
// Returns false with a Python error set on failure.
bool device_ptr(TensorObj* t, const void** ptr) {
  PyObject* buf = t->buf;
  if (!buf || buf == Py_None) {
    PyObject* r = PyObject_CallMethodNoArgs((PyObject*)t, s_device_buffer);
    if (!r) return false;
    Py_DECREF(r);
    buf = t->buf;
    if (!buf || buf == Py_None) {
      PyErr_SetString(PyExc_RuntimeError, "tensor has no device buffer");
      return false;
    }
  }
  if (Py_IS_TYPE(buf, &DevBufType)) {
    *ptr = (const void*)(uintptr_t)((DevBuf*)buf)->ptr;
    return true;
  }
  PyObject* p = PyObject_GetAttr(buf, s_ptr);
  if (!p) return false;
  *ptr = PyLong_AsVoidPtr(p);
  Py_DECREF(p);
  return !PyErr_Occurred();
}

// An elementwise operand: a one-element host value travels as an immediate
// (Tensor._imm), anything else by device pointer.
bool ew_operand(TensorObj* t, int tag, long long numel, Operand* o) {
  if (numel == 1 && t->host && t->host != Py_None && host_scalar(t->host, tag, &o->imm)) {
    o->ptr = nullptr;
    return true;
  }
  return device_ptr(t, &o->ptr);
}

inline bool concrete(PyObject* x) {
  TensorObj* t = (TensorObj*)x;
  return !t->symbolic || t->symbolic == Py_None;
}

// ------------------------------------------------------------- launching

PyObject* kernel_error(const char* what) {
  const char* msg = sf_last_error();
  PyErr_Format(g_kernel_error, "%s: %s", what, msg ? msg : "?");
  return nullptr;
}

PyObject* new_tensor(PyObject* dtype, PyObject* shape, PyObject* buf, PyObject* host) {
  TensorObj* t = (TensorObj*)g_tensor_type->tp_alloc(g_tensor_type, 0);
  if (!t) return nullptr;
  t->dtype = Py_NewRef(dtype);
  t->shape = Py_NewRef(shape);
  t->device = Py_NewRef(g_device);
  t->buf = Py_NewRef(buf ? buf : Py_None);
  t->host = Py_NewRef(host ? host : Py_None);
  t->symbolic = Py_NewRef(Py_None);
  t->born_trace = Py_NewRef(Py_None);
  t->sib = Py_NewRef(Py_None);
  t->pend = Py_NewRef(Py_None);
  return (PyObject*)t;
}

PyObject* push(const sf_op_desc& d, int out_tag, PyObject* out_shape, long long numel,
               const char* what) {
  void* out = nullptr;
  int st;
  Py_BEGIN_ALLOW_THREADS
  st = sf_queue_push(g_ordinal, &d, &out);
  Py_END_ALLOW_THREADS
  if (st != SF_OK) return kernel_error(what);
  PyObject* buf = new_devbuf(g_ordinal, out, (Py_ssize_t)(numel * g_width[out_tag]));
  if (!buf) return nullptr;
  PyObject* t = new_tensor(g_dtypes[out_tag], out_shape, buf, nullptr);
  Py_DECREF(buf);
  return t;
}

void contiguous_strides(const long long* dims, int nd, long long* st) {
  long long acc = 1;
  for (int i = nd - 1; i >= 0; --i) {
    st[i] = acc;
    acc *= dims[i];
  }
}

// Operand strides against an output of rank `ond` (right-aligned, 0 on
// broadcast dims).
void bcast_strides(const long long* dims, int nd, int ond, int64_t* out) {
  long long cs[SF_MAX_DIMS];
  contiguous_strides(dims, nd, cs);
  const int pad = ond - nd;
  for (int i = 0; i < ond; ++i) out[i] = 0;
  for (int i = 0; i < nd; ++i) out[pad + i] = dims[i] == 1 ? 0 : cs[i];
}

PyObject* make_shape(const long long* dims, int nd) {
  PyObject* t = PyTuple_New(nd);
  if (!t) return nullptr;
  for (int i = 0; i < nd; ++i) {
    PyObject* v = PyLong_FromLongLong(dims[i]);
    if (!v) {
      Py_DECREF(t);
      return nullptr;
    }
    PyTuple_SET_ITEM(t, i, v);
  }
  return t;
}

#define NOT_FAST ((PyObject*)1)  // "use the Python path" (no error set)

// binary elementwise with immediates for scalar operands (sa/sb: operand
// is a scalar already converted to the other operand's dtype)
PyObject* run_ew2(const FastOp& f, PyObject* a, PyObject* b, const double* sa, const double* sb) {
  TensorObj* ta = sa ? nullptr : (TensorObj*)a;
  TensorObj* tb = sb ? nullptr : (TensorObj*)b;
  TensorObj* like = ta ? ta : tb;
  const int tag = tag_of(like->dtype);
  if (!tag || tag == SF_DTYPE_BOOL) return NOT_FAST;
  if (ta && tb && ta->dtype != tb->dtype) return NOT_FAST;
  if ((f.flags & F_FLOATS_ONLY) && tag != SF_DTYPE_F32 && tag != SF_DTYPE_F64) return NOT_FAST;
  long long da[SF_MAX_DIMS], db[SF_MAX_DIMS], dout[SF_MAX_DIMS];
  int na = 0, nb = 0;
  long long ca = 1, cb = 1;
  if (ta && !shape_dims(ta->shape, da, &na, &ca)) return NOT_FAST;
  if (tb && !shape_dims(tb->shape, db, &nb, &cb)) return NOT_FAST;
  const int nd = na > nb ? na : nb;
  for (int i = 0; i < nd; ++i) {
    const int ia = i - (nd - na), ib = i - (nd - nb);
    const long long x = ia >= 0 ? da[ia] : 1, y = ib >= 0 ? db[ib] : 1;
    if (x == y || y == 1) dout[i] = x;
    else if (x == 1) dout[i] = y;
    else return NOT_FAST;  // the Python path raises the broadcast error
  }
  long long numel = 1;
  for (int i = 0; i < nd; ++i) numel *= dout[i];
  // reuse an operand's shape tuple when it is the output shape
  PyObject* oshape = nullptr;
  if (ta && na == nd && ca == numel) oshape = Py_NewRef(ta->shape);
  else if (tb && nb == nd && cb == numel) oshape = Py_NewRef(tb->shape);
  else oshape = make_shape(dout, nd);
  if (!oshape) return nullptr;
  sf_op_desc d;
  std::memset(&d, 0, sizeof(d));
  d.kind = SF_QOP_EW;
  d.op = f.opcode;
  d.dtype = tag;
  d.ndim = nd;
  d.n_in = 2;
  for (int i = 0; i < nd; ++i) d.shape[i] = dout[i];
  Operand oa, ob;
  bool ok = true;
  if (ta) {
    ok = ew_operand(ta, tag, ca, &oa);
    if (ok && oa.ptr) bcast_strides(da, na, nd, d.strides[0]);
  } else {
    oa.imm = *sa;
  }
  if (ok && tb) {
    ok = ew_operand(tb, tag, cb, &ob);
    if (ok && ob.ptr) bcast_strides(db, nb, nd, d.strides[1]);
  } else if (ok) {
    ob.imm = *sb;
  }
  if (!ok) {
    Py_DECREF(oshape);
    return nullptr;
  }
  d.in[0] = oa.ptr;
  d.imm[0] = oa.imm;
  d.in[1] = ob.ptr;
  d.imm[1] = ob.imm;
  PyObject* r = push(d, (f.flags & F_OUT_BOOL) ? SF_DTYPE_BOOL : tag, oshape, numel, "elementwise");
  Py_DECREF(oshape);
  return r;
}

PyObject* run_ew1(const FastOp& f, TensorObj* x) {
  const int tag = tag_of(x->dtype);
  if (!tag || tag == SF_DTYPE_BOOL) return NOT_FAST;
  if ((f.flags & F_FLOATS_ONLY) && tag != SF_DTYPE_F32 && tag != SF_DTYPE_F64) return NOT_FAST;
  long long dx[SF_MAX_DIMS];
  int nx;
  long long numel;
  if (!shape_dims(x->shape, dx, &nx, &numel)) return NOT_FAST;
  sf_op_desc d;
  std::memset(&d, 0, sizeof(d));
  d.kind = SF_QOP_EW;
  d.op = f.opcode;
  d.dtype = tag;
  d.ndim = nx;
  d.n_in = 1;
  for (int i = 0; i < nx; ++i) d.shape[i] = dx[i];
  Operand o;
  if (!ew_operand(x, tag, numel, &o)) return nullptr;
  if (o.ptr) contiguous_strides(dx, nx, (long long*)d.strides[0]);
  d.in[0] = o.ptr;
  d.imm[0] = o.imm;
  return push(d, (f.flags & F_OUT_BOOL) ? SF_DTYPE_BOOL : tag, x->shape, numel, "elementwise");
}

PyObject* run_matmul(TensorObj* a, TensorObj* b) {
  const int tag = tag_of(a->dtype);
  if (a->dtype != b->dtype || (tag != SF_DTYPE_F32 && tag != SF_DTYPE_F64)) return NOT_FAST;
  long long da[SF_MAX_DIMS], db[SF_MAX_DIMS];
  int na, nb;
  long long ca, cb;
  if (!shape_dims(a->shape, da, &na, &ca) || !shape_dims(b->shape, db, &nb, &cb)) return NOT_FAST;
  if (na != 2 || nb != 2 || da[1] != db[0]) return NOT_FAST;
  sf_op_desc d;
  std::memset(&d, 0, sizeof(d));
  d.kind = SF_QOP_MATMUL;
  d.dtype = tag;
  d.n_in = 2;
  d.m = da[0];
  d.k = da[1];
  d.n = db[1];
  if (!device_ptr(a, &d.in[0]) || !device_ptr(b, &d.in[1])) return nullptr;
  long long dims[2] = {da[0], db[1]};
  PyObject* oshape = make_shape(dims, 2);
  if (!oshape) return nullptr;
  PyObject* r = push(d, tag, oshape, da[0] * db[1], "matmul");
  Py_DECREF(oshape);
  return r;
}

PyObject* run_transpose(TensorObj* x) {
  const int tag = tag_of(x->dtype);
  if (!tag) return NOT_FAST;
  long long dx[SF_MAX_DIMS];
  int nx;
  long long numel;
  if (!shape_dims(x->shape, dx, &nx, &numel) || nx != 2) return NOT_FAST;
  const void* src;
  if (!device_ptr(x, &src)) return nullptr;
  void* out = nullptr;
  int st;
  Py_BEGIN_ALLOW_THREADS
  st = sf_transpose2d(g_ordinal, tag, dx[0], dx[1], src, &out);
  Py_END_ALLOW_THREADS
  if (st != SF_OK) return kernel_error("transpose");
  long long dims[2] = {dx[1], dx[0]};
  PyObject* oshape = make_shape(dims, 2);
  if (!oshape) {
    sf_free(g_ordinal, out);
    return nullptr;
  }
  PyObject* buf = new_devbuf(g_ordinal, out, (Py_ssize_t)(numel * g_width[tag]));
  PyObject* r = buf ? new_tensor(x->dtype, oshape, buf, nullptr) : nullptr;
  Py_XDECREF(buf);
  Py_DECREF(oshape);
  return r;
}

// attrs {"shape": seq of non-negative ints} -> a new tuple (or NOT_FAST)
PyObject* shape_attr(PyObject* attrs) {
  if (!attrs || !PyDict_CheckExact(attrs) || PyDict_GET_SIZE(attrs) != 1) return NOT_FAST;
  PyObject* v = PyDict_GetItemWithError(attrs, s_shape);
  if (!v) {
    PyErr_Clear();
    return NOT_FAST;
  }
  PyObject* tup;
  if (PyTuple_CheckExact(v)) tup = Py_NewRef(v);
  else if (PyList_CheckExact(v)) tup = PyList_AsTuple(v);
  else return NOT_FAST;
  if (!tup) return nullptr;
  const Py_ssize_t n = PyTuple_GET_SIZE(tup);
  bool ok = n <= SF_MAX_DIMS;
  for (Py_ssize_t i = 0; ok && i < n; ++i) {
    PyObject* d = PyTuple_GET_ITEM(tup, i);
    ok = PyLong_CheckExact(d) && PyLong_AsLongLong(d) >= 0;
  }
  if (!ok) {
    PyErr_Clear();
    Py_DECREF(tup);
    return NOT_FAST;
  }
  return tup;
}

PyObject* run_reshape(TensorObj* x, PyObject* target) {
  long long dx[SF_MAX_DIMS], dt[SF_MAX_DIMS];
  int nx, nt;
  long long cx, ct;
  if (!shape_dims(x->shape, dx, &nx, &cx) || !shape_dims(target, dt, &nt, &ct) || cx != ct)
    return NOT_FAST;
  PyObject* host = nullptr;
  if (x->host && x->host != Py_None) {
    host = PyObject_CallMethodOneArg(x->host, s_reshape, target);
    if (!host) return nullptr;
  }
  PyObject* buf = x->buf && x->buf != Py_None ? x->buf : nullptr;
  if (!buf && !host) return NOT_FAST;
  PyObject* r = new_tensor(x->dtype, target, buf, host);
  Py_XDECREF(host);
  return r;
}

PyObject* run_broadcast_to(TensorObj* x, PyObject* target) {
  const int tag = tag_of(x->dtype);
  if (!tag) return NOT_FAST;
  long long dx[SF_MAX_DIMS], dt[SF_MAX_DIMS];
  int nx, nt;
  long long cx, ct;
  if (!shape_dims(x->shape, dx, &nx, &cx) || !shape_dims(target, dt, &nt, &ct)) return NOT_FAST;
  if (nx > nt) return NOT_FAST;
  for (int i = 0; i < nx; ++i) {
    const long long s = dx[nx - 1 - i], t = dt[nt - 1 - i];
    if (s != t && s != 1) return NOT_FAST;
  }
  sf_op_desc d;
  std::memset(&d, 0, sizeof(d));
  d.kind = SF_QOP_EW;
  d.op = 0;  // identity
  d.dtype = tag;
  d.ndim = nt;
  d.n_in = 1;
  for (int i = 0; i < nt; ++i) d.shape[i] = dt[i];
  Operand o;
  if (!ew_operand(x, tag, cx, &o)) return nullptr;
  if (o.ptr) bcast_strides(dx, nx, nt, d.strides[0]);
  d.in[0] = o.ptr;
  d.imm[0] = o.imm;
  return push(d, tag, target, ct, "elementwise");
}

// Run fast op `f` on tensor inputs (scalar immediates for EW2 in sa/sb).
PyObject* run_fast(const FastOp& f, PyObject* const* in, Py_ssize_t n, PyObject* attrs,
                   const double* sa, const double* sb, PyObject** canon_attrs) {
  switch (f.kind) {
    case K_EW1:
      if (n != 1 || attrs) return NOT_FAST;
      return run_ew1(f, (TensorObj*)in[0]);
    case K_EW2:
      if (n != 2 || attrs) return NOT_FAST;
      return run_ew2(f, in[0], in[1], sa, sb);
    case K_MATMUL:
      if (n != 2 || attrs) return NOT_FAST;
      return run_matmul((TensorObj*)in[0], (TensorObj*)in[1]);
    case K_TRANSPOSE:
      if (n != 1 || attrs) return NOT_FAST;
      return run_transpose((TensorObj*)in[0]);
    case K_IDENTITY: {
      if (n != 1 || attrs) return NOT_FAST;
      TensorObj* x = (TensorObj*)in[0];
      PyObject* buf = x->buf && x->buf != Py_None ? x->buf : nullptr;
      PyObject* host = x->host && x->host != Py_None ? x->host : nullptr;
      if (!buf && !host) return NOT_FAST;
      return new_tensor(x->dtype, x->shape, buf, host);
    }
    case K_RESHAPE:
    case K_BROADCAST_TO: {
      if (n != 1) return NOT_FAST;
      PyObject* target = shape_attr(attrs);
      if (target == NOT_FAST || !target) return target;
      PyObject* r = f.kind == K_RESHAPE ? run_reshape((TensorObj*)in[0], target)
                                        : run_broadcast_to((TensorObj*)in[0], target);
      if (r && r != NOT_FAST && canon_attrs) {
        *canon_attrs = PyDict_New();
        if (!*canon_attrs || PyDict_SetItem(*canon_attrs, s_shape, target) < 0) {
          Py_XDECREF(*canon_attrs);
          *canon_attrs = nullptr;
          Py_DECREF(r);
          r = nullptr;
        }
      }
      Py_DECREF(target);
      return r;
    }
    default:
      return NOT_FAST;
  }
}

// After a fast launch: count it and offer it to active tapes (Python).
bool finish(FastOp& f, PyObject* ctx, PyObject* const* in, Py_ssize_t n, PyObject* out,
            PyObject* canon_attrs) {
  f.count++;
  if (!tapes_active(ctx)) return true;
  PyObject* ins = PyList_New(n);
  if (!ins) return false;
  for (Py_ssize_t i = 0; i < n; ++i) PyList_SET_ITEM(ins, i, Py_NewRef(in[i]));
  PyObject* outs = PyList_New(1);
  if (!outs) {
    Py_DECREF(ins);
    return false;
  }
  PyList_SET_ITEM(outs, 0, Py_NewRef(out));
  PyObject* attrs = canon_attrs ? Py_NewRef(canon_attrs) : PyDict_New();
  PyObject* r = attrs ? PyObject_CallFunctionObjArgs(g_notify, f.opdef, ins, outs, attrs, ctx,
                                                     nullptr)
                      : nullptr;
  Py_XDECREF(attrs);
  Py_DECREF(ins);
  Py_DECREF(outs);
  if (!r) return false;
  Py_DECREF(r);
  return true;
}

FastOp* lookup(PyObject* name) {
  if (!g_table) return nullptr;
  PyObject* idx = PyDict_GetItemWithError(g_table, name);
  if (!idx) {
    PyErr_Clear();
    return nullptr;
  }
  const long i = PyLong_AsLong(idx);
  return (i >= 0 && i < g_nops) ? &g_ops[i] : nullptr;
}

// ------------------------------------------------------- module functions

// dispatch(op, inputs, attrs=None) -> list[Tensor]   (reference ops.py:294-305)
PyObject* py_dispatch(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs < 2 || nargs > 3) {
    PyErr_SetString(PyExc_TypeError, "dispatch(op, inputs, attrs=None)");
    return nullptr;
  }
  PyObject* name = args[0];
  PyObject* inputs = args[1];
  PyObject* attrs = nargs == 3 ? args[2] : Py_None;
  // (fast_context binds the table to the live runtime first)
  PyObject* ctx = fast_context();
  FastOp* f = ctx && PyUnicode_CheckExact(name) ? lookup(name) : nullptr;
  if (f && (PyList_CheckExact(inputs) || PyTuple_CheckExact(inputs))) {
    PyObject* attr_arg = nullptr;
    bool attrs_ok = true;
    if (attrs != Py_None) {
      if (!PyDict_CheckExact(attrs)) attrs_ok = false;
      else if (PyDict_GET_SIZE(attrs)) attr_arg = attrs;
    }
    PyObject* const* in = PySequence_Fast_ITEMS(inputs);
    const Py_ssize_t n = PySequence_Fast_GET_SIZE(inputs);
    bool tensors = n <= 3;
    for (Py_ssize_t i = 0; tensors && i < n; ++i)
      tensors = is_tensor(in[i]) && concrete(in[i]);
    if (attrs_ok && tensors) {
      PyObject* canon = nullptr;
      PyObject* holder[3];  // keep the inputs alive across Python callbacks
      for (Py_ssize_t i = 0; i < n; ++i) holder[i] = Py_NewRef(in[i]);
      PyObject* out = run_fast(*f, holder, n, attr_arg, nullptr, nullptr, &canon);
      PyObject* res = nullptr;
      if (out && out != NOT_FAST) {
        if (finish(*f, ctx, holder, n, out, canon)) {
          res = PyList_New(1);
          if (res) PyList_SET_ITEM(res, 0, out);
          else Py_DECREF(out);
        } else {
          Py_DECREF(out);
        }
      }
      Py_XDECREF(canon);
      for (Py_ssize_t i = 0; i < n; ++i) Py_DECREF(holder[i]);
      if (out != NOT_FAST) return res;
    }
    if (PyErr_Occurred()) return nullptr;
  }
  if (!g_slow_dispatch) {
    PyErr_SetString(PyExc_RuntimeError, "_sfeager: fast path not configured");
    return nullptr;
  }
  return PyObject_Vectorcall(g_slow_dispatch, args, nargs, nullptr);
}

// Python scalar -> immediate in `tag`'s dtype, exactly as
// np.asarray(x, dtype=like.dtype) would convert it; false = not handled.
bool scalar_imm(PyObject* x, int tag, double* out) {
  if (PyFloat_CheckExact(x)) {
    const double v = PyFloat_AS_DOUBLE(x);
    if (tag == SF_DTYPE_F32) {
      *out = (double)(float)v;
      return true;
    }
    if (tag == SF_DTYPE_F64) {
      *out = v;
      return true;
    }
    return false;
  }
  if (PyLong_CheckExact(x)) {
    int overflow = 0;
    const long long v = PyLong_AsLongLongAndOverflow(x, &overflow);
    if (overflow) return false;
    if (tag == SF_DTYPE_F32 && v >= -(1LL << 24) && v <= (1LL << 24)) {
      *out = (double)v;
      return true;
    }
    if (tag == SF_DTYPE_F64 && v >= -(1LL << 53) && v <= (1LL << 53)) {
      *out = (double)v;
      return true;
    }
    if (tag == SF_DTYPE_I32 && v >= INT32_MIN && v <= INT32_MAX) {
      *out = (double)v;
      return true;
    }
  }
  return false;
}

PyObject* g_host_scalar = nullptr;  // _fastpath.host_scalar(value, dtype) -> read-only 0-d array
PyObject* g_scalar_cache = nullptr;  // (tag, value) -> that array
PyObject* g_empty_shape = nullptr;

// A fresh 0-d constant tensor holding `scalar` in `tag`'s dtype (reference
// _as_operand -> tensor_from_host, ops.py:370-383); the immutable host
// array is shared between tensors of the same value.
PyObject* const_tensor(PyObject* scalar, int tag) {
  PyObject* key = Py_BuildValue("(iO)", tag, scalar);
  if (!key) return nullptr;
  PyObject* arr = PyDict_GetItemWithError(g_scalar_cache, key);  // borrowed
  if (arr) {
    Py_INCREF(arr);
  } else {
    if (PyErr_Occurred()) {
      Py_DECREF(key);
      return nullptr;
    }
    arr = PyObject_CallFunctionObjArgs(g_host_scalar, scalar, g_dtypes[tag], nullptr);
    if (!arr) {
      Py_DECREF(key);
      return nullptr;
    }
    if (PyDict_GET_SIZE(g_scalar_cache) > 4096) PyDict_Clear(g_scalar_cache);
    if (PyDict_SetItem(g_scalar_cache, key, arr) < 0) {
      Py_DECREF(key);
      Py_DECREF(arr);
      return nullptr;
    }
  }
  Py_DECREF(key);
  PyObject* t = new_tensor(g_dtypes[tag], g_empty_shape, nullptr, arr);
  Py_DECREF(arr);
  return t;
}

// A binary operation with the reference's operand coercion (_binary /
// operator overloads, ops.py:370-485): Tensor (op) Tensor, or a Tensor with
// a Python scalar taken "like" the tensor.  Returns NOT_FAST to defer.
PyObject* fast_binary(PyObject* name, PyObject* a, PyObject* b) {
  PyObject* ctx = fast_context();
  if (!ctx) return NOT_FAST;
  FastOp* f = lookup(name);
  if (!f) return NOT_FAST;
  const bool at = is_tensor(a), bt = is_tensor(b);
  if ((at && !concrete(a)) || (bt && !concrete(b))) return NOT_FAST;
  double sa, sb;
  const double* psa = nullptr;
  const double* psb = nullptr;
  if (!at || !bt) {
    if (f->kind != K_EW2 || (!at && !bt)) return NOT_FAST;
    PyObject* like = at ? a : b;
    const int tag = tag_of(((TensorObj*)like)->dtype);
    if (at) {
      if (!scalar_imm(b, tag, &sb)) return NOT_FAST;
      psb = &sb;
    } else {
      if (!scalar_imm(a, tag, &sa)) return NOT_FAST;
      psa = &sa;
    }
  }
  PyObject* in[2];
  if ((psa || psb) && tapes_active(ctx)) {
    // a watching tape records the scalar as a constant tensor input (the
    // reference's _as_operand): build it (host bytes, no upload)
    const int tag = tag_of(((TensorObj*)(at ? a : b))->dtype);
    PyObject* c = const_tensor(at ? b : a, tag);
    if (!c) return nullptr;
    in[0] = at ? Py_NewRef(a) : c;
    in[1] = at ? c : Py_NewRef(b);
    psa = psb = nullptr;
  } else {
    in[0] = Py_NewRef(a);
    in[1] = Py_NewRef(b);
  }
  PyObject* out = run_fast(*f, in, 2, nullptr, psa, psb, nullptr);
  if (out && out != NOT_FAST && !finish(*f, ctx, in, 2, out, nullptr)) {
    Py_DECREF(out);
    out = nullptr;
  }
  Py_DECREF(in[0]);
  Py_DECREF(in[1]);
  return out;
}

// ------------------------------------------------------ wrapper callables
//
// FastWrapper(op_name, arity, slow): a callable that runs `op_name` on its
// tensor arguments through the fast path and returns the single output,
// calling slow(*args) (the reference-semantics Python wrapper) otherwise.

struct FastWrapper {
  PyObject_HEAD
  PyObject* name;
  PyObject* slow;
  int arity;
  vectorcallfunc vectorcall;
};

PyObject* FastWrapper_call(PyObject* o, PyObject* const* args, size_t nargsf, PyObject* kw) {
  FastWrapper* w = (FastWrapper*)o;
  const Py_ssize_t n = PyVectorcall_NARGS(nargsf);
  if (!kw && n == w->arity && !PyErr_Occurred()) {
    PyObject* out = NOT_FAST;
    if (n == 2) {
      out = fast_binary(w->name, args[0], args[1]);
    } else if (n == 1 && is_tensor(args[0]) && concrete(args[0])) {
      PyObject* ctx = fast_context();
      FastOp* f = ctx ? lookup(w->name) : nullptr;
      if (f) {
        {
          PyObject* in[1] = {Py_NewRef(args[0])};
          out = run_fast(*f, in, 1, nullptr, nullptr, nullptr, nullptr);
          if (out && out != NOT_FAST && !finish(*f, ctx, in, 1, out, nullptr)) {
            Py_DECREF(out);
            out = nullptr;
          }
          Py_DECREF(in[0]);
        }
      }
    }
    if (out != NOT_FAST) return out;
    if (PyErr_Occurred()) return nullptr;
  }
  return PyObject_Vectorcall(w->slow, args, nargsf, kw);
}

int FastWrapper_traverse(PyObject* o, visitproc visit, void* arg) {
  FastWrapper* w = (FastWrapper*)o;
  Py_VISIT(w->name);
  Py_VISIT(w->slow);
  return 0;
}

void FastWrapper_dealloc(PyObject* o) {
  PyObject_GC_UnTrack(o);
  FastWrapper* w = (FastWrapper*)o;
  Py_CLEAR(w->name);
  Py_CLEAR(w->slow);
  Py_TYPE(o)->tp_free(o);
}

PyObject* FastWrapper_new(PyTypeObject* type, PyObject* args, PyObject* kw) {
  PyObject *name, *slow;
  int arity;
  if (!PyArg_ParseTuple(args, "UiO", &name, &arity, &slow)) return nullptr;
  FastWrapper* w = (FastWrapper*)type->tp_alloc(type, 0);
  if (!w) return nullptr;
  w->name = Py_NewRef(name);
  w->slow = Py_NewRef(slow);
  w->arity = arity;
  w->vectorcall = FastWrapper_call;
  return (PyObject*)w;
}

PyObject* FastWrapper_get_name(PyObject* o, void*) {
  return PyObject_GetAttrString(((FastWrapper*)o)->slow, "__name__");
}

PyObject* FastWrapper_get_doc(PyObject* o, void*) {
  return PyObject_GetAttrString(((FastWrapper*)o)->slow, "__doc__");
}

PyGetSetDef FastWrapper_getset[] = {
    {"__name__", FastWrapper_get_name, nullptr, nullptr, nullptr},
    {"__doc__", FastWrapper_get_doc, nullptr, nullptr, nullptr},
    {nullptr}};

PyMemberDef FastWrapper_members[] = {
    {"slow", T_OBJECT, offsetof(FastWrapper, slow), READONLY, nullptr},
    {"op", T_OBJECT, offsetof(FastWrapper, name), READONLY, nullptr},
    {nullptr}};

PyTypeObject FastWrapperType = {PyVarObject_HEAD_INIT(nullptr, 0)};

// --------------------------------------------------- Tensor operators
// (reference ops.py:456-485: fwd(op)(self, other) = dispatch(op, [self,
// _as_operand(other, like=self)]); rev(op) swaps the operands)

PyObject* g_binop_slow = nullptr;  // ops._operator_slow(op, a, b, reflected)
PyObject* g_op_names[8] = {};     // add sub mul div matmul greater neg

PyObject* tensor_binop(int which, PyObject* a, PyObject* b, bool has_reflected) {
  const bool at = is_tensor(a);
  if (!at && !has_reflected) Py_RETURN_NOTIMPLEMENTED;
  PyObject* name = g_op_names[which];
  PyObject* out = fast_binary(name, a, b);
  if (out != NOT_FAST) return out;
  if (PyErr_Occurred()) return nullptr;
  if (!g_binop_slow) Py_RETURN_NOTIMPLEMENTED;
  return PyObject_CallFunctionObjArgs(g_binop_slow, name, a, b, at ? Py_False : Py_True, nullptr);
}

PyObject* T_add(PyObject* a, PyObject* b) { return tensor_binop(0, a, b, true); }
PyObject* T_sub(PyObject* a, PyObject* b) { return tensor_binop(1, a, b, true); }
PyObject* T_mul(PyObject* a, PyObject* b) { return tensor_binop(2, a, b, true); }
PyObject* T_div(PyObject* a, PyObject* b) { return tensor_binop(3, a, b, true); }
PyObject* T_matmul(PyObject* a, PyObject* b) { return tensor_binop(4, a, b, false); }

PyObject* T_neg(PyObject* a) {
  PyObject* args[3] = {g_op_names[6], nullptr, nullptr};
  PyObject* lst = PyList_New(1);
  if (!lst) return nullptr;
  PyList_SET_ITEM(lst, 0, Py_NewRef(a));
  args[1] = lst;
  PyObject* r = py_dispatch(nullptr, args, 2);
  Py_DECREF(lst);
  if (!r) return nullptr;
  PyObject* out = PyList_GetItem(r, 0);
  Py_XINCREF(out);
  Py_DECREF(r);
  return out;
}

PyObject* T_richcompare(PyObject* a, PyObject* b, int op) {
  switch (op) {
    case Py_EQ:
      return PyBool_FromLong(a == b);
    case Py_NE:
      return PyBool_FromLong(a != b);
    case Py_GT:
      return tensor_binop(5, a, b, false);
    default:
      Py_RETURN_NOTIMPLEMENTED;
  }
}

PyNumberMethods Tensor_number = {};

// ------------------------------------------------------- staged call path
//
// StagedFast: the repeat-call fast path of one staged function (reference:
// PolymorphicFunction.__call__ -> call_concrete -> dispatch("call_function")
// -> execute_graph, stageflow/staging.py:453-460, :353-407,
// stageflow/kernels.py:460-480).  Built by staging.py after a call that
// took the slow path, for a function whose program is one native plan and
// whose captures are all tensors.  A call with the same number of
// positional tensor arguments of the same dtypes and shapes (the same trace
// key) runs the plan directly: argument pointers plus the captures'
// pre-resolved pointers, one sf_plan_run, output tensors built here, the
// call_function dispatch counted.  Anything else returns MISS and the
// caller runs the reference path.

PyObject* g_miss = nullptr;
unsigned long long g_graph_launches = 0;
int g_call_idx = -1;  // table index of "call_function" (its eager counter)

struct StagedFast {
  PyObject_HEAD
  PyObject* rt;
  PyObject* keep;        // objects kept alive (program, plan, captures)
  PyObject* lock;        // the plan's Python lock (shared with Plan.run)
  PyObject* arg_dtypes;  // tuple
  PyObject* arg_shapes;  // tuple
  PyObject* out_dtypes;  // tuple
  PyObject* out_shapes;  // tuple
  PyObject* device;
  void* plan;
  int dev, n_args, n_in, n_out, structure;
  int* in_src;           // plan input -> explicit arg index, or -1 (capture)
  void** in_ptr;         // capture pointers pre-filled
  int* out_slot;
  Py_ssize_t* out_nbytes;
  vectorcallfunc vectorcall;
};

PyObject* StagedFast_call(PyObject* o, PyObject* const* args, size_t nargsf, PyObject* kw) {
  StagedFast* f = (StagedFast*)o;
  const Py_ssize_t n = PyVectorcall_NARGS(nargsf);
  if (kw || n != f->n_args) return Py_NewRef(g_miss);
  PyObject* ctx = fast_context();
  if (!ctx || f->rt != g_rt || tapes_active(ctx)) {
    if (PyErr_Occurred()) return nullptr;
    return Py_NewRef(g_miss);
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* a = args[i];
    if (!is_tensor(a) || !concrete(a)) return Py_NewRef(g_miss);
    TensorObj* t = (TensorObj*)a;
    if (t->dtype != PyTuple_GET_ITEM(f->arg_dtypes, i)) return Py_NewRef(g_miss);
    PyObject* want = PyTuple_GET_ITEM(f->arg_shapes, i);
    if (t->shape != want) {
      const int eq = PyObject_RichCompareBool(t->shape, want, Py_EQ);
      if (eq < 0) return nullptr;
      if (!eq) return Py_NewRef(g_miss);
    }
  }
  void* ins[256];
  void* outs[256];
  for (int k = 0; k < f->n_in; ++k) {
    const int src = f->in_src[k];
    if (src < 0) {
      ins[k] = f->in_ptr[k];
    } else {
      const void* p;
      if (!device_ptr((TensorObj*)args[src], &p)) return nullptr;
      ins[k] = (void*)p;
    }
  }
  // serialise with Plan.run on the same plan (non-blocking: busy -> MISS)
  PyObject* got = PyObject_CallMethod(f->lock, "acquire", "O", Py_False);
  if (!got) return nullptr;
  const int have = PyObject_IsTrue(got);
  Py_DECREF(got);
  if (have != 1) return Py_NewRef(g_miss);
  const int st = sf_plan_run(f->plan, ins, outs);
  PyObject* rel = PyObject_CallMethod(f->lock, "release", nullptr);
  Py_XDECREF(rel);
  if (st != SF_OK) return kernel_error("plan run");
  PyObject* res = PyTuple_New(f->n_out);
  if (!res) return nullptr;
  for (int j = 0; j < f->n_out; ++j) {
    PyObject* buf = new_devbuf(f->dev, outs[f->out_slot[j]], f->out_nbytes[j]);
    PyObject* t = buf ? new_tensor(PyTuple_GET_ITEM(f->out_dtypes, j),
                                   PyTuple_GET_ITEM(f->out_shapes, j), buf, nullptr)
                      : nullptr;
    Py_XDECREF(buf);
    if (!t) {
      Py_DECREF(res);
      return nullptr;
    }
    PyTuple_SET_ITEM(res, j, t);
  }
  if (f->n_out > 1) {  // siblings: reading one output enqueues the others' reads
    PyObject* sib = PyList_New(f->n_out);
    if (!sib) {
      Py_DECREF(res);
      return nullptr;
    }
    for (int j = 0; j < f->n_out; ++j) {
      PyObject* w = PyWeakref_NewRef(PyTuple_GET_ITEM(res, j), nullptr);
      if (!w) {
        Py_DECREF(sib);
        Py_DECREF(res);
        return nullptr;
      }
      PyList_SET_ITEM(sib, j, w);
    }
    for (int j = 0; j < f->n_out; ++j) {
      TensorObj* t = (TensorObj*)PyTuple_GET_ITEM(res, j);
      Py_XSETREF(t->sib, Py_NewRef(sib));
    }
    Py_DECREF(sib);
  }
  if (g_call_idx >= 0) g_ops[g_call_idx].count++;
  g_graph_launches++;
  switch (f->structure) {
    case 0:
      Py_DECREF(res);
      Py_RETURN_NONE;
    case 1: {
      PyObject* one = Py_NewRef(PyTuple_GET_ITEM(res, 0));
      Py_DECREF(res);
      return one;
    }
    case 2:
      return res;
    default: {
      PyObject* lst = PySequence_List(res);
      Py_DECREF(res);
      return lst;
    }
  }
}

void StagedFast_dealloc(PyObject* o) {
  StagedFast* f = (StagedFast*)o;
  PyObject_GC_UnTrack(o);
  Py_CLEAR(f->rt);
  Py_CLEAR(f->keep);
  Py_CLEAR(f->lock);
  Py_CLEAR(f->arg_dtypes);
  Py_CLEAR(f->arg_shapes);
  Py_CLEAR(f->out_dtypes);
  Py_CLEAR(f->out_shapes);
  Py_CLEAR(f->device);
  PyMem_Free(f->in_src);
  PyMem_Free(f->in_ptr);
  PyMem_Free(f->out_slot);
  PyMem_Free(f->out_nbytes);
  Py_TYPE(o)->tp_free(o);
}

int StagedFast_traverse(PyObject* o, visitproc visit, void* arg) {
  StagedFast* f = (StagedFast*)o;
  Py_VISIT(f->rt);
  Py_VISIT(f->keep);
  Py_VISIT(f->lock);
  return 0;
}

// StagedFast(rt, keep, lock, plan_handle, dev, device, arg_dtypes, arg_shapes,
//            in_src (list: arg index or -1), in_ptr (list: capture pointer or 0),
//            out_slots, out_nbytes, out_dtypes, out_shapes, structure)
PyObject* StagedFast_new(PyTypeObject* type, PyObject* args, PyObject*) {
  PyObject *rt, *keep, *lock, *device, *adt, *ash, *isrc, *iptr, *oslot, *onb, *odt, *osh;
  unsigned long long plan;
  int dev, structure;
  if (!PyArg_ParseTuple(args, "OOOKiOO!O!O!O!O!O!O!O!i", &rt, &keep, &lock, &plan, &dev,
                        &device, &PyTuple_Type, &adt, &PyTuple_Type, &ash, &PyList_Type, &isrc,
                        &PyList_Type, &iptr, &PyList_Type, &oslot, &PyList_Type, &onb,
                        &PyTuple_Type, &odt, &PyTuple_Type, &osh, &structure))
    return nullptr;
  const Py_ssize_t n_in = PyList_GET_SIZE(isrc), n_out = PyList_GET_SIZE(oslot);
  if (n_in > 256 || n_out > 256 || PyList_GET_SIZE(iptr) != n_in ||
      PyList_GET_SIZE(onb) != n_out || PyTuple_GET_SIZE(odt) != n_out ||
      PyTuple_GET_SIZE(osh) != n_out || PyTuple_GET_SIZE(adt) != PyTuple_GET_SIZE(ash)) {
    PyErr_SetString(PyExc_ValueError, "StagedFast: inconsistent arguments");
    return nullptr;
  }
  StagedFast* f = (StagedFast*)type->tp_alloc(type, 0);
  if (!f) return nullptr;
  f->rt = Py_NewRef(rt);
  f->keep = Py_NewRef(keep);
  f->lock = Py_NewRef(lock);
  f->arg_dtypes = Py_NewRef(adt);
  f->arg_shapes = Py_NewRef(ash);
  f->out_dtypes = Py_NewRef(odt);
  f->out_shapes = Py_NewRef(osh);
  f->device = Py_NewRef(device);
  f->plan = (void*)(uintptr_t)plan;
  f->dev = dev;
  f->n_args = (int)PyTuple_GET_SIZE(adt);
  f->n_in = (int)n_in;
  f->n_out = (int)n_out;
  f->structure = structure;
  f->in_src = (int*)PyMem_Calloc(n_in + 1, sizeof(int));
  f->in_ptr = (void**)PyMem_Calloc(n_in + 1, sizeof(void*));
  f->out_slot = (int*)PyMem_Calloc(n_out + 1, sizeof(int));
  f->out_nbytes = (Py_ssize_t*)PyMem_Calloc(n_out + 1, sizeof(Py_ssize_t));
  f->vectorcall = StagedFast_call;
  if (!f->in_src || !f->in_ptr || !f->out_slot || !f->out_nbytes) {
    Py_DECREF(f);
    return PyErr_NoMemory();
  }
  for (Py_ssize_t k = 0; k < n_in; ++k) {
    f->in_src[k] = (int)PyLong_AsLong(PyList_GET_ITEM(isrc, k));
    f->in_ptr[k] = PyLong_AsVoidPtr(PyList_GET_ITEM(iptr, k));
  }
  for (Py_ssize_t j = 0; j < n_out; ++j) {
    f->out_slot[j] = (int)PyLong_AsLong(PyList_GET_ITEM(oslot, j));
    f->out_nbytes[j] = PyLong_AsSsize_t(PyList_GET_ITEM(onb, j));
  }
  if (PyErr_Occurred()) {
    Py_DECREF(f);
    return nullptr;
  }
  return (PyObject*)f;
}

PyTypeObject StagedFastType = {PyVarObject_HEAD_INIT(nullptr, 0)};

// ---------------------------------------------------------- configuration

// bootstrap(rt_module_dict, thread_local, configure_cb, slow_dispatch,
//           binop_slow, host_scalar): where to find the
// live runtime (`_runtime` in paper_1903_01855_b200.runtime), the
// per-thread context, and the Python function that (re)binds the fast path
// when the live runtime changes (init_runtime).
PyObject* py_bootstrap(PyObject*, PyObject* args) {
  PyObject *rt_dict, *local, *cfg, *slow, *binop_slow, *host_scalar;
  if (!PyArg_ParseTuple(args, "O!OOOOO", &PyDict_Type, &rt_dict, &local, &cfg, &slow,
                        &binop_slow, &host_scalar))
    return nullptr;
  Py_XSETREF(g_host_scalar, Py_NewRef(host_scalar));
  if (!g_scalar_cache && !(g_scalar_cache = PyDict_New())) return nullptr;
  if (!g_empty_shape && !(g_empty_shape = PyTuple_New(0))) return nullptr;
  Py_XSETREF(g_rt_dict, Py_NewRef(rt_dict));
  Py_XSETREF(g_local, Py_NewRef(local));
  Py_XSETREF(g_configure, Py_NewRef(cfg));
  Py_XSETREF(g_slow_dispatch, Py_NewRef(slow));
  Py_XSETREF(g_binop_slow, Py_NewRef(binop_slow));
  Py_RETURN_NONE;
}

// configure(runtime, registry, single, ordinal, device, tensor_type,
//           dtypes (4-tuple by wire tag), ctx_type, slow_dispatch, notify,
//           kernel_error, binop_slow, fast_ops: [(name, opdef, kind, opcode, flags)])
PyObject* py_configure(PyObject*, PyObject* args) {
  PyObject *rt, *registry, *device, *ttype, *dts, *ctx_type, *slow, *notify, *kerr, *binop_slow,
      *ops;
  int single, ordinal;
  if (!PyArg_ParseTuple(args, "OOpiOO!O!OOOOOO!", &rt, &registry, &single, &ordinal, &device,
                        &PyType_Type, &ttype, &PyTuple_Type, &dts, &ctx_type, &slow, &notify,
                        &kerr, &binop_slow, &PyList_Type, &ops))
    return nullptr;
  if (!PyType_IsSubtype((PyTypeObject*)ttype, &TensorBaseType)) {
    PyErr_SetString(PyExc_TypeError, "tensor type must derive from TensorBase");
    return nullptr;
  }
  if (PyTuple_GET_SIZE(dts) != 4 || PyList_GET_SIZE(ops) > kMaxFast) {
    PyErr_SetString(PyExc_ValueError, "bad configure arguments");
    return nullptr;
  }
  const Py_ssize_t ot = slot_offset(ctx_type, "traces");
  const Py_ssize_t ok = slot_offset(ctx_type, "tapes");
  const Py_ssize_t os = slot_offset(ctx_type, "device_scopes");
  if (ot < 0 || ok < 0 || os < 0) return nullptr;
  PyObject* table = PyDict_New();
  if (!table) return nullptr;
  FastOp fresh[kMaxFast];
  const Py_ssize_t n = PyList_GET_SIZE(ops);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject *name, *opdef;
    int kind, opcode, flags;
    if (!PyArg_ParseTuple(PyList_GET_ITEM(ops, i), "UOiii", &name, &opdef, &kind, &opcode,
                          &flags)) {
      for (Py_ssize_t j = 0; j < i; ++j) {
        Py_DECREF(fresh[j].opdef);
        Py_DECREF(fresh[j].name);
      }
      Py_DECREF(table);
      return nullptr;
    }
    PyObject* idx = PyLong_FromSsize_t(i);
    if (!idx || PyDict_SetItem(table, name, idx) < 0) {
      Py_XDECREF(idx);
      for (Py_ssize_t j = 0; j < i; ++j) {
        Py_DECREF(fresh[j].opdef);
        Py_DECREF(fresh[j].name);
      }
      Py_DECREF(table);
      return nullptr;
    }
    Py_DECREF(idx);
    fresh[i].opdef = Py_NewRef(opdef);
    fresh[i].name = Py_NewRef(name);
    fresh[i].kind = kind;
    fresh[i].opcode = opcode;
    fresh[i].flags = flags;
  }
  for (int i = 0; i < g_nops; ++i) {
    Py_CLEAR(g_ops[i].opdef);
    Py_CLEAR(g_ops[i].name);
  }
  for (Py_ssize_t i = 0; i < n; ++i) g_ops[i] = fresh[i];
  g_nops = (int)n;
  Py_XSETREF(g_table, table);
  Py_XSETREF(g_rt, Py_NewRef(rt));
  Py_XSETREF(g_registry, Py_NewRef(registry));
  Py_XSETREF(g_device, Py_NewRef(device));
  Py_XSETREF(g_tensor_type, (PyTypeObject*)Py_NewRef(ttype));
  for (int i = 0; i < 4; ++i) Py_XSETREF(g_dtypes[i + 1], Py_NewRef(PyTuple_GET_ITEM(dts, i)));
  Py_XSETREF(g_slow_dispatch, Py_NewRef(slow));
  Py_XSETREF(g_notify, Py_NewRef(notify));
  Py_XSETREF(g_kernel_error, Py_NewRef(kerr));
  Py_XSETREF(g_binop_slow, Py_NewRef(binop_slow));
  off_traces = ot;
  off_tapes = ok;
  off_scopes = os;
  g_single = single != 0;
  g_ordinal = ordinal;
  g_call_idx = -1;
  for (int i = 0; i < g_nops; ++i)
    if (PyUnicode_CompareWithASCIIString(g_ops[i].name, "call_function") == 0) g_call_idx = i;
  g_graph_launches = 0;
  Py_RETURN_NONE;
}

// add_op(registry, name, opdef, kind, opcode, flags): a plugin registered
// after configure (no-op unless `registry` is the configured one)
PyObject* py_add_op(PyObject*, PyObject* args) {
  PyObject *registry, *name, *opdef;
  int kind, opcode, flags;
  if (!PyArg_ParseTuple(args, "OUOiii", &registry, &name, &opdef, &kind, &opcode, &flags))
    return nullptr;
  if (registry != g_registry || !g_table) Py_RETURN_FALSE;
  if (g_nops >= kMaxFast) Py_RETURN_FALSE;
  PyObject* idx = PyLong_FromLong(g_nops);
  if (!idx || PyDict_SetItem(g_table, name, idx) < 0) {
    Py_XDECREF(idx);
    return nullptr;
  }
  Py_DECREF(idx);
  FastOp& f = g_ops[g_nops++];
  f.opdef = Py_NewRef(opdef);
  f.name = Py_NewRef(name);
  f.kind = kind;
  f.opcode = opcode;
  f.flags = flags;
  f.count = 0;
  Py_RETURN_TRUE;
}

// drain(runtime) -> {op: count} of fast dispatches since the last drain,
// counters zeroed; {} unless `runtime` is the configured one
PyObject* py_drain(PyObject*, PyObject* rt) {
  PyObject* d = PyDict_New();
  if (!d || rt != g_rt) return d;
  if (g_graph_launches) {
    PyObject* v = PyLong_FromUnsignedLongLong(g_graph_launches);
    if (!v || PyDict_SetItemString(d, "<graph_launches>", v) < 0) {
      Py_XDECREF(v);
      Py_DECREF(d);
      return nullptr;
    }
    Py_DECREF(v);
    g_graph_launches = 0;
  }
  for (int i = 0; i < g_nops; ++i) {
    if (!g_ops[i].count) continue;
    PyObject* v = PyLong_FromUnsignedLongLong(g_ops[i].count);
    if (!v || PyDict_SetItem(d, g_ops[i].name, v) < 0) {
      Py_XDECREF(v);
      Py_DECREF(d);
      return nullptr;
    }
    Py_DECREF(v);
    g_ops[i].count = 0;
  }
  return d;
}

// pending(runtime) -> total fast dispatches not yet drained
PyObject* py_pending(PyObject*, PyObject* rt) {
  unsigned long long s = 0;
  if (rt == g_rt)
    for (int i = 0; i < g_nops; ++i) s += g_ops[i].count;
  return PyLong_FromUnsignedLongLong(s);
}

PyObject* py_set_enabled(PyObject*, PyObject* v) {
  const int on = PyObject_IsTrue(v);
  if (on < 0) return nullptr;
  const bool was = g_enabled;
  g_enabled = on != 0;
  return PyBool_FromLong(was);
}

PyMethodDef methods[] = {
    {"dispatch", (PyCFunction)(void (*)(void))py_dispatch, METH_FASTCALL,
     "dispatch(op, inputs, attrs=None) -> list of outputs (native fast path, else ops._dispatch_py)"},
    {"bootstrap", py_bootstrap, METH_VARARGS, "where to find the live runtime and context"},
    {"configure", py_configure, METH_VARARGS, "bind the fast path to a runtime"},
    {"add_op", py_add_op, METH_VARARGS, "add a fast op registered after configure"},
    {"drain", py_drain, METH_O, "fast-path dispatch counts since the last drain"},
    {"pending", py_pending, METH_O, "fast-path dispatches not yet drained"},
    {"set_enabled", py_set_enabled, METH_O, "enable/disable the fast path; returns the old state"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_sfeager",
                      "native eager front-end of paper_1903_01855_b200", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__sfeager(void) {
  s_owner = PyUnicode_InternFromString("owner");
  s_context = PyUnicode_InternFromString("context");
  s_runtime = PyUnicode_InternFromString("_runtime");
  s_device_buffer = PyUnicode_InternFromString("_device_buffer");
  s_ptr = PyUnicode_InternFromString("ptr");
  s_reshape = PyUnicode_InternFromString("reshape");
  s_shape = PyUnicode_InternFromString("shape");
  const char* names[7] = {"add", "sub", "mul", "div", "matmul", "greater", "neg"};
  for (int i = 0; i < 7; ++i) g_op_names[i] = PyUnicode_InternFromString(names[i]);

  DevBufType.tp_name = "_sfeager.DeviceBuffer";
  DevBufType.tp_doc = "One block of a device's caching allocator (sf_free on release).";
  DevBufType.tp_basicsize = sizeof(DevBuf);
  DevBufType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE;
  DevBufType.tp_new = PyType_GenericNew;
  DevBufType.tp_init = DevBuf_init;
  DevBufType.tp_dealloc = DevBuf_dealloc;
  DevBufType.tp_members = DevBuf_members;
  DevBufType.tp_weaklistoffset = offsetof(DevBuf, weakreflist);
  if (PyType_Ready(&DevBufType) < 0) return nullptr;

  Tensor_number.nb_add = T_add;
  Tensor_number.nb_subtract = T_sub;
  Tensor_number.nb_multiply = T_mul;
  Tensor_number.nb_true_divide = T_div;
  Tensor_number.nb_matrix_multiply = T_matmul;
  Tensor_number.nb_negative = T_neg;
  TensorBaseType.tp_name = "_sfeager.TensorBase";
  TensorBaseType.tp_doc = "Slot layout and operators of Tensor.";
  TensorBaseType.tp_basicsize = sizeof(TensorObj);
  TensorBaseType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE | Py_TPFLAGS_HAVE_GC;
  TensorBaseType.tp_new = PyType_GenericNew;
  TensorBaseType.tp_dealloc = Tensor_dealloc;
  TensorBaseType.tp_traverse = Tensor_traverse;
  TensorBaseType.tp_clear = Tensor_clear;
  TensorBaseType.tp_members = Tensor_members;
  TensorBaseType.tp_weaklistoffset = offsetof(TensorObj, weakreflist);
  TensorBaseType.tp_as_number = &Tensor_number;
  TensorBaseType.tp_richcompare = T_richcompare;
  TensorBaseType.tp_hash = PyBaseObject_Type.tp_hash;
  if (PyType_Ready(&TensorBaseType) < 0) return nullptr;

  FastWrapperType.tp_name = "_sfeager.FastWrapper";
  FastWrapperType.tp_doc = "FastWrapper(op, arity, slow): native fast path of an op wrapper.";
  FastWrapperType.tp_basicsize = sizeof(FastWrapper);
  FastWrapperType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC | Py_TPFLAGS_HAVE_VECTORCALL;
  FastWrapperType.tp_new = FastWrapper_new;
  FastWrapperType.tp_dealloc = FastWrapper_dealloc;
  FastWrapperType.tp_traverse = FastWrapper_traverse;
  FastWrapperType.tp_call = PyVectorcall_Call;
  FastWrapperType.tp_vectorcall_offset = offsetof(FastWrapper, vectorcall);
  FastWrapperType.tp_getset = FastWrapper_getset;
  FastWrapperType.tp_members = FastWrapper_members;
  if (PyType_Ready(&FastWrapperType) < 0) return nullptr;

  StagedFastType.tp_name = "_sfeager.StagedFast";
  StagedFastType.tp_doc = "Repeat-call fast path of one staged function.";
  StagedFastType.tp_basicsize = sizeof(StagedFast);
  StagedFastType.tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_GC | Py_TPFLAGS_HAVE_VECTORCALL;
  StagedFastType.tp_new = StagedFast_new;
  StagedFastType.tp_dealloc = StagedFast_dealloc;
  StagedFastType.tp_traverse = StagedFast_traverse;
  StagedFastType.tp_call = PyVectorcall_Call;
  StagedFastType.tp_vectorcall_offset = offsetof(StagedFast, vectorcall);
  if (PyType_Ready(&StagedFastType) < 0) return nullptr;
  g_miss = PyObject_CallNoArgs((PyObject*)&PyBaseObject_Type);
  if (!g_miss) return nullptr;

  PyObject* m = PyModule_Create(&moddef);
  if (!m) return nullptr;
  if (PyModule_AddObjectRef(m, "DeviceBuffer", (PyObject*)&DevBufType) < 0 ||
      PyModule_AddObjectRef(m, "TensorBase", (PyObject*)&TensorBaseType) < 0 ||
      PyModule_AddObjectRef(m, "FastWrapper", (PyObject*)&FastWrapperType) < 0 ||
      PyModule_AddObjectRef(m, "StagedFast", (PyObject*)&StagedFastType) < 0 ||
      PyModule_AddObjectRef(m, "MISS", g_miss) < 0 ||
      PyModule_AddIntConstant(m, "K_EW1", K_EW1) < 0 ||
      PyModule_AddIntConstant(m, "K_EW2", K_EW2) < 0 ||
      PyModule_AddIntConstant(m, "K_MATMUL", K_MATMUL) < 0 ||
      PyModule_AddIntConstant(m, "K_TRANSPOSE", K_TRANSPOSE) < 0 ||
      PyModule_AddIntConstant(m, "K_IDENTITY", K_IDENTITY) < 0 ||
      PyModule_AddIntConstant(m, "K_RESHAPE", K_RESHAPE) < 0 ||
      PyModule_AddIntConstant(m, "K_BROADCAST_TO", K_BROADCAST_TO) < 0 ||
      PyModule_AddIntConstant(m, "F_FLOATS_ONLY", F_FLOATS_ONLY) < 0 ||
      PyModule_AddIntConstant(m, "F_OUT_BOOL", F_OUT_BOOL) < 0) {
    Py_DECREF(m);
    return nullptr;
  }
  return m;
}
