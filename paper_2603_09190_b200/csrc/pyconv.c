/* _zpir_conv: Python int <-> little-endian u32 limb buffers, in C.
 *
 * The reference API carries big integers as Python ints (QueryMessage.ck_o,
 * ResponseMessage.t, PaillierCiphertext.c); converting 1024 x 2048-bit ints
 * with int.to_bytes / int.from_bytes costs ~0.4 ms each way in CPython,
 * more than the whole device answer. These two loops use CPython's
 * _PyLong_AsByteArray / _PyLong_FromByteArray directly.
 *
 *   ints_into(seq, buf, nlimbs)   writes len(seq) x nlimbs u32 LE into a
 *                                 writable buffer (numpy / pinned tensor);
 *                                 ValueError on negative or too-wide ints
 *   ints_from(buf, count, nlimbs) -> list of count Python ints
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* CPython 3.12/3.13 store ints as 30-bit digits behind lv_tag (ndigits << 3 |
 * sign); converting digits <-> 32-bit limbs directly is ~4x faster than the
 * byte-array API. Other versions use the byte-array API. */
#if PY_VERSION_HEX >= 0x030C0000 && PY_VERSION_HEX < 0x030E0000 && PYLONG_BITS_IN_DIGIT == 30
#define ZPIR_FAST_DIGITS 1
#include "cpython/longintrepr.h"

/* returns 0 ok, -1 negative, -2 too wide */
static int long_to_limbs(PyObject* v, uint32_t* o, Py_ssize_t nlimbs) {
  PyLongObject* L = (PyLongObject*)v;
  const uintptr_t tag = L->long_value.lv_tag;
  if ((tag & 3) == 2) return -1;
  const Py_ssize_t nd = (Py_ssize_t)(tag >> 3);
  const digit* d = L->long_value.ob_digit;
  uint64_t acc = 0;
  int bits = 0;
  Py_ssize_t li = 0;
  for (Py_ssize_t i = 0; i < nd; ++i) {
    acc |= (uint64_t)d[i] << bits;
    bits += 30;
    if (bits >= 32) {
      if (li >= nlimbs) return -2;
      o[li++] = (uint32_t)acc;
      acc >>= 32;
      bits -= 32;
    }
  }
  if (acc) {
    if (li >= nlimbs) return -2;
    o[li++] = (uint32_t)acc;
  }
  if (li < nlimbs) memset(o + li, 0, (size_t)(nlimbs - li) * 4);
  return 0;
}

static PyObject* limbs_to_long(const uint32_t* l, Py_ssize_t nlimbs) {
  digit dig[1024];
  Py_ssize_t k = 0;
  uint64_t acc = 0;
  int bits = 0;
  if (nlimbs > 900) return _PyLong_FromByteArray((const unsigned char*)l, (size_t)nlimbs * 4, 1, 0);
  for (Py_ssize_t i = 0; i < nlimbs; ++i) {
    acc |= (uint64_t)l[i] << bits;
    bits += 32;
    while (bits >= 30) {
      dig[k++] = (digit)(acc & 0x3fffffffu);
      acc >>= 30;
      bits -= 30;
    }
  }
  if (bits > 0) dig[k++] = (digit)acc;
  while (k > 0 && dig[k - 1] == 0) --k;
  if (k == 0) return PyLong_FromLong(0);
  return (PyObject*)_PyLong_FromDigits(0, k, dig);
}
#endif

static PyObject* ints_into(PyObject* self, PyObject* args) {
  PyObject* seq;
  Py_buffer view;
  Py_ssize_t nlimbs;
  if (!PyArg_ParseTuple(args, "Ow*n", &seq, &view, &nlimbs)) return NULL;
  PyObject* fast = PySequence_Fast(seq, "expected a sequence of ints");
  if (!fast) {
    PyBuffer_Release(&view);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  const size_t width = (size_t)nlimbs * 4;
  if ((size_t)view.len < (size_t)n * width) {
    PyErr_SetString(PyExc_ValueError, "buffer too small");
    goto fail;
  }
  PyObject** items = PySequence_Fast_ITEMS(fast);
  unsigned char* out = (unsigned char*)view.buf;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* v = items[i];
    PyObject* tmp = NULL;
    if (!PyLong_Check(v)) {
      PyObject* c = PyObject_GetAttrString(v, "c"); /* PaillierCiphertext */
      if (!c) goto fail;
      tmp = PyNumber_Index(c);
      Py_DECREF(c);
      if (!tmp) goto fail;
      v = tmp;
    }
#ifdef ZPIR_FAST_DIGITS
    {
      const int rc = long_to_limbs(v, (uint32_t*)(out + (size_t)i * width), nlimbs);
      if (rc) {
        Py_XDECREF(tmp);
        PyErr_SetString(PyExc_ValueError, rc == -1 ? "negative integers are not encodable"
                                                   : "integer wider than the limb width");
        goto fail;
      }
    }
#else
    if (_PyLong_Sign(v) < 0) {
      Py_XDECREF(tmp);
      PyErr_SetString(PyExc_ValueError, "negative integers are not encodable");
      goto fail;
    }
    if (_PyLong_AsByteArray((PyLongObject*)v, out + (size_t)i * width, width, 1, 0) < 0) {
      Py_XDECREF(tmp);
      PyErr_Clear();
      PyErr_SetString(PyExc_ValueError, "integer wider than the limb width");
      goto fail;
    }
#endif
    Py_XDECREF(tmp);
  }
  Py_DECREF(fast);
  PyBuffer_Release(&view);
  Py_RETURN_NONE;
fail:
  Py_DECREF(fast);
  PyBuffer_Release(&view);
  return NULL;
}

static PyObject* ints_from(PyObject* self, PyObject* args) {
  Py_buffer view;
  Py_ssize_t count, nlimbs;
  if (!PyArg_ParseTuple(args, "y*nn", &view, &count, &nlimbs)) return NULL;
  const size_t width = (size_t)nlimbs * 4;
  if ((size_t)view.len < (size_t)count * width) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "buffer too small");
    return NULL;
  }
  PyObject* list = PyList_New(count);
  if (!list) {
    PyBuffer_Release(&view);
    return NULL;
  }
  const unsigned char* p = (const unsigned char*)view.buf;
  for (Py_ssize_t i = 0; i < count; ++i) {
#ifdef ZPIR_FAST_DIGITS
    PyObject* v = limbs_to_long((const uint32_t*)(p + (size_t)i * width), nlimbs);
#else
    PyObject* v = _PyLong_FromByteArray(p + (size_t)i * width, width, 1, 0);
#endif
    if (!v) {
      Py_DECREF(list);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(list, i, v);
  }
  PyBuffer_Release(&view);
  return list;
}

#ifdef ZPIR_FAST_DIGITS
/* Raw CPython digits: buf[i*ndig .. +ndig) = the 30-bit digits of seq[i]
 * (zero-padded); the GPU regroups them into 32-bit limbs (zpir_digits_to_limbs). */
static PyObject* digits_into(PyObject* self, PyObject* args) {
  PyObject* seq;
  Py_buffer view;
  Py_ssize_t ndig, maxbits = 0;   /* maxbits > 0: reject wider values (the limb width) */
  if (!PyArg_ParseTuple(args, "Ow*n|n", &seq, &view, &ndig, &maxbits)) return NULL;
  PyObject* fast = PySequence_Fast(seq, "expected a sequence of ints");
  if (!fast) {
    PyBuffer_Release(&view);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  if ((size_t)view.len < (size_t)n * ndig * 4) {
    PyErr_SetString(PyExc_ValueError, "buffer too small");
    goto fail;
  }
  PyObject** items = PySequence_Fast_ITEMS(fast);
  uint32_t* out = (uint32_t*)view.buf;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* v = items[i];
    if (!PyLong_Check(v)) {
      PyErr_SetString(PyExc_TypeError, "expected int");
      goto fail;
    }
    PyLongObject* L = (PyLongObject*)v;
    const uintptr_t tag = L->long_value.lv_tag;
    if ((tag & 3) == 2) {
      PyErr_SetString(PyExc_ValueError, "negative integers are not encodable");
      goto fail;
    }
    const Py_ssize_t nd = (Py_ssize_t)(tag >> 3);
    if (nd > ndig) {
      PyErr_SetString(PyExc_ValueError, "integer wider than the limb width");
      goto fail;
    }
    if (maxbits > 0 && nd > 0) {
      const uint32_t top = (uint32_t)L->long_value.ob_digit[nd - 1];
      const Py_ssize_t bits = 30 * (nd - 1) + (32 - __builtin_clz(top));
      if (bits > maxbits) {
        PyErr_SetString(PyExc_ValueError, "integer wider than the limb width");
        goto fail;
      }
    }
    uint32_t* o = out + (size_t)i * ndig;
    if (nd) memcpy(o, L->long_value.ob_digit, (size_t)nd * 4);
    if (nd < ndig) memset(o + nd, 0, (size_t)(ndig - nd) * 4);
  }
  Py_DECREF(fast);
  PyBuffer_Release(&view);
  Py_RETURN_NONE;
fail:
  Py_DECREF(fast);
  PyBuffer_Release(&view);
  return NULL;
}

/* count ints from rows of ndig normalised 30-bit digits (zpir_limbs_to_digits). */
static PyObject* ints_from_digits(PyObject* self, PyObject* args) {
  Py_buffer view;
  Py_ssize_t count, ndig;
  if (!PyArg_ParseTuple(args, "y*nn", &view, &count, &ndig)) return NULL;
  if ((size_t)view.len < (size_t)count * ndig * 4) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "buffer too small");
    return NULL;
  }
  PyObject* list = PyList_New(count);
  if (!list) {
    PyBuffer_Release(&view);
    return NULL;
  }
  const uint32_t* p = (const uint32_t*)view.buf;
  for (Py_ssize_t i = 0; i < count; ++i) {
    const uint32_t* d = p + (size_t)i * ndig;
    Py_ssize_t k = ndig;
    while (k > 0 && d[k - 1] == 0) --k;
    PyObject* v = k ? (PyObject*)_PyLong_FromDigits(0, k, (digit*)d) : PyLong_FromLong(0);
    if (!v) {
      Py_DECREF(list);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(list, i, v);
  }
  PyBuffer_Release(&view);
  return list;
}
#endif

/* narrow_u32(src, dst, n): dst[i] = (uint32) src[i] for i < n, src a buffer of
 * 4- or 8-byte unsigned words (the query vector qu0 as numpy uint64 / uint32),
 * strided or not; the GIL is released for the copy. */
static PyObject* narrow_u32(PyObject* self, PyObject* args) {
  PyObject* src_obj;
  Py_buffer dst;
  Py_ssize_t n;
  if (!PyArg_ParseTuple(args, "Ow*n", &src_obj, &dst, &n)) return NULL;
  Py_buffer src;
  if (PyObject_GetBuffer(src_obj, &src, PyBUF_STRIDED_RO | PyBUF_FORMAT) < 0) {
    PyBuffer_Release(&dst);
    return NULL;
  }
  const Py_ssize_t item = src.itemsize;
  const Py_ssize_t stride = (src.ndim == 1 && src.strides) ? src.strides[0] : item;
  const Py_ssize_t len = (src.ndim == 1 && src.shape) ? src.shape[0] : src.len / item;
  if ((item != 4 && item != 8) || src.ndim > 1 || len < n || (size_t)dst.len < (size_t)n * 4) {
    PyBuffer_Release(&src);
    PyBuffer_Release(&dst);
    PyErr_SetString(PyExc_ValueError, "narrow_u32: need a 1-D buffer of 4/8-byte words");
    return NULL;
  }
  uint32_t* out = (uint32_t*)dst.buf;
  const char* p = (const char*)src.buf;
  Py_BEGIN_ALLOW_THREADS
  if (item == 8) {
    if (stride == 8) {
      const uint64_t* __restrict__ q = (const uint64_t*)p;
      uint32_t* __restrict__ o = out;
      for (Py_ssize_t i = 0; i < n; ++i) o[i] = (uint32_t)q[i];
    } else {
      for (Py_ssize_t i = 0; i < n; ++i) out[i] = (uint32_t)*(const uint64_t*)(p + i * stride);
    }
  } else if (stride == 4) {
    memcpy(out, p, (size_t)n * 4);
  } else {
    for (Py_ssize_t i = 0; i < n; ++i) out[i] = *(const uint32_t*)(p + i * stride);
  }
  Py_END_ALLOW_THREADS
  PyBuffer_Release(&src);
  PyBuffer_Release(&dst);
  Py_RETURN_NONE;
}

/* stage_rows(items, buf, item_bytes, rows, row_bytes, nthreads, words):
 * copies a batch of host arrays into one (pinned) staging buffer, item i at
 * buf + i * item_bytes, on nthreads threads with the GIL released -- the
 * host half of respond_batch_wire (64 queries: 8 MB of qu0 + 16 MB of ck_o).
 *   words = 0: item i is a C-contiguous (rows, w_i) byte matrix (w_i <=
 *              row_bytes); row r goes to buf + i item_bytes + r row_bytes,
 *              zero-padded to row_bytes (the ck_o wire fields -> u32 limbs)
 *   words = 1: item i is a 1-D buffer of 4- or 8-byte words (qu0), narrowed
 *              to u32 at buf + i item_bytes, zero-padded to row_bytes. */
typedef struct {
  const char* src;
  Py_ssize_t len, item, stride, w;
} StageItem;

typedef struct {
  StageItem* items;
  Py_ssize_t lo, hi, item_bytes, rows, row_bytes;
  int words;
  char* dst;
} StageJob;

static void* stage_worker(void* arg) {
  StageJob* j = (StageJob*)arg;
  for (Py_ssize_t i = j->lo; i < j->hi; ++i) {
    const StageItem* it = &j->items[i];
    char* out = j->dst + i * j->item_bytes;
    if (j->words) {
      uint32_t* o = (uint32_t*)out;
      if (it->item == 4 && it->stride == 4) {
        memcpy(o, it->src, (size_t)it->len * 4);
      } else if (it->item == 8 && it->stride == 8) {
        const uint64_t* q = (const uint64_t*)it->src;
        for (Py_ssize_t k = 0; k < it->len; ++k) o[k] = (uint32_t)q[k];
      } else {
        for (Py_ssize_t k = 0; k < it->len; ++k)
          o[k] = it->item == 8 ? (uint32_t) * (const uint64_t*)(it->src + k * it->stride)
                               : *(const uint32_t*)(it->src + k * it->stride);
      }
      if (it->len * 4 < j->row_bytes) memset(out + it->len * 4, 0, (size_t)(j->row_bytes - it->len * 4));
    } else if (it->w == j->row_bytes) {
      memcpy(out, it->src, (size_t)j->rows * j->row_bytes);
    } else {
      for (Py_ssize_t r = 0; r < j->rows; ++r) {
        memcpy(out + r * j->row_bytes, it->src + r * it->w, (size_t)it->w);
        memset(out + r * j->row_bytes + it->w, 0, (size_t)(j->row_bytes - it->w));
      }
    }
  }
  return NULL;
}

static PyObject* stage_rows(PyObject* self, PyObject* args) {
  PyObject* seq;
  Py_buffer dst;
  Py_ssize_t item_bytes, rows, row_bytes, nthreads;
  int words;
  if (!PyArg_ParseTuple(args, "Ow*nnnnp", &seq, &dst, &item_bytes, &rows, &row_bytes, &nthreads,
                        &words))
    return NULL;
  PyObject* fast = PySequence_Fast(seq, "expected a sequence of arrays");
  if (!fast) {
    PyBuffer_Release(&dst);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(fast);
  Py_buffer* views = (Py_buffer*)calloc((size_t)(n ? n : 1), sizeof(Py_buffer));
  StageItem* items = (StageItem*)calloc((size_t)(n ? n : 1), sizeof(StageItem));
  Py_ssize_t got = 0;
  PyObject* ret = NULL;
  if (!views || !items) {
    PyErr_NoMemory();
    goto done;
  }
  if ((size_t)dst.len < (size_t)n * item_bytes || row_bytes * (words ? 1 : rows) > item_bytes) {
    PyErr_SetString(PyExc_ValueError, "stage_rows: staging buffer too small");
    goto done;
  }
  for (; got < n; ++got) {
    PyObject* o = PySequence_Fast_GET_ITEM(fast, got);
    Py_buffer* v = &views[got];
    if (PyObject_GetBuffer(o, v, words ? (PyBUF_STRIDED_RO | PyBUF_FORMAT) : PyBUF_C_CONTIGUOUS) < 0)
      goto done;
    StageItem* it = &items[got];
    it->src = (const char*)v->buf;
    if (words) {
      it->item = v->itemsize;
      it->stride = (v->ndim == 1 && v->strides) ? v->strides[0] : v->itemsize;
      it->len = (v->ndim == 1 && v->shape) ? v->shape[0] : v->len / v->itemsize;
      if ((it->item != 4 && it->item != 8) || v->ndim > 1 || it->len * 4 > row_bytes) {
        PyErr_SetString(PyExc_ValueError, "stage_rows: need 1-D arrays of 4/8-byte words");
        ++got;
        goto done;
      }
    } else {
      if (rows <= 0 || v->len % rows || v->len / rows > row_bytes) {
        PyErr_SetString(PyExc_ValueError, "stage_rows: field rows wider than the limb width");
        ++got;
        goto done;
      }
      it->w = v->len / rows;
    }
  }
  {
    Py_ssize_t T = nthreads < 1 ? 1 : (nthreads > 32 ? 32 : nthreads);
    if (T > n) T = n ? n : 1;
    StageJob jobs[32];
    pthread_t th[32];
    int started[32] = {0};
    for (Py_ssize_t t = 0; t < T; ++t)
      jobs[t] = (StageJob){items, n * t / T, n * (t + 1) / T, item_bytes, rows, row_bytes, words,
                           (char*)dst.buf};
    Py_BEGIN_ALLOW_THREADS
    for (Py_ssize_t t = 1; t < T; ++t)
      started[t] = pthread_create(&th[t], NULL, stage_worker, &jobs[t]) == 0;
    stage_worker(&jobs[0]);
    for (Py_ssize_t t = 1; t < T; ++t) {
      if (started[t]) pthread_join(th[t], NULL);
      else stage_worker(&jobs[t]);     /* thread creation failed: copy here */
    }
    Py_END_ALLOW_THREADS
  }
  Py_INCREF(Py_None);
  ret = Py_None;
done:
  for (Py_ssize_t i = 0; i < got; ++i)
    if (views[i].obj) PyBuffer_Release(&views[i]);
  free(views);
  free(items);
  Py_DECREF(fast);
  PyBuffer_Release(&dst);
  return ret;
}

static PyMethodDef methods[] = {
    {"stage_rows", stage_rows, METH_VARARGS, "batch of host arrays -> one staging buffer (threads)"},
    {"narrow_u32", narrow_u32, METH_VARARGS, "4/8-byte words -> u32 buffer (truncating)"},
#ifdef ZPIR_FAST_DIGITS
    {"digits_into", digits_into, METH_VARARGS, "ints -> raw 30-bit digits written into a buffer"},
    {"ints_from_digits", ints_from_digits, METH_VARARGS, "30-bit digit rows -> list of ints"},
#endif
    {"ints_into", ints_into, METH_VARARGS, "ints -> u32 LE limbs written into a buffer"},
    {"ints_from", ints_from, METH_VARARGS, "u32 LE limbs -> list of ints"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_zpir_conv", NULL, -1, methods};

PyMODINIT_FUNC PyInit__zpir_conv(void) { return PyModule_Create(&mod); }
