// _tcflat: native flattening of a (TensorNetwork, ContractionTree) pair into
// the arrays of tc_plan_desc (include/tc.h).  Same output as the pure-Python
// paper_2006_15512_b200/flatten.py (which documents the format), but walks
// the Python objects through the C API: it runs on every public-API call and
// the Python loop cost ~27 ms on C2's 16k leaves / 16k internal nodes.
//
//   flatten(tensors, tree) -> (indices: list[Index], domain: bytes(int32),
//       leaf_idx_off: bytes(int64), leaf_idx: bytes(int32),
//       leaf_val_off: bytes(int64), leaf_val: bytes(float64),
//       left: bytes(int32), right: bytes(int32), root_slot: int)
//   flatten(tensors, tree, True): the same, but leaf_val holds one uint64
//       data address per tensor (no copy; the native FactorTree reads the
//       reference's dense 2^occ copy tensors in place) and a last element
//       keeps alive the arrays converted to float64 C order.
//
// Reads only n.tensors[k].indices / .values, index.id / .domain_size and
// node.tensor / .left / .right (reference network.py:83-124, tensor.py:18-62).
// Index identity is Index.id (tensor.py:29-33); leaf identity is the tensor
// object (network.py:143-148); slots follow serialize_plan (network.py:235-258):
// leaves in network order, then internal nodes in left-first postorder.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  char* p;
  size_t n, cap;
} Buf;

static int buf_put(Buf* b, const void* src, size_t len) {
  if (b->n + len > b->cap) {
    size_t c = b->cap ? b->cap * 2 : 4096;
    while (c < b->n + len) c *= 2;
    char* q = (char*)PyMem_Realloc(b->p, c);
    if (!q) {
      PyErr_NoMemory();
      return -1;
    }
    b->p = q;
    b->cap = c;
  }
  memcpy(b->p + b->n, src, len);
  b->n += len;
  return 0;
}

static PyObject* buf_bytes(Buf* b) { return PyBytes_FromStringAndSize(b->p ? b->p : "", (Py_ssize_t)b->n); }

// pointer -> int open-addressing map (leaf tensor object -> slot, tree node ->
// slot, Index object -> dense id); key and value share a 16-byte entry, so a
// probe touches one cache line
typedef struct {
  uintptr_t key;
  int64_t val;
} PmEnt;
typedef struct {
  PmEnt* e;
  size_t mask;
} PtrMap;

static int pm_init(PtrMap* m, size_t n) {
  size_t c = 16;
  while (c < 2 * n + 2) c <<= 1;
  m->e = (PmEnt*)PyMem_Calloc(c, sizeof(PmEnt));
  m->mask = c - 1;
  if (!m->e) {
    PyErr_NoMemory();
    return -1;
  }
  return 0;
}
static void pm_free(PtrMap* m) { PyMem_Free(m->e); }
// full-avalanche mix (murmur3 finalizer): the map masks the LOW bits, and object
// addresses share their low bits (fixed allocation strides), so a plain
// multiplicative hash clusters them into long linear-probe runs
static inline size_t pm_hash(uintptr_t k) {
  uint64_t x = (uint64_t)k;
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (size_t)x;
}
static void pm_set(PtrMap* m, uintptr_t k, int64_t v) {
  size_t h = pm_hash(k) & m->mask;
  while (m->e[h].key && m->e[h].key != k) h = (h + 1) & m->mask;
  m->e[h].key = k;
  m->e[h].val = v;
}
static int64_t pm_get(const PtrMap* m, uintptr_t k, int64_t dflt) {
  size_t h = pm_hash(k) & m->mask;
  while (m->e[h].key) {
    if (m->e[h].key == k) return m->e[h].val;
    h = (h + 1) & m->mask;
  }
  return dflt;
}

static PyObject *s_indices, *s_values, *s_id, *s_domain_size, *s_tensor, *s_left, *s_right;

// Attribute reads of __slots__ classes (this package's Tensor / Index /
// ContractionTree): the member descriptor's offset is looked up once per
// (type, name) and the slot read directly, the same value PyObject_GetAttr
// returns for a type with generic attribute access (a member descriptor is a
// data descriptor: it wins over any instance dict).  Other classes (the
// reference's dict-based dataclasses) take PyObject_GetAttr.
typedef struct {
  PyTypeObject* type;
  Py_ssize_t off;  // -1: not a plain object slot
} SlotCache;

static Py_ssize_t slot_offset(PyTypeObject* tp, PyObject* name) {
  if (tp->tp_getattro != PyObject_GenericGetAttr) return -1;
  PyObject* d = _PyType_Lookup(tp, name);  // borrowed
  if (!d || !Py_IS_TYPE(d, &PyMemberDescr_Type)) return -1;
  PyMemberDef* m = ((PyMemberDescrObject*)d)->d_member;
  return (m->type == Py_T_OBJECT_EX && !(m->flags & Py_AUDIT_READ)) ? m->offset : -1;
}

static inline PyObject* get_attr(PyObject* o, PyObject* name, SlotCache* c) {  // new reference
  PyTypeObject* tp = Py_TYPE(o);
  if (tp != c->type) {
    c->type = tp;
    c->off = slot_offset(tp, name);
  }
  if (c->off >= 0) {
    PyObject* v = *(PyObject**)((char*)o + c->off);
    if (v) {
      Py_INCREF(v);
      return v;
    }
  }
  return PyObject_GetAttr(o, name);  // unset slot: the AttributeError as usual
}

// append the row-major float64 contents of `values` to vals; returns entries or -1
static Py_ssize_t put_values(Buf* vals, PyObject* values) {
  // fast path: an aligned, C-contiguous float64 ndarray (what Tensor holds)
  if (PyArray_Check(values)) {
    PyArrayObject* arr = (PyArrayObject*)values;
    if (PyArray_TYPE(arr) == NPY_DOUBLE && PyArray_IS_C_CONTIGUOUS(arr) && PyArray_ISNOTSWAPPED(arr)) {
      const Py_ssize_t n = PyArray_SIZE(arr);
      return buf_put(vals, PyArray_DATA(arr), (size_t)n * 8) == 0 ? n : -1;
    }
  }
  Py_buffer v;
  if (PyObject_GetBuffer(values, &v, PyBUF_STRIDES | PyBUF_FORMAT) == 0) {
    const char* f = v.format ? v.format : "B";
    if (f[0] == '<' || f[0] == '=' || f[0] == '@') f++;
    if (v.itemsize == 8 && f[0] == 'd' && f[1] == 0) {
      Py_ssize_t n = v.len / 8;
      int rc;
      if (PyBuffer_IsContiguous(&v, 'C')) {
        rc = buf_put(vals, v.buf, (size_t)v.len);
      } else {
        size_t at = vals->n;
        double zero = 0.0;
        rc = 0;
        for (Py_ssize_t i = 0; i < n && rc == 0; ++i) rc = buf_put(vals, &zero, 8);
        if (rc == 0) rc = PyBuffer_ToContiguous(vals->p + at, &v, v.len, 'C');
      }
      PyBuffer_Release(&v);
      return rc == 0 ? n : -1;
    }
    PyBuffer_Release(&v);
  } else {
    PyErr_Clear();
  }
  // anything else (other dtype, non-buffer): let numpy convert
  PyObject* np = PyImport_ImportModule("numpy");
  if (!np) return -1;
  PyObject* arr = PyObject_CallMethod(np, "ascontiguousarray", "Os", values, "float64");
  Py_DECREF(np);
  if (!arr) return -1;
  Py_ssize_t n = put_values(vals, arr);
  Py_DECREF(arr);
  return n;
}

// pointer mode: append the address of `values`' float64 C-contiguous data
// (converted with numpy.ascontiguousarray when needed; the converted array is
// kept alive in `keep`); returns the entry count or -1
static Py_ssize_t put_pointer(Buf* ptrs, PyObject* keep, PyObject* values) {
  PyObject* arr = values;
  Py_INCREF(arr);
  if (!(PyArray_Check(arr) && PyArray_TYPE((PyArrayObject*)arr) == NPY_DOUBLE &&
        PyArray_IS_C_CONTIGUOUS((PyArrayObject*)arr) && PyArray_ISNOTSWAPPED((PyArrayObject*)arr) &&
        PyArray_ISALIGNED((PyArrayObject*)arr))) {
    PyObject* np = PyImport_ImportModule("numpy");
    Py_DECREF(arr);
    if (!np) return -1;
    arr = PyObject_CallMethod(np, "ascontiguousarray", "Os", values, "float64");
    Py_DECREF(np);
    if (!arr) return -1;
    if (PyList_Append(keep, arr) < 0) {
      Py_DECREF(arr);
      return -1;
    }
  }
  const Py_ssize_t n = PyArray_SIZE((PyArrayObject*)arr);
  const uint64_t ptr = (uint64_t)(uintptr_t)PyArray_DATA((PyArrayObject*)arr);
  Py_DECREF(arr);  // owned by the tensor or by `keep`
  return buf_put(ptrs, &ptr, 8) == 0 ? n : -1;
}

static PyObject* flatten(PyObject* self, PyObject* args) {
  PyObject *tensors_in, *tree;
  int ptr_mode = 0;
  if (!PyArg_ParseTuple(args, "OO|p", &tensors_in, &tree, &ptr_mode)) return NULL;
  PyObject* keep = ptr_mode ? PyList_New(0) : NULL;
  if (ptr_mode && !keep) return NULL;
  SlotCache c_indices = {0}, c_values = {0}, c_domain = {0}, c_id = {0}, c_tensor = {0}, c_left = {0}, c_right = {0};
  PyObject* tensors = PySequence_Fast(tensors_in, "n.tensors must be a sequence");
  if (!tensors) return NULL;
  const Py_ssize_t nl = PySequence_Fast_GET_SIZE(tensors);
  PyObject** tv = PySequence_Fast_ITEMS(tensors);

  PyObject* result = NULL;
  PyObject* indices = PyList_New(0);
  PyObject* pos = PyDict_New();  // Index.id -> dense id
  Buf dom = {0}, ioff = {0}, iarr = {0}, voff = {0}, vals = {0}, lft = {0}, rgt = {0};
  PtrMap leaf = {0}, ixp = {0};
  size_t pm_size = 0, pm_cap = 4096;
  int32_t* occ = NULL;  // occurrences of each distinct Index object
  size_t occ_cap = 0;
  if (!indices || !pos) goto done;
  if (pm_init(&leaf, (size_t)nl) < 0 || pm_init(&ixp, pm_cap) < 0) goto done;

  int64_t off = 0, voffv = 0;
  if (buf_put(&ioff, &off, 8) < 0 || buf_put(&voff, &voffv, 8) < 0) goto done;
  for (Py_ssize_t k = 0; k < nl; ++k) {
    PyObject* ten = tv[k];
    pm_set(&leaf, (uintptr_t)ten, k);
    PyObject* inds = get_attr(ten, s_indices, &c_indices);
    if (!inds) goto done;
    PyObject* fi = PySequence_Fast(inds, "tensor.indices must be a sequence");
    Py_DECREF(inds);
    if (!fi) goto done;
    const Py_ssize_t r = PySequence_Fast_GET_SIZE(fi);
    PyObject** iv = PySequence_Fast_ITEMS(fi);
    for (Py_ssize_t q = 0; q < r; ++q) {
      PyObject* ix = iv[q];
      // identity by object first (a bond's two tensors usually share the Index
      // object); equal-by-id distinct objects are merged after the loop
      int64_t known = pm_get(&ixp, (uintptr_t)ix, -1);
      int32_t di;
      if (known >= 0) {
        di = (int32_t)known;
        occ[di]++;
      } else {
        di = (int32_t)PyList_GET_SIZE(indices);
        PyObject* ds = get_attr(ix, s_domain_size, &c_domain);
        long dsz = ds ? PyLong_AsLong(ds) : -1;
        Py_XDECREF(ds);
        int32_t dsz32 = (int32_t)dsz;
        if (dsz < 0 || PyList_Append(indices, ix) < 0 || buf_put(&dom, &dsz32, 4) < 0) {
          if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "bad index domain_size");
          Py_DECREF(fi);
          goto done;
        }
        if (pm_size >= pm_cap) {  // grow the pointer map (rehash); `indices` owns the keys
          PtrMap bigger;
          if (pm_init(&bigger, 2 * pm_cap) < 0) {
            Py_DECREF(fi);
            goto done;
          }
          for (size_t h = 0; h <= ixp.mask; ++h)
            if (ixp.e[h].key) pm_set(&bigger, ixp.e[h].key, ixp.e[h].val);
          pm_free(&ixp);
          ixp = bigger;
          pm_cap *= 2;
        }
        pm_set(&ixp, (uintptr_t)ix, di);
        pm_size++;
        if ((size_t)di >= occ_cap) {
          occ_cap = occ_cap ? 2 * occ_cap : 4096;
          int32_t* q2 = (int32_t*)PyMem_Realloc(occ, occ_cap * sizeof(int32_t));
          if (!q2) {
            PyErr_NoMemory();
            Py_DECREF(fi);
            goto done;
          }
          occ = q2;
        }
        occ[di] = 1;
      }
      if (buf_put(&iarr, &di, 4) < 0) {
        Py_DECREF(fi);
        goto done;
      }
    }
    Py_DECREF(fi);
    off += r;
    if (buf_put(&ioff, &off, 8) < 0) goto done;
    PyObject* values = get_attr(ten, s_values, &c_values);
    if (!values) goto done;
    Py_ssize_t nv = ptr_mode ? put_pointer(&vals, keep, values) : put_values(&vals, values);
    Py_DECREF(values);
    if (nv < 0) goto done;
    voffv += nv;
    if (buf_put(&voff, &voffv, 8) < 0) goto done;
  }

  // Index identity is Index.id (tensor.py:29-33).  Objects seen twice are
  // bonds already; the singly-seen ones (free indices, or a bond whose two
  // tensors hold distinct but equal Index objects) are matched by id, and
  // later duplicates are folded into the first, keeping first-appearance order.
  {
    const Py_ssize_t nu = PyList_GET_SIZE(indices);
    int32_t* remap = (int32_t*)PyMem_Malloc((size_t)(nu ? nu : 1) * sizeof(int32_t));
    if (!remap) {
      PyErr_NoMemory();
      goto done;
    }
    int merged = 0;
    for (Py_ssize_t u = 0; u < nu; ++u) {
      remap[u] = (int32_t)u;
      if (occ[u] != 1) continue;
      PyObject* key = get_attr(PyList_GET_ITEM(indices, u), s_id, &c_id);
      if (!key) {
        PyMem_Free(remap);
        goto done;
      }
      PyObject* d = PyDict_GetItemWithError(pos, key);
      if (d) {
        remap[u] = (int32_t)PyLong_AsLong(d);
        merged = 1;
      } else if (!PyErr_Occurred()) {
        PyObject* dv = PyLong_FromSsize_t(u);
        if (!dv || PyDict_SetItem(pos, key, dv) < 0) {
          Py_XDECREF(dv);
          Py_DECREF(key);
          PyMem_Free(remap);
          goto done;
        }
        Py_DECREF(dv);
      }
      Py_DECREF(key);
      if (PyErr_Occurred()) {
        PyMem_Free(remap);
        goto done;
      }
    }
    if (merged) {  // compact: dense ids in first-appearance order of each id
      int32_t* dense = (int32_t*)PyMem_Malloc((size_t)nu * sizeof(int32_t));
      PyObject* kept = PyList_New(0);
      Buf dom2 = {0};
      int32_t nxt = 0;
      int ok = dense && kept;
      for (Py_ssize_t u = 0; u < nu && ok; ++u) {
        if (remap[u] == (int32_t)u) {
          dense[u] = nxt++;
          ok = PyList_Append(kept, PyList_GET_ITEM(indices, u)) == 0 &&
               buf_put(&dom2, ((int32_t*)dom.p) + u, 4) == 0;
        } else {
          dense[u] = dense[remap[u]];
        }
      }
      if (ok) {
        int32_t* ia = (int32_t*)iarr.p;
        for (size_t q = 0; q < iarr.n / 4; ++q) ia[q] = dense[ia[q]];
        Py_DECREF(indices);
        indices = kept;
        kept = NULL;
        PyMem_Free(dom.p);
        dom = dom2;
        dom2.p = NULL;
      }
      Py_XDECREF(kept);
      PyMem_Free(dom2.p);
      PyMem_Free(dense);
      if (!ok) {
        if (!PyErr_Occurred()) PyErr_NoMemory();
        PyMem_Free(remap);
        goto done;
      }
    }
    PyMem_Free(remap);
  }

  // right-first preorder, reversed = left-first postorder (network.py:114-124).
  // Pass 1 reads each node's attributes once and records its parent; pass 2
  // (reverse order: children before parents) numbers the internal nodes.
  {
    typedef struct {
      PyObject* node;  // owned
      int64_t parent;  // seq index of the parent, -1 for the root
      int64_t kid[2];  // slots of left/right (internal nodes)
      int64_t leaf;    // leaf slot (-1: not in the network), or -2: internal
      int side;        // 0: left child, 1: right child
    } Ent;
    typedef struct {
      PyObject* node;
      int64_t parent;
      int side;
    } Pend;
    size_t cap = 1024, sp = 0, ns = 0, scap = 1024;
    Pend* stk = (Pend*)PyMem_Malloc(cap * sizeof(Pend));
    Ent* ent = (Ent*)PyMem_Malloc(scap * sizeof(Ent));
    if (!stk || !ent) {
      PyMem_Free(stk);
      PyMem_Free(ent);
      PyErr_NoMemory();
      goto done;
    }
    Py_INCREF(tree);
    stk[sp++] = (Pend){tree, -1, 0};  // owned references on the stack and in ent
    while (sp) {
      Pend pd = stk[--sp];
      if (ns == scap) {
        scap *= 2;
        Ent* q = (Ent*)PyMem_Realloc(ent, scap * sizeof(Ent));
        if (!q) {
          Py_DECREF(pd.node);
          PyErr_NoMemory();
          goto tree_fail;
        }
        ent = q;
      }
      Ent* e = &ent[ns++];
      e->node = pd.node;
      e->parent = pd.parent;
      e->side = pd.side;
      e->kid[0] = e->kid[1] = -1;
      PyObject* t = get_attr(pd.node, s_tensor, &c_tensor);
      if (!t) goto tree_fail;
      if (t != Py_None) {
        e->leaf = pm_get(&leaf, (uintptr_t)t, -1);
        Py_DECREF(t);
        continue;
      }
      Py_DECREF(t);
      e->leaf = -2;
      if (sp + 2 > cap) {
        cap *= 2;
        Pend* q = (Pend*)PyMem_Realloc(stk, cap * sizeof(Pend));
        if (!q) {
          PyErr_NoMemory();
          goto tree_fail;
        }
        stk = q;
      }
      PyObject* l = get_attr(pd.node, s_left, &c_left);
      if (!l) goto tree_fail;
      stk[sp++] = (Pend){l, (int64_t)(ns - 1), 0};
      PyObject* r = get_attr(pd.node, s_right, &c_right);
      if (!r) goto tree_fail;
      stk[sp++] = (Pend){r, (int64_t)(ns - 1), 1};
    }
    {
      int64_t nxt = nl, root_slot = -1;
      for (size_t q = ns; q-- > 0;) {
        Ent* e = &ent[q];
        int64_t s;
        if (e->leaf != -2) {
          s = e->leaf;
        } else {
          int32_t ls = (int32_t)e->kid[0], rs = (int32_t)e->kid[1];
          if (buf_put(&lft, &ls, 4) < 0 || buf_put(&rgt, &rs, 4) < 0) goto tree_fail;
          s = nxt++;
        }
        if (e->parent >= 0) ent[e->parent].kid[e->side] = s;
        else root_slot = s;
      }
      result = ptr_mode ? Py_BuildValue("(ONNNNNNNLO)", indices, buf_bytes(&dom), buf_bytes(&ioff), buf_bytes(&iarr),
                                        buf_bytes(&voff), buf_bytes(&vals), buf_bytes(&lft), buf_bytes(&rgt),
                                        (long long)root_slot, keep)
                        : Py_BuildValue("(ONNNNNNNL)", indices, buf_bytes(&dom), buf_bytes(&ioff), buf_bytes(&iarr),
                                        buf_bytes(&voff), buf_bytes(&vals), buf_bytes(&lft), buf_bytes(&rgt),
                                        (long long)root_slot);
    }
  tree_fail:
    for (size_t q = 0; q < ns; ++q) Py_DECREF(ent[q].node);
    for (size_t q = 0; q < sp; ++q) Py_DECREF(stk[q].node);
    PyMem_Free(stk);
    PyMem_Free(ent);
  }

done:
  pm_free(&leaf);
  pm_free(&ixp);
  PyMem_Free(occ);
  PyMem_Free(dom.p);
  PyMem_Free(ioff.p);
  PyMem_Free(iarr.p);
  PyMem_Free(voff.p);
  PyMem_Free(vals.p);
  PyMem_Free(lft.p);
  PyMem_Free(rgt.p);
  Py_XDECREF(indices);
  Py_XDECREF(pos);
  Py_XDECREF(keep);
  Py_DECREF(tensors);
  return result;
}

// positions(indices, queries) -> list[int]: for each query Index, the position
// of the first entry of `indices` that is the same object, else the first with
// an equal .id (Index equality, tensor.py:29-33), else -1.  One pointer scan
// of the (long) index table instead of a dict over all of it.
static PyObject* positions(PyObject* self, PyObject* args) {
  PyObject *indices_in, *queries_in;
  if (!PyArg_ParseTuple(args, "OO", &indices_in, &queries_in)) return NULL;
  PyObject* ind = PySequence_Fast(indices_in, "indices must be a sequence");
  if (!ind) return NULL;
  PyObject* qs = PySequence_Fast(queries_in, "queries must be a sequence");
  if (!qs) {
    Py_DECREF(ind);
    return NULL;
  }
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(ind), m = PySequence_Fast_GET_SIZE(qs);
  PyObject** iv = PySequence_Fast_ITEMS(ind);
  PyObject** qv = PySequence_Fast_ITEMS(qs);
  PyObject* out = PyList_New(m);
  Py_ssize_t* pos = (Py_ssize_t*)PyMem_Malloc((size_t)(m ? m : 1) * sizeof(Py_ssize_t));
  PtrMap qm = {0};
  if (!out || !pos || pm_init(&qm, (size_t)m) < 0) goto fail;
  for (Py_ssize_t q = 0; q < m; ++q) pos[q] = -1;
  for (Py_ssize_t q = m; q-- > 0;) pm_set(&qm, (uintptr_t)qv[q], q);  // first listed query wins per object
  {
    Py_ssize_t left = m;
    for (Py_ssize_t k = 0; k < n && left; ++k) {
      const int64_t q = pm_get(&qm, (uintptr_t)iv[k], -1);
      if (q < 0) continue;
      for (Py_ssize_t r = 0; r < m; ++r)  // every query holding this object
        if (qv[r] == iv[k] && pos[r] < 0) pos[r] = k, --left;
    }
    // queries that are not the network's own objects: match by id
    for (Py_ssize_t r = 0; r < m; ++r) {
      if (pos[r] >= 0) continue;
      PyObject* want = PyObject_GetAttr(qv[r], s_id);
      if (!want) goto fail;
      for (Py_ssize_t k = 0; k < n; ++k) {
        PyObject* have = PyObject_GetAttr(iv[k], s_id);
        if (!have) {
          Py_DECREF(want);
          goto fail;
        }
        const int eq = PyObject_RichCompareBool(have, want, Py_EQ);
        Py_DECREF(have);
        if (eq < 0) {
          Py_DECREF(want);
          goto fail;
        }
        if (eq) {
          pos[r] = k;
          break;
        }
      }
      Py_DECREF(want);
    }
  }
  for (Py_ssize_t q = 0; q < m; ++q) PyList_SET_ITEM(out, q, PyLong_FromSsize_t(pos[q]));
  pm_free(&qm);
  PyMem_Free(pos);
  Py_DECREF(ind);
  Py_DECREF(qs);
  return out;
fail:
  pm_free(&qm);
  PyMem_Free(pos);
  Py_XDECREF(out);
  Py_DECREF(ind);
  Py_DECREF(qs);
  if (!PyErr_Occurred()) PyErr_NoMemory();
  return NULL;
}

static PyMethodDef methods[] = {
    {"positions", positions, METH_VARARGS, "positions(indices, queries) -> first position of each query (identity, then id)"},
    {"flatten", flatten, METH_VARARGS, "flatten(tensors, tree) -> plan arrays (see paper_2006_15512_b200/flatten.py)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_tcflat", NULL, -1, methods};

PyMODINIT_FUNC PyInit__tcflat(void) {
  import_array();
  s_indices = PyUnicode_InternFromString("indices");
  s_values = PyUnicode_InternFromString("values");
  s_id = PyUnicode_InternFromString("id");
  s_domain_size = PyUnicode_InternFromString("domain_size");
  s_tensor = PyUnicode_InternFromString("tensor");
  s_left = PyUnicode_InternFromString("left");
  s_right = PyUnicode_InternFromString("right");
  return PyModule_Create(&mod);
}
