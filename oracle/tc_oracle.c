/*
 * tc_oracle.c — TEST INFRASTRUCTURE ONLY.  A plain-C, single-threaded CPU
 * restatement of the reference execution path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker.
 * Nothing in paper_2006_15512_b200/ links, imports or calls this file.
 *
 * Restates (all paths relative to /root/reference):
 *   contract_pair        pkg/src/tensorcount/tensor.py:96-108
 *       shared = indices of a that are in b (a's order); kept_a ++ kept_b;
 *       row-major output; sum over shared assignments (row-major odometer).
 *   add (slice sum)      pkg/src/tensorcount/tensor.py:111-115
 *   slice_tensor         pkg/src/tensorcount/tensor.py:118-125
 *   _slice_plan          pkg/src/tensorcount/slicing.py:30-41
 *   mem_cost             pkg/src/tensorcount/slicing.py:52-67
 *   choose_slice_index   pkg/src/tensorcount/slicing.py:70-79
 *   _execute_tracked     pkg/src/tensorcount/slicing.py:91-109
 *   sliced_execute       pkg/src/tensorcount/slicing.py:112-146
 *
 * Pinned against fixtures produced by the reference itself
 * (tests/golden/make_golden.py) — see tests/test_oracle.py.
 *
 * Plan format: the same flattened arrays as include/tc.h's tc_plan_desc.
 * Sizes use unsigned __int128 (the reference uses Python ints).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
  int32_t ni, nl, nn, root;
  const int32_t* dom;
  const int32_t* srank;
  const int64_t* lidx_off;
  const int32_t* lidx;
  const int64_t* lval_off;
  const double* lval;
  const int32_t* left;
  const int32_t* right;
} oplan;

/* a dense tensor: rank, index ids (row-major order), values */
typedef struct {
  int rank;
  int32_t* idx;
  double* val;
  int64_t size;
} oten;

static int has(const int32_t* ids, int n, int32_t x) {
  for (int k = 0; k < n; ++k)
    if (ids[k] == x) return 1;
  return 0;
}

/* ---- symbolic index sets (network.py:166-175), as sorted-free lists ---- */
static int32_t** g_sets;
static int* g_nset;

static void build_sets(const oplan* p) {
  int S = p->nl + p->nn;
  g_sets = (int32_t**)calloc(S, sizeof(int32_t*));
  g_nset = (int*)calloc(S, sizeof(int));
  for (int l = 0; l < p->nl; ++l) {
    int n = (int)(p->lidx_off[l + 1] - p->lidx_off[l]);
    g_sets[l] = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    memcpy(g_sets[l], p->lidx + p->lidx_off[l], sizeof(int32_t) * n);
    g_nset[l] = n;
  }
  for (int k = 0; k < p->nn; ++k) {
    int v = p->nl + k, a = p->left[k], b = p->right[k];
    g_sets[v] = (int32_t*)malloc(sizeof(int32_t) * (g_nset[a] + g_nset[b] + 1));
    int n = 0;
    for (int q = 0; q < g_nset[a]; ++q)
      if (!has(g_sets[b], g_nset[b], g_sets[a][q])) g_sets[v][n++] = g_sets[a][q];
    for (int q = 0; q < g_nset[b]; ++q)
      if (!has(g_sets[a], g_nset[a], g_sets[b][q])) g_sets[v][n++] = g_sets[b][q];
    g_nset[v] = n;
  }
}

static void free_sets(const oplan* p) {
  int S = p->nl + p->nn;
  for (int s = 0; s < S; ++s) free(g_sets[s]);
  free(g_sets);
  free(g_nset);
}

static u128 set_bytes(const oplan* p, int s, const char* drop) {
  u128 out = 8;
  for (int q = 0; q < g_nset[s]; ++q)
    if (!drop[g_sets[s][q]]) out *= (u128)p->dom[g_sets[s][q]];
  return out;
}

/* slicing.py:52-67 — postorder (children precede parents in slot order) */
static u128 mem_cost_(const oplan* p, const char* drop) {
  int S = p->nl + p->nn;
  u128* peak = (u128*)malloc(sizeof(u128) * S);
  u128* live = (u128*)malloc(sizeof(u128) * S);
  for (int l = 0; l < p->nl; ++l) peak[l] = live[l] = set_bytes(p, l, drop);
  for (int k = 0; k < p->nn; ++k) {
    int v = p->nl + k, a = p->left[k], b = p->right[k];
    u128 out = set_bytes(p, v, drop);
    u128 x = peak[a], y = live[a] + peak[b], z = live[a] + live[b] + out;
    u128 m = x > y ? x : y;
    peak[v] = m > z ? m : z;
    live[v] = out;
  }
  u128 r = peak[p->root];
  free(peak);
  free(live);
  return r;
}

void oracle_mem_cost(const oplan* p, const int32_t* drop_ids, int n_drop, uint64_t* lo, uint64_t* hi) {
  char* drop = (char*)calloc(p->ni + 1, 1);
  for (int k = 0; k < n_drop; ++k) drop[drop_ids[k]] = 1;
  build_sets(p);
  u128 r = mem_cost_(p, drop);
  free_sets(p);
  free(drop);
  *lo = (uint64_t)r;
  *hi = (uint64_t)(r >> 64);
}

/* bonds = indices occurring in two leaves */
static char* bond_mask(const oplan* p) {
  int* occ = (int*)calloc(p->ni + 1, sizeof(int));
  for (int64_t q = 0; q < p->lidx_off[p->nl]; ++q) occ[p->lidx[q]]++;
  char* m = (char*)calloc(p->ni + 1, 1);
  for (int i = 0; i < p->ni; ++i) m[i] = occ[i] == 2;
  free(occ);
  return m;
}

/* slicing.py:70-79: min over candidates (sorted by sort_key) of (cost, key) */
static int choose_(const oplan* p, char* already, const char* bond) {
  int best = -1;
  u128 bc = 0;
  for (int i = 0; i < p->ni; ++i) {
    if (!bond[i] || already[i]) continue;
    already[i] = 1;
    u128 c = mem_cost_(p, already);
    already[i] = 0;
    if (best < 0 || c < bc || (c == bc && p->srank[i] < p->srank[best])) {
      best = i;
      bc = c;
    }
  }
  return best;
}

int oracle_choose_slice_index(const oplan* p, const int32_t* already_ids, int n_already) {
  char* already = (char*)calloc(p->ni + 1, 1);
  for (int k = 0; k < n_already; ++k) already[already_ids[k]] = 1;
  char* bond = bond_mask(p);
  build_sets(p);
  int r = choose_(p, already, bond);
  free_sets(p);
  free(bond);
  free(already);
  return r;
}

/* ---- numeric path ------------------------------------------------------ */
static int64_t dsize(const oplan* p, const int32_t* ids, int n) {
  int64_t s = 1;
  for (int q = 0; q < n; ++q) s *= p->dom[ids[q]];
  return s;
}

/* tensor.py:96-108 */
static oten contract_pair_(const oplan* p, const oten* a, const oten* b) {
  int32_t sh[128], ka[128], kb[128];
  int ns = 0, na = 0, nb = 0;
  for (int q = 0; q < a->rank; ++q) {
    if (has(b->idx, b->rank, a->idx[q])) sh[ns++] = a->idx[q];
    else ka[na++] = a->idx[q];
  }
  for (int q = 0; q < b->rank; ++q)
    if (!has(a->idx, a->rank, b->idx[q])) kb[nb++] = b->idx[q];
  oten c;
  c.rank = na + nb;
  c.idx = (int32_t*)malloc(sizeof(int32_t) * (c.rank + 1));
  memcpy(c.idx, ka, sizeof(int32_t) * na);
  memcpy(c.idx + na, kb, sizeof(int32_t) * nb);
  c.size = dsize(p, c.idx, c.rank);
  c.val = (double*)calloc((size_t)c.size + 1, sizeof(double));
  /* row-major strides of a and b per index id */
  int64_t sa[128], sb[128], st = 1;
  for (int q = a->rank - 1; q >= 0; --q) {
    sa[q] = st;
    st *= p->dom[a->idx[q]];
  }
  st = 1;
  for (int q = b->rank - 1; q >= 0; --q) {
    sb[q] = st;
    st *= p->dom[b->idx[q]];
  }
  int64_t ssize = dsize(p, sh, ns);
  int digit[128];
  for (int64_t o = 0; o < c.size; ++o) {
    /* decode o (row-major over kept_a ++ kept_b) */
    int64_t rem = o, oa = 0, ob = 0;
    for (int q = c.rank - 1; q >= 0; --q) {
      int32_t i = c.idx[q];
      int64_t d = rem % p->dom[i];
      rem /= p->dom[i];
      for (int r = 0; r < a->rank; ++r)
        if (a->idx[r] == i) oa += d * sa[r];
      for (int r = 0; r < b->rank; ++r)
        if (b->idx[r] == i) ob += d * sb[r];
    }
    double total = 0.0;
    for (int q = 0; q < ns; ++q) digit[q] = 0;
    for (int64_t s = 0; s < ssize; ++s) {
      int64_t xa = oa, xb = ob;
      for (int q = 0; q < ns; ++q) {
        for (int r = 0; r < a->rank; ++r)
          if (a->idx[r] == sh[q]) xa += digit[q] * sa[r];
        for (int r = 0; r < b->rank; ++r)
          if (b->idx[r] == sh[q]) xb += digit[q] * sb[r];
      }
      total += a->val[xa] * b->val[xb];
      for (int q = ns - 1; q >= 0; --q) { /* row-major odometer, last fastest */
        if (++digit[q] < p->dom[sh[q]]) break;
        digit[q] = 0;
      }
    }
    c.val[o] = total;
  }
  return c;
}

/* tensor.py:118-125 on leaf l with assignment vals[] for chosen ids */
static oten slice_leaf(const oplan* p, int l, const char* chosen_mask, const int* value_of) {
  oten t;
  int n = (int)(p->lidx_off[l + 1] - p->lidx_off[l]);
  const int32_t* ids = p->lidx + p->lidx_off[l];
  const double* v = p->lval + p->lval_off[l];
  int64_t stride[128], st = 1;
  for (int q = n - 1; q >= 0; --q) {
    stride[q] = st;
    st *= p->dom[ids[q]];
  }
  t.idx = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  t.rank = 0;
  int64_t base = 0;
  for (int q = 0; q < n; ++q) {
    if (chosen_mask[ids[q]]) base += value_of[ids[q]] * stride[q];
    else t.idx[t.rank++] = ids[q];
  }
  t.size = dsize(p, t.idx, t.rank);
  t.val = (double*)malloc(sizeof(double) * ((size_t)t.size + 1));
  for (int64_t e = 0; e < t.size; ++e) {
    int64_t rem = e, src = base;
    for (int q = n - 1; q >= 0; --q) {
      if (chosen_mask[ids[q]]) continue;
      int64_t d = rem % p->dom[ids[q]];
      rem /= p->dom[ids[q]];
      src += d * stride[q];
    }
    t.val[e] = v[src];
  }
  return t;
}

/* slicing.py:91-109 on the (sliced) plan; returns the root tensor; *peak */
static oten execute_tracked_(const oplan* p, const char* chosen_mask, const int* value_of, u128* peak_out) {
  int S = p->nl + p->nn;
  oten* res = (oten*)calloc(S, sizeof(oten));
  /* full postorder sequence with leaves (network.py:114-124) */
  int* seq = (int*)malloc(sizeof(int) * S);
  int* st = (int*)malloc(sizeof(int) * S);
  int ns = 0, top = 0;
  st[top++] = p->root;
  while (top) {
    int v = st[--top];
    seq[ns++] = v;
    if (v >= p->nl) {
      st[top++] = p->left[v - p->nl];
      st[top++] = p->right[v - p->nl];
    }
  }
  u128 live = 0, peak = 0;
  for (int q = ns - 1; q >= 0; --q) {
    int v = seq[q];
    if (v < p->nl) {
      res[v] = slice_leaf(p, v, chosen_mask, value_of);
      live += (u128)res[v].size * 8;
    } else {
      int a = p->left[v - p->nl], b = p->right[v - p->nl];
      res[v] = contract_pair_(p, &res[a], &res[b]);
      live += (u128)res[v].size * 8;
      if (live > peak) peak = live;
      live -= (u128)(res[a].size + res[b].size) * 8;
      free(res[a].idx);
      free(res[a].val);
      free(res[b].idx);
      free(res[b].val);
    }
    if (live > peak) peak = live;
  }
  oten r = res[p->root];
  free(res);
  free(seq);
  free(st);
  *peak_out = peak;
  return r;
}

/*
 * slicing.py:112-146.  mode: 0 = no budget, 1 = greedy to `budget`,
 * 2 = explicit slice ids.  Returns 0 ok, 3 budget infeasible.
 * out_idx/out_val receive the result (reference index order, row-major).
 */
int oracle_sliced_execute(const oplan* p, int mode, int64_t budget, const int32_t* ids, int n_ids,
                          double* out_val, int64_t out_cap, int32_t* out_idx, int* out_rank,
                          int32_t* chosen, int* n_chosen, uint64_t* est_lo, uint64_t* est_hi,
                          uint64_t* peak_lo, uint64_t* peak_hi, int64_t* num_slices) {
  char* mask = (char*)calloc(p->ni + 1, 1);
  char* bond = bond_mask(p);
  build_sets(p);
  int nc = 0;
  if (mode == 1) {
    while (budget < 0 || mem_cost_(p, mask) > (u128)budget) {
      int pick = choose_(p, mask, bond);
      if (pick < 0) {
        free_sets(p);
        free(bond);
        free(mask);
        *n_chosen = nc;
        return 3;
      }
      chosen[nc++] = pick;
      mask[pick] = 1;
    }
  } else if (mode == 2) {
    for (int k = 0; k < n_ids; ++k) {
      chosen[nc++] = ids[k];
      mask[ids[k]] = 1;
    }
  }
  *n_chosen = nc;
  u128 est = mem_cost_(p, mask);
  *est_lo = (uint64_t)est;
  *est_hi = (uint64_t)(est >> 64);
  int* value_of = (int*)calloc(p->ni + 1, sizeof(int));
  int64_t nsl = 1;
  for (int k = 0; k < nc; ++k) nsl *= p->dom[chosen[k]];
  *num_slices = nsl;
  u128 peak = 0;
  oten total = {0, 0, 0, 0};
  for (int64_t s = 0; s < nsl; ++s) { /* itertools.product order: first chosen slowest */
    int64_t rem = s;
    for (int k = nc - 1; k >= 0; --k) {
      value_of[chosen[k]] = (int)(rem % p->dom[chosen[k]]);
      rem /= p->dom[chosen[k]];
    }
    u128 pk;
    oten part = execute_tracked_(p, mask, value_of, &pk);
    if (pk > peak) peak = pk;
    if (s == 0) {
      total = part;
    } else { /* tensor.py:111-115 (same index order every slice) */
      for (int64_t e = 0; e < total.size; ++e) total.val[e] = total.val[e] + part.val[e];
      free(part.idx);
      free(part.val);
    }
  }
  *peak_lo = (uint64_t)peak;
  *peak_hi = (uint64_t)(peak >> 64);
  *out_rank = total.rank;
  for (int q = 0; q < total.rank; ++q) out_idx[q] = total.idx[q];
  for (int64_t e = 0; e < total.size && e < out_cap; ++e) out_val[e] = total.val[e];
  free(total.idx);
  free(total.val);
  free(value_of);
  free_sets(p);
  free(bond);
  free(mask);
  return 0;
}
