/* TEST INFRASTRUCTURE — exact weighted model count of a CNF by a clause-frontier
 * dynamic program.  Used only by tests/, tools/make_golden_sliced.py and the
 * bench's parity record as an independent anchor for counts the reference
 * cannot produce on this hardware (its dense per-slice working set exceeds host
 * RAM at the C3-C5 sizes).  Never linked into the product (libtc).
 *
 * What it restates: the reference's own count oracle `brute_force_count`
 * (pkg/src/tensorcount/formula.py:183-215): WMC = sum over all assignments that
 * satisfy every clause (clause_satisfied, formula.py:179-180) of the product of
 * the per-variable weight pairs (WeightFunction.pair, formula.py:70-71, default
 * (1,1)).  The tensor network built by reduce_formula (reduction.py:80-100)
 * contracts to exactly this number, which is what every reference test of the
 * count checks (test_acceptance.py:75-79, test_driver.py:150-160).
 *
 * Instead of 2^n enumeration the sum is evaluated variable by variable
 * (1..n): a state is the set of *pending* clauses (first variable assigned,
 * last variable not yet) that are already satisfied; assigning v ORs in the
 * clauses v satisfies, and a clause whose last variable is v must be satisfied
 * when v is assigned.  Assignments with equal states have identical futures, so
 * their weights are summed.  This is exact up to FP64 summation order.
 *
 * Optional per-variable fixing (fix[v] in {0,1}) restricts the sum to
 * assignments with those values: the value of one slice of a network whose
 * sliced bonds are variable-copy bonds (factoring.py:194-206).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KW 4 /* 256 pending-clause bits */

typedef struct {
  uint64_t k[KW];
  double v;
  int used;
} slot_t;

typedef struct {
  slot_t* s;
  size_t cap, n;
} table_t;

static uint64_t hkey(const uint64_t* k) {
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < KW; ++i) {
    h ^= k[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
  }
  return h ^ (h >> 33);
}

static int t_init(table_t* t, size_t cap) {
  t->s = (slot_t*)calloc(cap, sizeof(slot_t));
  t->cap = cap;
  t->n = 0;
  return t->s ? 0 : -1;
}

static int t_add(table_t* t, const uint64_t* k, double v);

static int t_grow(table_t* t) {
  table_t u;
  if (t_init(&u, t->cap * 2)) return -1;
  for (size_t i = 0; i < t->cap; ++i)
    if (t->s[i].used) t_add(&u, t->s[i].k, t->s[i].v);
  free(t->s);
  *t = u;
  return 0;
}

static int t_add(table_t* t, const uint64_t* k, double v) {
  if ((t->n + 1) * 10 > t->cap * 7 && t_grow(t)) return -1;
  size_t i = hkey(k) & (t->cap - 1);
  for (;;) {
    slot_t* s = &t->s[i];
    if (!s->used) {
      memcpy(s->k, k, sizeof(s->k));
      s->v = v;
      s->used = 1;
      t->n++;
      return 0;
    }
    if (!memcmp(s->k, k, sizeof(s->k))) {
      s->v += v;
      return 0;
    }
    i = (i + 1) & (t->cap - 1);
  }
}

/* lits: concatenated clause literals, off[m+1]; w0/w1/fix indexed by variable
 * (1..n, entry 0 unused; fix[v] = -1 for a free variable).  Returns 0 on success,
 * -1 out of memory, -2 more than 256 pending clauses, -3 more than max_states
 * states.  *out = count, *peak = largest state table. */
int wmc_dp(int32_t n, int32_t m, const int32_t* lits, const int64_t* off, const double* w0, const double* w1,
           const int8_t* fix, int64_t max_states, double* out, int64_t* peak) {
  *out = 0.0;
  *peak = 1;
  for (int32_t c = 0; c < m; ++c)
    if (off[c + 1] == off[c]) return 0; /* empty clause: unsatisfiable */
  int32_t* first = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  int32_t* last = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  int32_t* bit = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  /* per-variable occurrence lists: (clause, sign) */
  int64_t* vo = (int64_t*)calloc((size_t)n + 2, sizeof(int64_t));
  int64_t total = off[m];
  int32_t* oc = (int32_t*)malloc(sizeof(int32_t) * (total ? total : 1));
  int8_t* os = (int8_t*)malloc(total ? total : 1);
  int rc = 0;
  table_t cur = {0}, nxt = {0};
  if (!first || !last || !bit || !vo || !oc || !os) { rc = -1; goto done; }
  for (int32_t c = 0; c < m; ++c) {
    int32_t lo = n + 1, hi = 0;
    for (int64_t j = off[c]; j < off[c + 1]; ++j) {
      int32_t v = abs(lits[j]);
      if (v < lo) lo = v;
      if (v > hi) hi = v;
      vo[v + 1]++;
    }
    first[c] = lo;
    last[c] = hi;
    bit[c] = -1;
  }
  for (int32_t v = 1; v <= n + 1; ++v) vo[v] += vo[v - 1];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 2));
    if (!fill) { rc = -1; goto done; }
    memcpy(fill, vo, sizeof(int64_t) * ((size_t)n + 2));
    for (int32_t c = 0; c < m; ++c)
      for (int64_t j = off[c]; j < off[c + 1]; ++j) {
        int32_t v = abs(lits[j]);
        oc[fill[v]] = c;
        os[fill[v]] = lits[j] > 0;
        fill[v]++;
      }
    free(fill);
  }
  /* clauses opening at each variable, in clause order */
  int64_t* ob = (int64_t*)calloc((size_t)n + 2, sizeof(int64_t));
  int32_t* ol = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  if (!ob || !ol) { free(ob); free(ol); rc = -1; goto done; }
  for (int32_t c = 0; c < m; ++c) ob[first[c] + 1]++;
  for (int32_t v = 1; v <= n + 1; ++v) ob[v] += ob[v - 1];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 2));
    memcpy(fill, ob, sizeof(int64_t) * ((size_t)n + 2));
    for (int32_t c = 0; c < m; ++c) ol[fill[first[c]]++] = c;
    free(fill);
  }
  uint64_t freemask[KW];
  for (int i = 0; i < KW; ++i) freemask[i] = ~0ull;
  if (t_init(&cur, 1024) || t_init(&nxt, 1024)) { rc = -1; goto done2; }
  {
    uint64_t z[KW] = {0};
    t_add(&cur, z, 1.0);
  }
  for (int32_t v = 1; v <= n; ++v) {
    for (int64_t j = ob[v]; j < ob[v + 1]; ++j) {
      int32_t c = ol[j], b = -1;
      for (int i = 0; i < KW && b < 0; ++i)
        if (freemask[i]) {
          b = i * 64 + __builtin_ctzll(freemask[i]);
          freemask[i] &= ~(1ull << (b & 63));
        }
      if (b < 0) { rc = -2; goto done2; }
      bit[c] = b;
    }
    uint64_t pos[KW] = {0}, neg[KW] = {0}, close[KW] = {0};
    for (int64_t j = vo[v]; j < vo[v + 1]; ++j) {
      int32_t c = oc[j], b = bit[c];
      if (os[j]) pos[b >> 6] |= 1ull << (b & 63);
      else neg[b >> 6] |= 1ull << (b & 63);
      if (last[c] == v) close[b >> 6] |= 1ull << (b & 63);
    }
    /* a clause closes at its last variable, which always occurs in it */
    nxt.n = 0;
    memset(nxt.s, 0, nxt.cap * sizeof(slot_t));
    for (size_t i = 0; i < cur.cap; ++i) {
      if (!cur.s[i].used) continue;
      for (int val = 0; val < 2; ++val) {
        if (fix && fix[v] >= 0 && fix[v] != val) continue;
        const uint64_t* add = val ? pos : neg;
        uint64_t k[KW];
        int ok = 1;
        for (int q = 0; q < KW; ++q) {
          k[q] = cur.s[i].k[q] | add[q];
          if ((k[q] & close[q]) != close[q]) ok = 0;
          k[q] &= ~close[q];
        }
        if (!ok) continue;
        if (t_add(&nxt, k, cur.s[i].v * (val ? w1[v] : w0[v]))) { rc = -1; goto done2; }
      }
    }
    for (int64_t j = vo[v]; j < vo[v + 1]; ++j) {
      int32_t c = oc[j];
      if (last[c] == v && bit[c] >= 0) {
        freemask[bit[c] >> 6] |= 1ull << (bit[c] & 63);
        bit[c] = -1;
      }
    }
    table_t tmp = cur;
    cur = nxt;
    nxt = tmp;
    if ((int64_t)cur.n > *peak) *peak = (int64_t)cur.n;
    if (max_states > 0 && (int64_t)cur.n > max_states) { rc = -3; goto done2; }
    /* keep the spare table no larger than needed */
    if (nxt.cap < cur.cap) {
      free(nxt.s);
      if (t_init(&nxt, cur.cap)) { rc = -1; goto done2; }
    }
  }
  {
    double s = 0.0;
    for (size_t i = 0; i < cur.cap; ++i)
      if (cur.s[i].used) s += cur.s[i].v;
    *out = s;
  }
done2:
  free(ob);
  free(ol);
done:
  free(cur.s);
  free(nxt.s);
  free(first);
  free(last);
  free(bit);
  free(vo);
  free(oc);
  free(os);
  return rc;
}
