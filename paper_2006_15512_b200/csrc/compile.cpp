// Host program compiler (see compile.hpp).
//
// What it decides, per internal node of the (sliced) contraction tree:
//   * the PHYSICAL shape of every tensor.  FactorTree's copy-tensor pieces
//     (factoring.py:194-206) are generalised diagonals: an identity piece
//     I[a,b] or a rank-3 piece delta[a,b,c] is exactly zero unless all its
//     indices agree.  A leaf whose entries are zero off such a diagonal is
//     stored over its "tie blocks" (one physical variable per block of
//     indices that must agree), and ties propagate through contractions by
//     union-find (a component of tied indices is one variable of the
//     product).  Every tensor is then a dense array over its physical
//     variables; the structurally-zero entries of the reference's dense
//     tensors are never stored, read, or multiplied.  The result is
//     identical: each dropped term is an exact 0 (x*0 = 0 and acc + 0 = acc
//     for finite values; only the sign of an exact zero can differ), so a
//     dense sum and the compressed sum agree bit for bit on the nonzero
//     terms in the same order.  A contraction's variables fall into M (A and
//     C), N (B and C), K (A and B, summed) and batch (A, B and C; only tied
//     networks have these).  TC_NO_TIES=1 keeps every index its own
//     variable (dense semantics).
//   * kernel class — TINY (whole small subtrees evaluated in one CTA's shared
//     memory, many subtrees per launch), STREAM (big tensor x <=64-entry
//     operand, HBM-bound), GEMM (FP64 DMMA, optional batch variables),
//     GENERIC (mixed radix fallback), ALIAS (C is A's buffer with variables
//     renamed: contractions with an all-ones tie piece, e.g. every identity
//     and delta piece of a copy tensor);
//   * the memory layout of every intermediate.  The reference always emits
//     kept_a ++ kept_b (tensor.py:108) and numpy pays a transpose copy per
//     tensordot (60-70% of CPU time).  Here layouts are chosen
//     top-down so that a STREAM node's output is an in-place relabel of its
//     big input and a GEMM's operands are K-lowest matrices; the permutation
//     is folded into the producing kernel's addressing and no separate
//     transpose pass exists;
//   * a static arena: offsets from a first-fit simulation in postorder, with
//     write-after-read edges added to the launch DAG wherever a buffer reuses
//     memory, so independent branches may run concurrently in the CUDA graph.
#include "compile.hpp"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <future>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <tuple>

namespace tc {

namespace {

constexpr int64_t kTinyMax = 4096;           // entries per tiny tensor
constexpr int32_t kTinySmemCap = 16 * 1024;  // doubles of intermediates per tiny CTA (128 KB; the
                                             // rest of the 227 KB holds the staged batch)
constexpr int64_t kAlign = 256;
constexpr int64_t kSMs = 148;                // B200 SM count (split-K sizing)
constexpr int kMaxTie = 4;                   // physical variables of one operand in one component
constexpr int64_t kLateReleaseMax = (int64_t)1 << 30;  // late release (chain-link fusion) up to 1 GiB

[[noreturn]] void fail(int st, const std::string& m) { throw Error{st, m}; }

// First-fit arena simulation.  Memory classes (hoisting): class 1 holds the
// slice-invariant tensors (written once per pass, in the prologue), class 0
// the per-slice ones.  A range freed by one class is only reused by the same
// class, so the write-after-read edges within each class are complete (an
// invariant writer between two per-slice users of a range would otherwise
// carry their ordering, and it is not in the per-slice graph).
struct Alloc {
  std::map<int64_t, int64_t> free_[3];                   // off -> size
  std::map<int64_t, std::pair<int64_t, int>> seg[3];     // off -> (end, last reader step)
  // Each memory class has its own region: class 1 (slice-invariant, the
  // prologue's) starts above the pinned prefix; class 0 (per slice) is
  // allocated in a tagged address space (offsets >= kTag) and relocated above
  // class 1's region at the end of the compile (relocate()), so a slice
  // lane's private copy holds only the per-slice region.  Without hoisting
  // there is one class and no tag.
  // Class 2 (the block tier: per-slice nodes that run once per block of
  // slices) lives in the lane-private part too, above class 0 (tag kTag2).
  static constexpr int64_t kTag = (int64_t)1 << 56;
  static constexpr int64_t kTag2 = (int64_t)2 << 56;
  bool split = false;
  int64_t top_[3] = {0, 0, 0};  // per-class high-water mark (absolute, tagged for classes 0 / 2 when split)
  int64_t hi[3] = {0, 0, 0};    // highest end of any allocation per memory class

  bool no_reuse = false;  // every buffer gets fresh memory: no WAR edges at all
  // pinned region [0, pin_end): buffers that are never released (hoisting
  // boundary tensors); the simulation proper starts above it
  int64_t pin_top = 0, pin_end = 0;

  void reserve_pinned(int64_t bytes) {
    pin_end = bytes;
    for (int c = 0; c < 3; ++c) top_[c] = std::max(top_[c], bytes);
  }
  void split_classes() {  // after reserve_pinned, before any alloc
    split = true;
    top_[0] = kTag;
    top_[2] = kTag2;
  }
  int64_t alloc_pinned(int64_t size) {
    size = (size + kAlign - 1) / kAlign * kAlign;
    const int64_t o = pin_top;
    pin_top += size;
    if (pin_top > pin_end) fail(TC_BAD_ARG, "pinned arena region overflow");
    return o;
  }
  // final layout: [pinned | class 1 | class 0 | class 2]; returns the class-0 base
  int64_t region0_base() const {
    if (!split) return pin_end;
    return (top_[1] + kAlign - 1) / kAlign * kAlign;
  }
  int64_t region2_base() const { return region0_base() + (top_[0] - kTag + kAlign - 1) / kAlign * kAlign; }
  int64_t arena_end() const {
    if (!split) return std::max(top_[0], top_[1]);
    return region2_base() + (top_[2] - kTag2);
  }
  int64_t relocate(int64_t off) const {
    if (!split || off < kTag) return off;
    return off >= kTag2 ? off - kTag2 + region2_base() : off - kTag + region0_base();
  }

  int64_t alloc(int64_t size, std::vector<int>& hazards, int cl = 0) {
    size = (size + kAlign - 1) / kAlign * kAlign;
    const int r = split ? cl : 0;  // the region (top) this class allocates from
    int64_t& top = top_[r];
    if (no_reuse) {
      int64_t o = top;
      top += size;
      hi[cl] = std::max(hi[cl], top);
      return o;
    }
    auto& fr = free_[cl];
    int64_t off = -1;
    for (auto it = fr.begin(); it != fr.end(); ++it) {
      if (it->second >= size) {
        off = it->first;
        int64_t rest = it->second - size;
        fr.erase(it);
        if (rest > 0) fr[off + size] = rest;
        break;
      }
    }
    if (off < 0) {
      // extend: reuse a free block of this class touching the top
      if (!fr.empty()) {
        auto last = std::prev(fr.end());
        if (last->first + last->second == top) {
          off = last->first;
          fr.erase(last);
          top = off + size;
        }
      }
      if (off < 0) {
        off = top;
        top += size;
      }
    }
    // hazards: previous readers of any byte we are about to overwrite
    auto& sg = seg[cl];
    int64_t end = off + size;
    auto it = sg.upper_bound(off);
    if (it != sg.begin()) --it;
    while (it != sg.end() && it->first < end) {
      int64_t s0 = it->first, s1 = it->second.first;
      int rd = it->second.second;
      if (s1 <= off) {
        ++it;
        continue;
      }
      hazards.push_back(rd);
      it = sg.erase(it);
      if (s0 < off) sg[s0] = {off, rd};
      if (s1 > end) sg[end] = {s1, rd};
      it = sg.lower_bound(std::min(s1, end));
    }
    hi[cl] = std::max(hi[cl], end);
    return off;
  }

  void release(int64_t off, int64_t size, int reader, int cl = 0) {
    if (no_reuse || off < pin_end) return;  // (class-0 offsets are tagged, never below pin_end)
    size = (size + kAlign - 1) / kAlign * kAlign;
    seg[cl][off] = {off + size, reader};
    auto& fr = free_[cl];
    auto nx = fr.lower_bound(off);
    int64_t o = off, s = size;
    if (nx != fr.end() && nx->first == off + size) {
      s += nx->second;
      nx = fr.erase(nx);
    }
    if (nx != fr.begin()) {
      auto pv = std::prev(nx);
      if (pv->first + pv->second == o) {
        o = pv->first;
        s += pv->second;
        fr.erase(pv);
      }
    }
    fr[o] = s;
  }
};

// linear-probe map for the small key sets of one node (layouts of rank <= ~64)
template <class V>
struct SmallMap {
  std::vector<std::pair<int, V>> kv;
  V& operator[](int k) {
    for (auto& e : kv)
      if (e.first == k) return e.second;
    kv.push_back({k, V{}});
    return kv.back().second;
  }
};

// first-fit shared-memory allocator of one tiny group (doubles, 16-byte
// granules): lowest-offset free block that fits, coalescing frees, top trim
struct SmemFit {
  std::vector<std::pair<int32_t, int32_t>> fr;  // sorted (off, size)
  int32_t top = 0;
  void reset() {
    fr.clear();
    top = 0;
  }
  int32_t alloc(int32_t n) {
    n = (n + 1) & ~1;
    for (size_t q = 0; q < fr.size(); ++q)
      if (fr[q].second >= n) {
        const int32_t o = fr[q].first, rest = fr[q].second - n;
        if (rest) fr[q] = {o + n, rest};
        else fr.erase(fr.begin() + q);
        return o;
      }
    const int32_t o = top;
    top += n;
    return o;
  }
  void free(int32_t o, int32_t n) {
    n = (n + 1) & ~1;
    auto it = std::lower_bound(fr.begin(), fr.end(), std::make_pair(o, (int32_t)0));
    it = fr.insert(it, {o, n});
    size_t q = (size_t)(it - fr.begin());
    if (q + 1 < fr.size() && fr[q + 1].first == o + fr[q].second) {
      fr[q].second += fr[q + 1].second;
      fr.erase(fr.begin() + q + 1);
    }
    if (q > 0 && fr[q - 1].first + fr[q - 1].second == fr[q].first) {
      fr[q - 1].second += fr[q].second;
      fr.erase(fr.begin() + q);
    }
    if (!fr.empty() && fr.back().first + fr.back().second == top) {
      top = fr.back().first;
      fr.pop_back();
    }
  }
};

BitRuns make_runs(const std::vector<std::pair<int, int>>& bits) {  // (src bit, dst bit), src ascending
  BitRuns r{};
  r.n = 0;
  for (size_t j = 0; j < bits.size(); ++j) {
    int s = bits[j].first, d = bits[j].second;
    if (r.n > 0) {
      int k = r.n - 1;
      if (r.src[k] + r.len[k] == s && r.dst[k] + r.len[k] == d) {
        r.len[k]++;
        continue;
      }
    }
    if (r.n >= kMaxRuns) throw Error{-1, "runs"};
    r.src[r.n] = (uint8_t)s;
    r.dst[r.n] = (uint8_t)d;
    r.len[r.n] = 1;
    r.n++;
  }
  return r;
}

// Split [0, n) into up to 8 contiguous ranges (at least `grain` items each)
// run on worker threads; f(lo, hi) must not throw.
// worker threads for the host compile (TC_COMPILE_THREADS, default 8)
int compile_threads() {
  static const int t = [] {
    const char* e = std::getenv("TC_COMPILE_THREADS");
    const int v = e ? std::atoi(e) : 8;
    return std::max(1, std::min(64, v));
  }();
  return t;
}

template <class F>
void parallel_for(int n, int grain, F f) {
  const int T = std::max(1, std::min(compile_threads(), n / std::max(1, grain)));
  if (T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int w = 1; w < T; ++w) th.emplace_back(f, (int)((int64_t)n * w / T), (int)((int64_t)n * (w + 1) / T));
  f(0, (int)((int64_t)n / T));
  for (auto& x : th) x.join();
}

// One component of tied indices at a contraction: its variable in C (-1:
// summed) and its variables in the operands A (left) and B (right).
struct Comp {
  int32_t c;
  int8_t na, nb;
  int32_t a[kMaxTie], b[kMaxTie];
  int32_t key() const { return std::min(na ? a[0] : INT_MAX, nb ? b[0] : INT_MAX); }
};

// Coarsest partition of the kept positions of a dim-2 leaf (<= 4 of them)
// such that every nonzero entry agrees within each block (restricted growth
// strings in lexicographic order; first minimum wins).  lab[q] = block.
// Works on the set of kept-digit patterns of the nonzero entries (a 16-bit
// mask) against each partition's mask of diagonal patterns.
struct TiePartitions {
  // per r: (labels, blocks, allowed-pattern mask) in RGS order
  std::vector<std::tuple<std::vector<int>, int, uint32_t>> by_r[5];
  TiePartitions() {
    for (int r = 2; r <= 4; ++r) {
      std::vector<int> cur(r, 0);
      for (;;) {
        int blocks = 0;
        for (int x : cur) blocks = std::max(blocks, x + 1);
        uint32_t allowed = 0;
        for (int pat = 0; pat < (1 << r); ++pat) {
          bool ok = true;
          for (int x = 0; x < r && ok; ++x)
            for (int y = x + 1; y < r && ok; ++y)
              if (cur[x] == cur[y] && ((pat >> x) & 1) != ((pat >> y) & 1)) ok = false;
          if (ok) allowed |= 1u << pat;
        }
        by_r[r].emplace_back(cur, blocks, allowed);
        int q = r - 1;
        for (; q >= 1; --q) {
          int m = 0;
          for (int t = 0; t < q; ++t) m = std::max(m, cur[t]);
          if (cur[q] <= m) {
            cur[q]++;
            for (int t = q + 1; t < r; ++t) cur[t] = 0;
            break;
          }
        }
        if (q < 1) break;
      }
    }
  }
};

bool leaf_ties(const Plan& p, int l, const std::vector<char>& drop, std::vector<int>& lab) {
  static const TiePartitions parts;
  const auto& ro = p.ref_order[l];
  int kq[4];
  int r = 0;
  for (size_t q = 0; q < ro.size(); ++q)
    if (!drop[ro[q]]) {
      if (p.dom[ro[q]] != 2 || r == 4) return false;
      kq[r++] = (int)q;
    }
  if (r < 2 || p.leaf_size(l) > 4096) return false;
  const double* v = p.lval.data() + p.lval_off[l];
  const int64_t n = p.leaf_size(l);
  int64_t stride[16];
  if (ro.size() > 16) return false;
  int64_t st = 1;
  for (int q = (int)ro.size() - 1; q >= 0; --q) {
    stride[q] = st;
    st *= p.dom[ro[q]];
  }
  uint32_t nz = 0;  // kept-digit patterns of the nonzero entries
  for (int64_t e = 0; e < n; ++e) {
    if (v[e] == 0.0) continue;
    int pat = 0;
    for (int x = 0; x < r; ++x) pat |= (int)((e / stride[kq[x]]) & 1) << x;
    nz |= 1u << pat;
  }
  const std::vector<int>* best = nullptr;
  int best_blocks = r;
  for (const auto& [labs, blocks, allowed] : parts.by_r[r])
    if (blocks < best_blocks && (nz & ~allowed) == 0) {
      best = &labs;
      best_blocks = blocks;
    }
  if (!best) return false;
  lab.assign(ro.size(), -1);
  for (int x = 0; x < r; ++x) lab[kq[x]] = (*best)[x];
  return true;
}

}  // namespace

Program compile_program(const Plan& p, const std::vector<int>& chosen_in, int64_t no_reuse_limit) {
  Program g;
  // section timings to stderr when TC_COMPILE_TIMING is set (diagnostics)
  static const bool timing = std::getenv("TC_COMPILE_TIMING") != nullptr;
  auto tlast = std::chrono::steady_clock::now();
  std::string prev = "start";
  auto tmark = [&](const char* name) {
    if (!timing) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[compile] %-22s %8.2f ms\n", prev.c_str(),
                 std::chrono::duration<double, std::milli>(now - tlast).count());
    tlast = now;
    prev = name;
  };
  const int S = p.nslots();
  std::vector<char> drop(p.NI, 0);
  for (int i : chosen_in) {
    if (i < 0 || i >= p.NI) fail(TC_BAD_ARG, "slice index id out of range");
    if (!p.is_bond[i]) fail(TC_NOT_A_BOND, "slice index is not a bond index of the network");
    if (drop[i]) fail(TC_BAD_ARG, "slice index listed twice");
    drop[i] = 1;
  }
  g.chosen = chosen_in;
  g.num_slices = 1;
  for (int i : chosen_in) {
    g.chosen_dim.push_back(p.dom[i]);
    if (__builtin_mul_overflow(g.num_slices, (int64_t)p.dom[i], &g.num_slices))
      fail(TC_OVERFLOW, "number of slices exceeds 2^63");
  }
  // The reference accounting (mem_cost / tracked peak, slicing.py:52-67,
  // 91-109) and the dense per-node work only feed the statistics: computed
  // on a second thread while the program is built.
  std::vector<u128> dsize(S);
  u128 dense_bytes = 0, dense_flops = 0, mem_est = 0, peak_obs = 0;
  auto accounting = std::async(std::launch::async, [&] {
    mem_est = mem_cost(p, drop);
    peak_obs = tracked_peak(p, drop);
    for (int s = 0; s < S; ++s) dsize[s] = set_bytes(p, p.sets[s], drop) / 8;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k, a = p.left[k], b = p.right[k];
      // |A u B| = |A| |B| / |A n B|
      u128 sh = 1;
      const auto& Ea = p.sets[a];
      const auto& Eb = p.sets[b];
      for (size_t x = 0, y = 0; x < Ea.size() && y < Eb.size();) {
        if (Ea[x] < Eb[y]) ++x;
        else if (Eb[y] < Ea[x]) ++y;
        else {
          if (!drop[Ea[x]]) sh *= (u128)p.dom[Ea[x]];
          ++x, ++y;
        }
      }
      dense_flops += 2 * (dsize[a] / sh) * dsize[b];
      dense_bytes += (u128)8 * (dsize[a] + dsize[b] + dsize[v]);
    }
  });

  tmark("physical variables");
  // ---- physical variables: tie blocks of leaves, union-find at nodes --------
  // mem[s]: (logical index, variable) pairs sorted by logical index; a
  // variable is named by the smallest logical index of its block.
  // A non-finite leaf value makes a skipped structural-zero term Inf*0 = NaN
  // in the reference's dense sum: such plans run on dense variables and
  // without relabel aliases (the reference's arithmetic, term for term).
  bool ties = std::getenv("TC_NO_TIES") == nullptr && p.all_finite;
  // Tie-aware slicing: a sliced bond fixes every index tied to it (the dense
  // leaves are zero unless the whole tie class agrees), so those indices are
  // sliced too ("implied", same value, same place value in the slice id).
  // pdrop is the physical slice set; the reference accounting keeps `drop`.
  // Classes holding a free index or two sliced indices are left alone.
  std::vector<char> pdrop = drop;
  std::vector<int> implied_src(p.NI, -1);
  if (ties && !chosen_in.empty()) {
    std::vector<int> cu(p.NI);
    for (int i = 0; i < p.NI; ++i) cu[i] = i;
    auto cfind = [&](int x) {
      while (cu[x] != x) x = cu[x] = cu[cu[x]];
      return x;
    };
    const std::vector<char> none(p.NI, 0);
    std::vector<int> lab2;
    for (int l = 0; l < p.NL; ++l) {
      if (!leaf_ties(p, l, none, lab2)) continue;
      const auto& ro = p.ref_order[l];
      for (size_t q = 0; q < ro.size(); ++q)
        for (size_t q2 = q + 1; q2 < ro.size(); ++q2)
          if (lab2[q] >= 0 && lab2[q] == lab2[q2]) {
            const int x = cfind(ro[q]), y = cfind(ro[q2]);
            if (x != y) cu[std::max(x, y)] = std::min(x, y);
          }
    }
    std::vector<int> nsl(p.NI, 0), src(p.NI, -1);
    std::vector<char> has_free(p.NI, 0);
    for (int i = 0; i < p.NI; ++i) {
      const int r = cfind(i);
      if (drop[i]) nsl[r]++, src[r] = i;
      if (!p.is_bond[i]) has_free[r] = 1;
    }
    for (int i = 0; i < p.NI; ++i) {
      const int r = cfind(i);
      if (!drop[i] && nsl[r] == 1 && !has_free[r] && p.dom[i] == p.dom[src[r]]) {
        pdrop[i] = 1;
        implied_src[i] = src[r];
      }
    }
  }
  // Per-slot tables live in two pools (no per-node allocations): leaves at
  // fixed offsets, internal nodes appended in postorder (a recomputed node
  // appends again; capacity is reserved before each pass so spans stay valid).
  using MPair = std::pair<int, int>;
  struct MemSpan {
    const MPair *b, *e;
    const MPair* begin() const { return b; }
    const MPair* end() const { return e; }
    size_t size() const { return (size_t)(e - b); }
    const MPair& operator[](size_t i) const { return b[i]; }
  };
  struct IntSpan {
    const int *b, *e;
    const int* begin() const { return b; }
    const int* end() const { return e; }
    size_t size() const { return (size_t)(e - b); }
    int operator[](size_t i) const { return b[i]; }
  };
  // Slot tables are spans into arenas whose vectors are reserved up front and
  // never reallocated: the leaf arena, one arena per worker of the parallel
  // first pass, one per push-down round.
  struct Arena {
    std::vector<MPair> m;
    std::vector<int> v;
    std::vector<Comp> c;
  };
  std::vector<std::unique_ptr<Arena>> arenas;
  auto new_arena = [&](size_t nm, size_t nv, size_t nc) {
    arenas.emplace_back(new Arena);
    Arena& a = *arenas.back();
    a.m.reserve(nm + 1);
    a.v.reserve(nv + 1);
    a.c.reserve(nc + 1);
    return &a;
  };
  std::vector<const MPair*> mB(S, nullptr), mE(S, nullptr);
  std::vector<const int*> vB(S, nullptr), vE(S, nullptr);
  std::vector<const Comp*> cB(p.NN, nullptr), cE(p.NN, nullptr);
  auto mem = [&](int s) { return MemSpan{mB[s], mE[s]}; };
  auto varsv = [&](int s) { return IntSpan{vB[s], vE[s]}; };
  std::vector<MPair> mpool;  // leaves
  std::vector<int> vpool;
  std::vector<char> leaf_tied(p.NL, 0);
  // Tie push-down: when a contraction reads two variables of an internal
  // operand as one (a diagonal read: a copy-tensor piece ties two indices the
  // operand keeps separately), the operand's off-diagonal entries are
  // computed and never used.  The tie is pushed down to the node where the
  // two indices first meet (they come from different children there) and
  // realised as a merge at that node, so every tensor on the way is computed
  // directly on the diagonal: half the work and bytes per tie, and no gather.
  std::vector<std::vector<std::pair<int, int>>> req(p.NN);
  auto has_logical = [&](int s, int l) {
    const auto m = mem(s);
    auto f = std::lower_bound(m.begin(), m.end(), std::make_pair(l, INT_MIN));
    return f != m.end() && f->first == l;
  };
  int pushdown_rounds = 0;
  auto build_leaves = [&]() {
    // leaf l owns [off[l], off[l] + kept) in both pools
    std::vector<int64_t> off(p.NL + 1, 0);
    for (int l = 0; l < p.NL; ++l) {
      int64_t k = 0;
      for (int i : p.ref_order[l]) k += !pdrop[i];
      off[l + 1] = off[l] + k;
    }
    mpool.assign(off[p.NL], MPair{0, 0});
    vpool.assign(off[p.NL], 0);
    parallel_for(p.NL, 4096, [&](int l0, int l1) {
      std::vector<int> lab;
      for (int l = l0; l < l1; ++l) {
        const auto& ro = p.ref_order[l];
        MPair* m = mpool.data() + off[l];
        int n = 0;
        leaf_tied[l] = ties && leaf_ties(p, l, pdrop, lab);
        if (leaf_tied[l]) {
          int bmin[8];
          for (int q = 0; q < 8; ++q) bmin[q] = INT_MAX;
          for (size_t q = 0; q < ro.size(); ++q)
            if (lab[q] >= 0) bmin[lab[q]] = std::min(bmin[lab[q]], ro[q]);
          for (size_t q = 0; q < ro.size(); ++q)
            if (lab[q] >= 0) m[n++] = {ro[q], bmin[lab[q]]};
        } else {
          for (int i : ro)
            if (!pdrop[i]) m[n++] = {i, i};
        }
        std::sort(m, m + n);
        mB[l] = m;
        mE[l] = m + n;
        int* vv = vpool.data() + off[l];
        for (int q = 0; q < n; ++q) vv[q] = m[q].second;
        std::sort(vv, vv + n);
        vB[l] = vv;
        vE[l] = vv + (std::unique(vv, vv + n) - vv);
      }
    });
  };
  build_leaves();
  // Requests known before the pass: a tied leaf piece whose block holds two
  // indices of its sibling subtree (the common copy-tensor case) is pushed
  // down symbolically; the rounds below catch ties that arise deeper.
  auto push_down = [&](int u, int l1, int l2) {
    auto in_set = [&](int sl, int l) { return std::binary_search(p.sets[sl].begin(), p.sets[sl].end(), l); };
    for (;;) {
      const int ku = u - p.NL, ca = p.left[ku], cb = p.right[ku];
      const int c1 = in_set(ca, l1) ? ca : cb, c2 = in_set(ca, l2) ? ca : cb;
      if (c1 == c2 && !p.is_leaf(c1)) {
        u = c1;
        continue;
      }
      req[ku].push_back({l1, l2});
      return;
    }
  };
  if (ties) {
    for (int l = 0; l < p.NL; ++l) {
      if (!leaf_tied[l] || p.parent[l] < 0) continue;
      const int v = p.parent[l], k = v - p.NL;
      const int x = p.left[k] == l ? p.right[k] : p.left[k];
      if (p.is_leaf(x)) continue;
      const auto m = mem(l);
      for (size_t i = 0; i < m.size(); ++i)
        for (size_t j = i + 1; j < m.size(); ++j)
          if (m[i].second == m[j].second && std::binary_search(p.sets[x].begin(), p.sets[x].end(), m[i].first) &&
              std::binary_search(p.sets[x].begin(), p.sets[x].end(), m[j].first))
            push_down(x, m[i].first, m[j].first);
    }
  }
  tmark("phys: node passes");
  // One node of the bottom-up pass: union-find over the operands' variables
  // (shared logical indices, realised push-down requests) -> components, the
  // node's (logical, variable) table and sorted variables, into arena `ar`.
  struct Scratch {
    std::vector<int> uf, own_a, own_b, cidx;
    std::vector<Comp> cs;
  };
  auto make_scratch = [&]() {
    Scratch sc;
    sc.uf.assign(p.NI, -1);
    sc.own_a.assign(p.NI, -1);
    sc.own_b.assign(p.NI, -1);
    sc.cidx.assign(p.NI, -1);
    return sc;
  };
  auto process_node = [&](int k, Scratch& sc, Arena& ar, bool& overflow) {
    const int v = p.NL + k, a = p.left[k], b = p.right[k];
    auto& uf = sc.uf;
    auto& own_a = sc.own_a;
    auto& own_b = sc.own_b;
    auto& cidx = sc.cidx;
    auto& cs = sc.cs;
    auto find = [&](int x) {
      while (uf[x] != x) {
        uf[x] = uf[uf[x]];
        x = uf[x];
      }
      return x;
    };
    const MemSpan Ma = mem(a), Mb = mem(b);
    const IntSpan Va = varsv(a), Vb = varsv(b);
    for (auto& e : Ma) own_a[e.first] = e.second;
    for (auto& e : Mb) own_b[e.first] = e.second;
    for (int x : Va) uf[x] = x;
    for (int x : Vb) uf[x] = x;
    for (auto& e : Mb)
      if (own_a[e.first] >= 0) {
        int r1 = find(own_a[e.first]), r2 = find(e.second);
        if (r1 != r2) uf[std::max(r1, r2)] = std::min(r1, r2);
      }
    for (auto& q : req[k]) {  // pushed-down ties realised here
      const int x = own_a[q.first] >= 0 ? own_a[q.first] : own_b[q.first];
      const int y = own_a[q.second] >= 0 ? own_a[q.second] : own_b[q.second];
      if (x < 0 || y < 0) continue;
      int r1 = find(x), r2 = find(y);
      if (r1 != r2) uf[std::max(r1, r2)] = std::min(r1, r2);
    }
    cs.clear();
    auto comp_of = [&](int var) -> Comp& {
      int r = find(var);
      if (cidx[r] < 0) {
        cidx[r] = (int)cs.size();
        Comp c{};
        c.c = -1;
        cs.push_back(c);
      }
      return cs[cidx[r]];
    };
    for (int x : Va) {
      Comp& c = comp_of(x);
      if (c.na == kMaxTie) overflow = true;
      else c.a[c.na++] = x;
    }
    for (int x : Vb) {
      Comp& c = comp_of(x);
      if (c.nb == kMaxTie) overflow = true;
      else c.b[c.nb++] = x;
    }
    // kept logical indices -> component's C variable (smallest kept index)
    const size_t m0 = ar.m.size();
    {
      size_t x = 0, y = 0;
      for (;;) {  // merge the kept entries of both (each sorted by logical index)
        while (x < Ma.size() && own_b[Ma[x].first] >= 0) ++x;
        while (y < Mb.size() && own_a[Mb[y].first] >= 0) ++y;
        if (x == Ma.size() && y == Mb.size()) break;
        if (y == Mb.size() || (x < Ma.size() && Ma[x].first < Mb[y].first)) ar.m.push_back(Ma[x++]);
        else ar.m.push_back(Mb[y++]);
      }
    }
    for (size_t q = m0; q < ar.m.size(); ++q) {
      Comp& c = comp_of(ar.m[q].second);
      if (c.c < 0) c.c = ar.m[q].first;  // sorted: first kept = smallest
    }
    for (size_t q = m0; q < ar.m.size(); ++q) ar.m[q].second = comp_of(ar.m[q].second).c;
    mB[v] = ar.m.data() + m0;
    mE[v] = ar.m.data() + ar.m.size();
    const size_t v0 = ar.v.size();
    for (const Comp& c : cs)
      if (c.c >= 0) ar.v.push_back(c.c);
    std::sort(ar.v.begin() + v0, ar.v.end());
    vB[v] = ar.v.data() + v0;
    vE[v] = ar.v.data() + ar.v.size();
    // reset scratch (before reordering cs: cidx indexes into it)
    for (int x : Va) cidx[find(x)] = -1;
    for (int x : Vb) cidx[find(x)] = -1;
    for (int x : Va) uf[x] = -1;
    for (int x : Vb) uf[x] = -1;
    for (auto& e : Ma) own_a[e.first] = -1;
    for (auto& e : Mb) own_b[e.first] = -1;
    std::sort(cs.begin(), cs.end(), [](const Comp& x, const Comp& y) { return x.key() < y.key(); });
    const size_t c0 = ar.c.size();
    ar.c.insert(ar.c.end(), cs.begin(), cs.end());
    cB[k] = ar.c.data() + c0;
    cE[k] = ar.c.data() + ar.c.size();
  };
  // arena sizes for a set of nodes (upper bounds: kept entries <= |set|)
  auto bounds = [&](int k, size_t& nm, size_t& nc) {
    const int v = p.NL + k;
    nm += p.sets[v].size();
    nc += p.sets[p.left[k]].size() + p.sets[p.right[k]].size();
  };
  // subtree sizes (internal nodes): a subtree's internal slots are the
  // contiguous postorder range (v - cnt[v], v]
  std::vector<int> cnt(S, 0);
  for (int k = 0; k < p.NN; ++k) {
    const int v = p.NL + k;
    cnt[v] = 1 + cnt[p.left[k]] + cnt[p.right[k]];
  }
  Scratch main_sc = make_scratch();
  // push-down rounds recompute only the nodes on paths from new requests up
  std::vector<char> dirty(S, 0);
  for (int attempt = 0;; ++attempt) {
    bool overflow = false;
    if (attempt == 0 || std::all_of(dirty.begin(), dirty.end(), [](char x) { return x != 0; })) {
      // full pass: maximal subtrees of <= L nodes on worker threads, the
      // rest (the spine above them) in postorder on this thread
      const int L = std::max(256, p.NN / 64);
      std::vector<int> task_roots;
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k;
        if (cnt[v] <= L && (p.parent[v] < 0 || cnt[p.parent[v]] > L)) task_roots.push_back(v);
      }
      std::vector<char> in_task(p.NN, 0);
      int64_t task_nodes = 0;
      for (int r : task_roots) {
        for (int k = r - p.NL - cnt[r] + 1; k <= r - p.NL; ++k) in_task[k] = 1;
        task_nodes += cnt[r];
      }
      const int T = (int)std::max<int64_t>(1, std::min<int64_t>(compile_threads(), task_nodes / 1024));
      std::vector<int> cut{0};
      {
        int64_t acc = 0;
        for (size_t q = 0; q < task_roots.size(); ++q) {
          acc += cnt[task_roots[q]];
          if ((int)cut.size() < T && acc * T >= task_nodes * (int64_t)cut.size()) cut.push_back((int)q + 1);
        }
        while ((int)cut.size() <= T) cut.push_back((int)task_roots.size());
      }
      std::vector<Arena*> war(T);
      for (int w = 0; w < T; ++w) {
        size_t nm = 0, nc = 0;
        for (int q = cut[w]; q < cut[w + 1]; ++q)
          for (int k = task_roots[q] - p.NL - cnt[task_roots[q]] + 1; k <= task_roots[q] - p.NL; ++k) bounds(k, nm, nc);
        war[w] = new_arena(nm, nm, nc);
      }
      std::vector<char> wover(T, 0);
      auto work = [&](int w) {
        Scratch sc = w == 0 ? std::move(main_sc) : make_scratch();
        bool ov = false;
        for (int q = cut[w]; q < cut[w + 1]; ++q)
          for (int k = task_roots[q] - p.NL - cnt[task_roots[q]] + 1; k <= task_roots[q] - p.NL; ++k)
            process_node(k, sc, *war[w], ov);
        wover[w] = ov;
        if (w == 0) main_sc = std::move(sc);
      };
      std::vector<std::thread> th;
      for (int w = 1; w < T; ++w) th.emplace_back(work, w);
      work(0);
      for (auto& x : th) x.join();
      if (timing) std::fprintf(stderr, "[compile]   pass: %d threads, %zu task roots, %lld task nodes of %d\n", T, task_roots.size(), (long long)task_nodes, p.NN);
      tmark("phys: spine");
      for (int w = 0; w < T; ++w) overflow |= (bool)wover[w];
      size_t nm = 0, nc = 0;
      for (int k = 0; k < p.NN; ++k)
        if (!in_task[k]) bounds(k, nm, nc);
      Arena* top = new_arena(nm, nm, nc);
      for (int k = 0; k < p.NN && !overflow; ++k)
        if (!in_task[k]) process_node(k, main_sc, *top, overflow);
    } else {
      // a push-down round: the requested nodes and everything above them
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k;
        dirty[v] = dirty[v] || dirty[p.left[k]] || dirty[p.right[k]];
      }
      size_t nm = 0, nc = 0;
      for (int k = 0; k < p.NN; ++k)
        if (dirty[p.NL + k]) bounds(k, nm, nc);
      Arena* ar = new_arena(nm, nm, nc);
      for (int k = 0; k < p.NN && !overflow; ++k)
        if (dirty[p.NL + k]) process_node(k, main_sc, *ar, overflow);
    }
    tmark("phys: requests");
    if (!overflow) {
      bool pushed = false;
      std::fill(dirty.begin(), dirty.end(), 0);
      if (ties && pushdown_rounds < 8) {
        for (int k = 0; k < p.NN; ++k) {
          const int ch[2] = {p.left[k], p.right[k]};
          for (const Comp* cp = cB[k]; cp != cE[k]; ++cp) {
            const Comp& c = *cp;
            for (int side = 0; side < 2; ++side) {
              const int n = side ? c.nb : c.na;
              const int32_t* vv = side ? c.b : c.a;
              if (n < 2 || p.is_leaf(ch[side])) continue;
              for (int t = 1; t < n; ++t) {
                int u = ch[side];
                const int l1 = vv[0], l2 = vv[t];
                for (;;) {
                  const int ku = u - p.NL, ca = p.left[ku], cb = p.right[ku];
                  const int c1 = has_logical(ca, l1) ? ca : cb, c2 = has_logical(ca, l2) ? ca : cb;
                  if (c1 == c2 && !p.is_leaf(c1)) {
                    u = c1;
                    continue;
                  }
                  req[ku].push_back({l1, l2});
                  dirty[u] = 1;
                  pushed = true;
                  break;
                }
              }
            }
          }
        }
      }
      tmark("phys: node passes");
      if (pushed) {
        if (timing) std::fprintf(stderr, "[compile] tie push-down round %d\n", pushdown_rounds);
        ++pushdown_rounds;
        continue;
      }
      for (int l = 0; l < p.NL; ++l) g.n_tied_leaves += leaf_tied[l];
      break;
    }
    if (!ties || attempt > 8) fail(TC_BAD_ARG, "tie component too large");
    ties = false;  // pathological tie structure: fall back to dense variables
    for (auto& r : req) r.clear();
    build_leaves();
    std::fill(dirty.begin(), dirty.end(), 1);  // all dirty: the next attempt is a full pass
  }
  struct EffView {
    const std::vector<const int*>*b, *e;
    IntSpan operator[](int s) const { return IntSpan{(*b)[s], (*e)[s]}; }
  } eff{&vB, &vE};
  auto comps = [&](int v) { return std::make_pair(cB[v - p.NL], cE[v - p.NL]); };
  std::vector<int64_t> size(S);
  for (int s = 0; s < S; ++s) {
    u128 z = 1;
    for (int i : varsv(s)) z *= (u128)p.dom[i];
    if (z > ((u128)1 << 50)) fail(TC_OOM, "intermediate tensor larger than 2^50 entries");
    size[s] = (int64_t)z;
  }
  auto var_of = [&](int s, int logical) {
    const auto m = mem(s);
    return std::lower_bound(m.begin(), m.end(), std::make_pair(logical, INT_MIN))->second;
  };
  // natural layout: the reference's row-major order (first index slowest),
  // LSB-first, one entry per variable (first occurrence)
  std::vector<int> seen_mark(p.NI, -1);
  auto natural = [&](int s) {
    std::vector<int> o;
    const auto& ro = p.ref_order[s];
    o.reserve(varsv(s).size());
    for (auto it = ro.rbegin(); it != ro.rend(); ++it) {
      if (pdrop[*it]) continue;
      const int var = var_of(s, *it);
      if (seen_mark[var] == s) continue;
      seen_mark[var] = s;
      o.push_back(var);
    }
    return o;
  };

  tmark("classification");
  // ---- classification --------------------------------------------------------
  g.cls.assign(S, NC_LEAF);
  auto all2 = [&](int s) {
    for (int i : eff[s])
      if (p.dom[i] != 2) return false;
    return true;
  };
  for (int k = 0; k < p.NN; ++k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    auto tok = [&](int x) { return p.is_leaf(x) ? size[x] <= kTinyMax : g.cls[x] == NC_TINY; };
    int8_t c;
    if (std::max({size[a], size[b], size[v]}) <= kTinyMax && tok(a) && tok(b)) {
      c = NC_TINY;
    } else if (all2(a) && all2(b)) {
      const bool b_small = eff[b].size() <= eff[a].size();
      int ks = 0, f = 0, big_bits = 0;
      bool diag = false;
      for (auto [cp, ce] = comps(v); cp != ce; ++cp) {
        const int nbig = b_small ? cp->na : cp->nb;
        if (cp->c < 0) ks++;
        else if (nbig == 0) f++;
        big_bits = std::max(big_bits, nbig);
        diag |= cp->na > 1 || cp->nb > 1;
      }
      const int sm = b_small ? b : a;
      (void)sm;
      if (ks <= 4 && f <= 5 && ks + f <= 7 && big_bits <= 2)
        c = NC_STREAM;
      else if (!diag)
        c = NC_GEMM;  // any m, n, k: tile bits beyond the shape are virtual
      else
        c = NC_GENERIC;
    } else {
      c = NC_GENERIC;
    }
    g.cls[v] = c;
  }

  tmark("layouts (top-down)");
  // ---- layouts (top-down) ----------------------------------------------------
  g.layout.assign(S, {});
  parallel_for(p.NL, 4096, [&](int l0, int l1) {
    for (int l = l0; l < l1; ++l) {  // natural() without the shared first-occurrence marks
      std::vector<int> o;
      const auto& ro = p.ref_order[l];
      o.reserve(varsv(l).size());
      for (auto it = ro.rbegin(); it != ro.rend(); ++it) {
        if (pdrop[*it]) continue;
        const int var = var_of(l, *it);
        if (std::find(o.begin(), o.end(), var) == o.end()) o.push_back(var);
      }
      g.layout[l] = std::move(o);
    }
  });
  std::vector<int> pos(p.NI, -1);
  auto set_pos = [&](const std::vector<int>& L) {
    for (size_t q = 0; q < L.size(); ++q) pos[L[q]] = (int)q;
  };
  auto clr_pos = [&](const std::vector<int>& L) {
    for (int i : L) pos[i] = -1;
  };
  if (!p.is_leaf(p.root)) g.layout[p.root] = natural(p.root);
  auto want = [&](int child, std::vector<int> L) {
    if (p.is_leaf(child)) return;
    g.layout[child] = std::move(L);
  };
  std::vector<const Comp*> ccomp(p.NI, nullptr);  // C variable -> its component (per node)
  std::vector<const Comp*> K, M, N, Bt;
  for (int k = p.NN - 1; k >= 0; --k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    const std::vector<int>& L = g.layout[v];
    auto [c0, c1] = comps(v);
    switch (g.cls[v]) {
      case NC_STREAM: {
        const bool b_small = eff[b].size() <= eff[a].size();
        const int big = b_small ? a : b, sm = b_small ? b : a;
        auto bigv = [&](const Comp* c) { return b_small ? c->a : c->b; };
        auto nbig = [&](const Comp* c) { return b_small ? c->na : c->nb; };
        K.clear();
        for (const Comp* c = c0; c != c1; ++c) {
          if (c->c >= 0) ccomp[c->c] = c;
          else K.push_back(c);
        }
        std::sort(K.begin(), K.end(), [&](const Comp* x, const Comp* y) { return bigv(x)[0] < bigv(y)[0]; });
        // kept big variables at their C positions, a summed one at each
        // new (small-only) variable's position: C is an in-place relabel of
        // the big operand when no diagonal read is involved.  Both bits of a
        // diagonal read go to the top, so the read touches exactly the
        // diagonal half of the big operand in contiguous runs.
        std::vector<int> Lg;
        size_t si = 0;
        std::vector<const Comp*> K1;
        for (const Comp* c : K)
          if (nbig(c) == 1) K1.push_back(c);
        for (int i : L) {
          const Comp* c = ccomp[i];
          if (nbig(c) == 1) Lg.push_back(bigv(c)[0]);
          else if (nbig(c) == 0 && si < K1.size()) Lg.push_back(bigv(K1[si++])[0]);
        }
        while (si < K1.size()) Lg.push_back(bigv(K1[si++])[0]);
        for (int i : L) {
          const Comp* c = ccomp[i];
          if (nbig(c) > 1)
            for (int t = 0; t < nbig(c); ++t) Lg.push_back(bigv(c)[t]);
        }
        for (const Comp* c : K)
          if (nbig(c) > 1)
            for (int t = 0; t < nbig(c); ++t) Lg.push_back(bigv(c)[t]);
        for (const Comp* c = c0; c != c1; ++c)
          if (c->c >= 0) ccomp[c->c] = nullptr;
        want(big, Lg);
        if (!p.is_leaf(sm)) want(sm, natural(sm));
        break;
      }
      case NC_GEMM: {
        K.clear();
        M.clear();
        N.clear();
        Bt.clear();
        for (const Comp* c = c0; c != c1; ++c) {
          if (c->c < 0) K.push_back(c);
          else if (c->na && c->nb) Bt.push_back(c);
          else if (c->na) M.push_back(c);
          else N.push_back(c);
        }
        std::sort(K.begin(), K.end(), [&](const Comp* x, const Comp* y) { return x->a[0] < y->a[0]; });
        // K order: follow a fixed-layout (leaf) operand when there is one
        int ref = p.is_leaf(a) ? a : (p.is_leaf(b) ? b : -1);
        if (ref >= 0) {
          set_pos(g.layout[ref]);
          const bool ra = ref == a;
          std::sort(K.begin(), K.end(), [&](const Comp* x, const Comp* y) {
            return pos[ra ? x->a[0] : x->b[0]] < pos[ra ? y->a[0] : y->b[0]];
          });
          clr_pos(g.layout[ref]);
        }
        set_pos(L);
        auto by_c = [&](const Comp* x, const Comp* y) { return pos[x->c] < pos[y->c]; };
        std::sort(M.begin(), M.end(), by_c);
        std::sort(N.begin(), N.end(), by_c);
        std::sort(Bt.begin(), Bt.end(), by_c);
        clr_pos(L);
        std::vector<int> La, Lb;
        for (const Comp* c : K) La.push_back(c->a[0]), Lb.push_back(c->b[0]);
        for (const Comp* c : M) La.push_back(c->a[0]);
        for (const Comp* c : N) Lb.push_back(c->b[0]);
        for (const Comp* c : Bt) La.push_back(c->a[0]), Lb.push_back(c->b[0]);
        want(a, La);
        want(b, Lb);
        break;
      }
      case NC_TINY:
        break;  // tiny subtrees use natural layouts, built with their descriptors
      default:
        if (!p.is_leaf(a)) want(a, natural(a));
        if (!p.is_leaf(b)) want(b, natural(b));
    }
  }

  // physical values of a leaf: raw values when untied, else the compressed
  // block diagonal in the leaf's layout order (cvals)
  auto leaf_strides = [&](int l) {
    const auto& ro = p.ref_order[l];
    std::vector<int64_t> stride(ro.size());
    int64_t st = 1;
    for (int q = (int)ro.size() - 1; q >= 0; --q) {
      stride[q] = st;
      st *= p.dom[ro[q]];
    }
    return stride;
  };
  // raw offset (kept indices only) of physical entry e of leaf l
  auto leaf_entry_src = [&](int l, int64_t e, const std::vector<int64_t>& stride) {
    const auto& Ll = g.layout[l];
    const auto& ro = p.ref_order[l];
    int64_t src = 0, rem = e;
    for (size_t t = 0; t < Ll.size(); ++t) {
      const int d = (int)(rem % p.dom[Ll[t]]);
      rem /= p.dom[Ll[t]];
      for (size_t q = 0; q < ro.size(); ++q)
        if (!pdrop[ro[q]] && var_of(l, ro[q]) == Ll[t]) src += d * stride[q];
    }
    return src;
  };
  std::vector<int64_t> cval_off(p.NL, -1);
  for (int l = 0; l < p.NL; ++l) {
    if (!leaf_tied[l]) continue;
    bool sl = false;
    for (int i : p.ref_order[l]) sl |= (bool)pdrop[i];
    if (sl) continue;  // sliced leaves are gathered per slice (k_select)
    auto stride = leaf_strides(l);
    cval_off[l] = (int64_t)g.cvals.size();
    for (int64_t e = 0; e < size[l]; ++e) g.cvals.push_back(p.lval[p.lval_off[l] + leaf_entry_src(l, e, stride)]);
  }
  auto leaf_phys = [&](int l, int64_t e) {
    return cval_off[l] >= 0 ? g.cvals[cval_off[l] + e] : p.lval[p.lval_off[l] + e];
  };

  tmark("exact relabels");
  // ---- exact relabels ---------------------------------------------------------
  // C IS the big operand's buffer (no launch, no traffic) when the small
  // operand is an all-ones tie piece (every big variable maps to one C
  // variable at the same address bit, nothing is summed, x*1 == x), or, with
  // dense variables, a 2x2 identity piece (x*1 + y*0 == x for finite y).
  // These are the non-carrier pieces of factored copy tensors
  // (factoring.py:194-206).
  // A leaf every index of which is sliced (chosen or implied by its tie
  // class) selects one scalar per slice; it is 1.0 for every slice when every
  // entry whose tied indices agree is 1.0 (the non-carrier pieces of a sliced
  // variable's copy tensor).
  auto unit_when_sliced = [&](int l) {
    const auto& ro = p.ref_order[l];
    if (ro.empty() || ro.size() > 8) return false;
    int cls_idx[8], classes[8], nc = 0;
    for (size_t q = 0; q < ro.size(); ++q) {
      const int i = ro[q];
      if (!pdrop[i] || p.dom[i] != 2) return false;
      const int c = drop[i] ? i : implied_src[i];
      if (c < 0) return false;
      int k = 0;
      while (k < nc && classes[k] != c) ++k;
      if (k == nc) classes[nc++] = c;
      cls_idx[q] = k;
    }
    const double* v = p.lval.data() + p.lval_off[l];
    for (int m = 0; m < (1 << nc); ++m) {
      int64_t e = 0;
      for (size_t q = 0; q < ro.size(); ++q) e = e * 2 + ((m >> cls_idx[q]) & 1);
      if (v[e] != 1.0) return false;
    }
    return true;
  };
  std::vector<int> alias_src(S, -1);
  if (!std::getenv("TC_NO_ALIAS") && p.all_finite) {
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k, a = p.left[k], b = p.right[k];
      if (g.cls[v] != NC_STREAM) continue;
      const bool b_small = eff[b].size() <= eff[a].size();
      const int big = b_small ? a : b, sm = b_small ? b : a;
      if (p.is_leaf(big) || !p.is_leaf(sm)) continue;
      const auto& Lv = g.layout[v];
      const auto& Lg = g.layout[big];
      if (Lv.size() != Lg.size()) continue;
      auto [c0, c1] = comps(v);
      bool ok = false;
      if (leaf_tied[sm]) {
        ok = true;
        for (int64_t e = 0; ok && e < size[sm]; ++e) ok = leaf_phys(sm, e) == 1.0;
        for (const Comp* c = c0; ok && c != c1; ++c) {
          const int nbig = b_small ? c->na : c->nb;
          if (c->c < 0 || nbig != 1) ok = false;
        }
        if (ok) {
          for (const Comp* c = c0; c != c1; ++c) ccomp[c->c] = c;
          for (size_t i = 0; ok && i < Lv.size(); ++i) {
            const Comp* c = ccomp[Lv[i]];
            ok = c && (b_small ? c->a[0] : c->b[0]) == Lg[i];
          }
          for (const Comp* c = c0; c != c1; ++c) ccomp[c->c] = nullptr;
        }
      } else if (eff[sm].size() == 0 && unit_when_sliced(sm)) {
        // a unit piece whose indices are all (implied-)sliced: the selected
        // scalar is 1.0 for every slice, C = A * 1.0 == A
        ok = true;
        for (const Comp* c = c0; ok && c != c1; ++c) {
          const int nbig = b_small ? c->na : c->nb;
          if (c->c < 0 || nbig != 1) ok = false;
        }
        if (ok) {
          for (const Comp* c = c0; c != c1; ++c) ccomp[c->c] = c;
          for (size_t i = 0; ok && i < Lv.size(); ++i) {
            const Comp* c = ccomp[Lv[i]];
            ok = c && (b_small ? c->a[0] : c->b[0]) == Lg[i];
          }
          for (const Comp* c = c0; c != c1; ++c) ccomp[c->c] = nullptr;
        }
      } else if (p.sets[sm].size() == 2 && eff[sm].size() == 2) {
        // dense identity piece: one summed index s, one new index f
        int s = -1, f = -1, nk = 0, nf = 0;
        for (const Comp* c = c0; c != c1; ++c) {
          const int nbig = b_small ? c->na : c->nb;
          if (c->c < 0) s = b_small ? c->a[0] : c->b[0], nk++;
          else if (nbig == 0) f = c->c, nf++;
        }
        const double* q = p.lval.data() + p.lval_off[sm];
        ok = nk == 1 && nf == 1 && q[0] == 1.0 && q[3] == 1.0 && q[1] == 0.0 && q[2] == 0.0;
        for (size_t i = 0; ok && i < Lv.size(); ++i) ok = Lv[i] == Lg[i] || (Lg[i] == s && Lv[i] == f);
      }
      if (!ok) continue;
      g.cls[v] = NC_ALIAS;
      alias_src[v] = big;
      g.n_alias++;
    }
  }

  // ---- slice order: which chosen indices vary fastest ------------------------
  // msk[s]: the chosen indices (bit = lexicographic position) slot s depends on
  // (a sliced leaf holds them, a tied index counts as its source).  A per-slice
  // node whose mask misses every "fast" index runs once per block (the slices
  // that differ only in the fast indices, consecutive in iteration order).  The
  // fast set minimises the executed bytes of a pass; the first three chosen
  // indices stay slow, so ranges that fix them (the rank blocks of up to 8
  // GPUs, the timed samples) map onto themselves.  TC_SLICE_ORDER=0 keeps the
  // reference's order (fast = the last chosen index only); TC_BLOCK=0 runs
  // every variant node per slice.
  const int nch = (int)g.chosen.size();
  std::vector<uint64_t> msk(S, 0);
  uint64_t fast_mask = 0;
  std::vector<int> iter_order;  // chosen positions, slowest first
  for (int j = 0; j < nch; ++j) iter_order.push_back(j);
  {
    std::vector<int> chosen_pos(p.NI, -1);
    for (int j = 0; j < nch; ++j) chosen_pos[g.chosen[j]] = j;
    const bool block_env = !(std::getenv("TC_BLOCK") && std::atoi(std::getenv("TC_BLOCK")) == 0);
    const bool order_env = !(std::getenv("TC_SLICE_ORDER") && std::atoi(std::getenv("TC_SLICE_ORDER")) == 0);
    const bool hoist_on = !(std::getenv("TC_HOIST") && std::atoi(std::getenv("TC_HOIST")) == 0);
    if (nch >= 1 && nch <= 62 && block_env && hoist_on) {
      for (int l = 0; l < p.NL; ++l)
        for (int i : p.ref_order[l])
          if (pdrop[i]) msk[l] |= 1ull << chosen_pos[drop[i] ? i : implied_src[i]];
      // per-mask executed bytes of the variant nodes
      std::map<uint64_t, double> wb;
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k, a = p.left[k], b = p.right[k];
        msk[v] = msk[a] | msk[b];  // (a relabel alias carries its source's mask: the union is the same)
        if (msk[v]) wb[msk[v]] += 8.0 * (double)(size[a] + size[b] + size[v]);
      }
      // candidates: the chosen indices after the first three; for many-index
      // slice sets (more than 12 -- C3's 30 -- run in ranges of a few hundred
      // slices, whose free indices are the last ones) only the last 8, so an
      // aligned range of 256 slices stays closed
      const int keep = nch > 12 ? nch - 8 : std::min(3, nch - 1);
      std::vector<int> cand;
      for (int j = keep; j < nch; ++j) cand.push_back(j);
      double NS = (double)g.num_slices, best = -1;
      auto cost = [&](uint64_t fm) {
        double B = 1;
        for (int j = 0; j < nch; ++j)
          if (fm >> j & 1) B *= g.chosen_dim[j];
        double c = 0;
        for (auto& [m, b] : wb) c += b * ((m & fm) ? NS : NS / B);
        return c;
      };
      if (order_env) {
        for (uint64_t sub = 1; sub < (1ull << cand.size()); ++sub) {
          uint64_t fm = 0;
          for (size_t q = 0; q < cand.size(); ++q)
            if (sub >> q & 1) fm |= 1ull << cand[q];
          const double c = cost(fm);
          if (best < 0 || c < best * (1 - 1e-12)) best = c, fast_mask = fm;
        }
      } else {
        fast_mask = 1ull << (nch - 1);
      }
      iter_order.clear();
      for (int j = 0; j < nch; ++j)
        if (!(fast_mask >> j & 1)) iter_order.push_back(j);
      for (int j = 0; j < nch; ++j)
        if (fast_mask >> j & 1) iter_order.push_back(j);
    }
  }
  g.ord_dim.assign(g.chosen_dim.begin(), g.chosen_dim.end());
  g.ord_pv_lex.assign(nch, 1);
  for (int j = nch - 2; j >= 0; --j) g.ord_pv_lex[j] = g.ord_pv_lex[j + 1] * g.chosen_dim[j + 1];
  g.ord_pv_iter.assign(nch, 1);
  for (int q = nch - 2; q >= 0; --q)
    g.ord_pv_iter[iter_order[q]] = g.ord_pv_iter[iter_order[q + 1]] * g.chosen_dim[iter_order[q + 1]];
  for (int q = 0; q < nch; ++q)
    if (iter_order[q] != q) {
      g.permuted = true;
      g.closed_granule = g.ord_pv_lex[q] * g.chosen_dim[q];
      break;
    }

  tmark("leaves");
  // ---- leaves: plain, compressed, or per-slice selected ----------------------
  g.loc.assign(S, Loc{LOC_LEAF, 0});
  const std::vector<int64_t>& pv = g.ord_pv_iter;  // k_select decodes the iteration id
  std::vector<int> chosen_slot(p.NI, -1);
  for (size_t j = 0; j < g.chosen.size(); ++j) chosen_slot[g.chosen[j]] = (int)j;
  const int64_t nraw = (int64_t)p.lval.size();
  for (int l = 0; l < p.NL; ++l) {
    const auto& ro = p.ref_order[l];
    bool sl = false;
    for (int i : ro) sl |= (bool)pdrop[i];
    if (!sl) {
      // compressed leaves follow the raw values in the device leaf buffer
      g.loc[l] = cval_off[l] >= 0 ? Loc{LOC_LEAF, nraw + cval_off[l]} : Loc{LOC_LEAF, p.lval_off[l]};
      continue;
    }
    g.loc[l] = Loc{LOC_SLICED, g.sliced_doubles};
    auto stride = leaf_strides(l);
    int32_t t0 = (int32_t)g.sel_terms.size();
    for (size_t q = 0; q < ro.size(); ++q)
      if (pdrop[ro[q]]) {
        int j = chosen_slot[drop[ro[q]] ? ro[q] : implied_src[ro[q]]];
        g.sel_terms.push_back(SelTerm{pv[j], g.chosen_dim[j], stride[q]});
      }
    int32_t nt = (int32_t)g.sel_terms.size() - t0;
    // physical entries in layout order (LSB-first = reversed ref order)
    for (int64_t e = 0; e < size[l]; ++e)
      g.sel_ent.push_back(SelEntry{g.sliced_doubles + e, p.lval_off[l] + leaf_entry_src(l, e, stride), t0, nt});
    g.sliced_doubles += size[l];
  }

  // ---- slice-invariant hoisting ---------------------------------------------
  // The reference re-executes the whole tree per slice (slicing.py:139-145).
  // A node none of whose leaves holds a sliced index computes the same tensor
  // for every slice, so it runs once per pass over the slices (the runtime's
  // prologue graph) and only the `variant` nodes run per slice.  Variance is
  // data flow: a sliced leaf is variant, a node is variant iff an operand is
  // (an alias node is its source's buffer, so it inherits the source's).
  // An invariant tensor read by a variant node ("boundary") must survive every
  // slice: it lives in a pinned region at the start of the arena that the
  // postorder simulation never hands out again.  Every other buffer keeps the
  // simulation's offsets: the prologue finishes before the first slice, so an
  // invariant tensor that only invariant nodes read may share memory with
  // variant ones.  TC_HOIST=0 re-runs everything per slice (bit-identical).
  const bool hoist_env = !(std::getenv("TC_HOIST") && std::atoi(std::getenv("TC_HOIST")) == 0);
  const bool hoist = hoist_env && !g.chosen.empty();
  std::vector<char> var_(S, 0), boundary(S, 0);
  const int hoist_dbg = std::getenv("TC_HOIST_DBG") ? std::atoi(std::getenv("TC_HOIST_DBG")) : 0;
  if (hoist) {
    for (int l = 0; l < p.NL; ++l) var_[l] = g.loc[l].kind == LOC_SLICED;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      var_[v] = g.cls[v] == NC_ALIAS ? var_[alias_src[v]] : (char)(var_[p.left[k]] | var_[p.right[k]]);
      if (hoist_dbg && ((hoist_dbg & 1) && g.cls[v] == NC_TINY)) var_[v] = 1;  // diagnostics: keep class per slice
      if (hoist_dbg && ((hoist_dbg & 2) && g.cls[v] == NC_GEMM)) var_[v] = 1;
      if (hoist_dbg && ((hoist_dbg & 4) && g.cls[v] == NC_STREAM)) var_[v] = 1;
    }
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      if (var_[v] || g.cls[v] == NC_ALIAS) continue;
      // the node that reads v's buffer: look through aliases of it
      int cur = v, u = p.parent[v];
      while (u >= 0 && g.cls[u] == NC_ALIAS && alias_src[u] == cur) cur = u, u = p.parent[u];
      if (u >= 0 && g.cls[u] == NC_ALIAS) continue;  // the tie-piece side of an alias: never read
      boundary[v] = u < 0 || var_[u];                 // the root is read by k_rootcopy every slice
    }
    g.hoisted = true;
  }
  // ---- slice blocks -----------------------------------------------------------
  // Slices run in lexicographic order, the last chosen index fastest, so the
  // block_dim consecutive slices that differ only in it form a block.  A
  // per-slice node none of whose leaves holds that index (or an index tied to
  // it) computes the same tensor for every slice of a block: it runs once per
  // block (the runtime's block graph, on the block's lane before its slices).
  // Its tensors live in their own lane-private memory class (class 2), and
  // the ones read by per-slice nodes ("block boundary") are never released,
  // so they survive the block.  TC_BLOCK=0 runs them per slice (bit-identical).
  std::vector<char> blk_(S, 0), blkb(S, 0);
  if (hoist && fast_mask) {
    bool any = false;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      const uint64_t m = g.cls[v] == NC_ALIAS ? msk[alias_src[v]] : msk[v];
      blk_[v] = var_[v] && !(m & fast_mask);
      any = any || (blk_[v] && g.cls[v] != NC_ALIAS);
    }
    if (any) {
      g.block_dim = 1;
      for (int j = 0; j < nch; ++j)
        if (fast_mask >> j & 1) g.block_dim *= g.chosen_dim[j];
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k;
        if (!blk_[v] || g.cls[v] == NC_ALIAS) continue;
        int cur = v, u = p.parent[v];
        while (u >= 0 && g.cls[u] == NC_ALIAS && alias_src[u] == cur) cur = u, u = p.parent[u];
        if (u >= 0 && g.cls[u] == NC_ALIAS) continue;  // the tie-piece side of an alias: never read
        blkb[v] = u < 0 || !blk_[u];                    // read per slice (or by k_rootcopy)
      }
    } else {
      std::fill(blk_.begin(), blk_.end(), 0);
    }
  }
  // arena memory class: 1 slice-invariant, 2 block tier, 0 per slice
  auto mcl = [&](int slot) { return hoist && !var_[slot] ? 1 : blk_[slot] ? 2 : 0; };
  // a block-boundary buffer (looked up through relabel aliases) is never released
  auto kept = [&](int slot) {
    while (slot >= p.NL && g.cls[slot] == NC_ALIAS) slot = alias_src[slot];
    return (bool)blkb[slot];
  };

  tmark("tiny groups");
  // ---- tiny groups -------------------------------------------------------------
  std::vector<char> forced(S, 0);
  std::vector<std::vector<int>> groups;  // internal slots, postorder
  std::vector<int> group_of(S, -1);
  std::vector<int32_t> group_smem;
  auto is_tiny = [&](int s) { return !p.is_leaf(s) && g.cls[s] == NC_TINY; };
  auto is_troot = [&](int s) {
    return is_tiny(s) && (forced[s] || p.parent[s] < 0 || !is_tiny(p.parent[s]));
  };
  // A group is evaluated node after node by one CTA, so its cost is its node
  // count, while the subtree's critical path is its depth (C3's largest tiny
  // subtree: 5043 nodes, depth 177).  Along every node's deeper tiny child
  // the group continues; the other child becomes a group of its own (a root
  // in global memory, evaluated by another CTA of an earlier level) when its
  // subtree has >= TC_TINY_SPLIT nodes and the node's subtree is bushy (0: one
  // group per tiny subtree).
  {
    static const int split = std::getenv("TC_TINY_SPLIT") ? std::atoi(std::getenv("TC_TINY_SPLIT")) : 8;
    if (split > 0) {
      std::vector<int> cnt_t(S, 0), dep_t(S, 0);
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k, a = p.left[k], b = p.right[k];
        if (!is_tiny(v)) continue;
        const int ca = is_tiny(a) ? cnt_t[a] : 0, cb = is_tiny(b) ? cnt_t[b] : 0;
        const int da = is_tiny(a) ? dep_t[a] : 0, db = is_tiny(b) ? dep_t[b] : 0;
        cnt_t[v] = 1 + ca + cb;
        dep_t[v] = 1 + std::max(da, db);
        // only inside bushy subtrees (nodes >= 8x depth): cutting a near-chain
        // adds levels (launches) without shortening its critical path (C2)
        if (is_tiny(a) && is_tiny(b) && cnt_t[v] >= 8 * dep_t[v]) {
          const int light = (da > db || (da == db && ca >= cb)) ? b : a;
          if (cnt_t[light] >= split) forced[light] = 1;
        }
      }
    }
  }
  // Each group root r collects its tiny subtree (stopping at other roots) and
  // simulates first-fit smem in postorder; a group over the smem cap forces
  // r's tiny children to be roots and is re-collected (a group's node set
  // changes only through its own overflow, so a worklist reaches the same
  // fixpoint as re-grouping the whole forest).  Offsets are kept for the
  // descriptor pass below.
  std::vector<int32_t> soff(S, -1);  // smem offset of a non-root tiny node
  // TC_TINY_WAVES=0: one node after the other in postorder (round-1 order)
  static const bool waves_on = !(std::getenv("TC_TINY_WAVES") && std::atoi(std::getenv("TC_TINY_WAVES")) == 0);
  std::vector<int> hgt(S, 0);  // height within the node's tiny group
  {
    std::vector<std::pair<int, int32_t>> done;  // (root, peak)
    std::vector<std::vector<int>> gnodes;
    std::vector<int> work, nodes, st;
    SmemFit fit;
    for (int k = 0; k < p.NN; ++k)
      if (is_troot(p.NL + k)) work.push_back(p.NL + k);
    while (!work.empty()) {
      const int r = work.back();
      work.pop_back();
      for (;;) {
        nodes.clear();
        st.assign(1, r);
        while (!st.empty()) {
          int v = st.back();
          st.pop_back();
          nodes.push_back(v);
          for (int c : {p.kid_l(v), p.kid_r(v)})
            if (is_tiny(c) && !is_troot(c)) st.push_back(c);
        }
        std::sort(nodes.begin(), nodes.end());
        fit.reset();
        int32_t peak = 0;
        if (waves_on) {
          // waves: nodes of equal height within the group are independent and
          // run on different warps (k_tiny); smem is allocated wave by wave
          // (a wave's outputs, then the frees of its inputs)
          for (int v : nodes) {  // ascending slot = postorder: children first
            int h = 0;
            for (int c : {p.kid_l(v), p.kid_r(v)})
              if (is_tiny(c) && !is_troot(c)) h = std::max(h, hgt[c] + 1);
            hgt[v] = h;
          }
          std::stable_sort(nodes.begin(), nodes.end(), [&](int x, int y) { return hgt[x] < hgt[y]; });
          for (size_t w0 = 0; w0 < nodes.size();) {
            size_t w1 = w0;
            while (w1 < nodes.size() && hgt[nodes[w1]] == hgt[nodes[w0]]) ++w1;
            for (size_t q = w0; q < w1; ++q)
              if (nodes[q] != r) {
                soff[nodes[q]] = fit.alloc((int32_t)size[nodes[q]]);
                peak = std::max(peak, fit.top);
              }
            for (size_t q = w0; q < w1; ++q)
              for (int c : {p.kid_l(nodes[q]), p.kid_r(nodes[q])})
                if (c != r && is_tiny(c) && !is_troot(c)) fit.free(soff[c], (int32_t)size[c]);
            w0 = w1;
          }
        } else {
          for (int v : nodes) {
            if (v != r) {
              soff[v] = fit.alloc((int32_t)size[v]);
              peak = std::max(peak, fit.top);
            }
            for (int c : {p.kid_l(v), p.kid_r(v)})
              if (c != r && is_tiny(c) && !is_troot(c)) fit.free(soff[c], (int32_t)size[c]);
          }
        }
        if (peak > kTinySmemCap) {
          if (!is_tiny(p.kid_l(r)) && !is_tiny(p.kid_r(r))) fail(TC_BAD_ARG, "tiny split failed");
          for (int c : {p.kid_l(r), p.kid_r(r)})
            if (is_tiny(c) && !forced[c]) {
              forced[c] = 1;
              work.push_back(c);
            }
          continue;
        }
        done.push_back({r, peak});
        gnodes.push_back(nodes);
        break;
      }
    }
    // groups in postorder of their roots
    std::vector<int> ord(done.size());
    for (size_t q = 0; q < ord.size(); ++q) ord[q] = (int)q;
    std::sort(ord.begin(), ord.end(), [&](int x, int y) { return done[x].first < done[y].first; });
    for (int q : ord) {
      for (int v : gnodes[q]) group_of[v] = (int)groups.size();
      groups.push_back(std::move(gnodes[q]));
      group_smem.push_back(done[q].second);
    }
  }
  // group levels: a group consuming a forced root of another group runs later
  std::vector<int> glevel(groups.size(), 0);
  int nlevels = groups.empty() ? 0 : 1;
  for (size_t gi = 0; gi < groups.size(); ++gi) {  // groups are in postorder of roots
    for (int v : groups[gi])
      for (int c : {p.kid_l(v), p.kid_r(v)})
        if (is_tiny(c) && group_of[c] != (int)gi)
          glevel[gi] = std::max(glevel[gi], glevel[group_of[c]] + 1);
    nlevels = std::max(nlevels, glevel[gi] + 1);
  }
  // Level 0 splits into launches by when the chain first needs each group
  // (the consumer's position in emission order): the graph starts the
  // early-needed groups first and runs the rest beside the stream chain.
  int nbuckets = groups.empty() ? 0 : 1;
  if (!groups.empty() && !std::getenv("TC_TINY_ONE")) {
    std::vector<int> ord_nt(S, -1);
    int cnt2 = 0;
    for (int k = 0; k < p.NN; ++k)
      if (g.cls[p.NL + k] != NC_TINY && g.cls[p.NL + k] != NC_ALIAS) ord_nt[p.NL + k] = cnt2++;
    int n0 = 0;
    for (size_t gi = 0; gi < groups.size(); ++gi) n0 += glevel[gi] == 0;
    if (n0 >= 8 && cnt2 >= 16) {
      std::vector<int> bkt(groups.size(), 0);
      int used[4] = {0, 0, 0, 0};
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        if (glevel[gi] != 0) continue;
        int par = p.parent[groups[gi].back()];
        while (par >= 0 && g.cls[par] == NC_ALIAS) par = p.parent[par];
        const int c = par >= 0 ? ord_nt[par] : -1;
        const int b = c < cnt2 / 8 ? 0 : c < cnt2 / 4 ? 1 : c < cnt2 / 2 ? 2 : 3;
        bkt[gi] = b;
        used[b] = 1;
      }
      int remap[4], nb = 0;
      for (int b = 0; b < 4; ++b) remap[b] = used[b] ? nb++ : -1;
      for (size_t gi = 0; gi < groups.size(); ++gi) glevel[gi] = glevel[gi] == 0 ? remap[bkt[gi]] : glevel[gi] + nb - 1;
      nlevels += nb - 1;
      nbuckets = nb;
    }
  }
  if (std::getenv("TC_TINY_DEBUG")) {
    std::vector<size_t> sz;
    for (auto& gr : groups) sz.push_back(gr.size());
    std::sort(sz.rbegin(), sz.rend());
    int64_t work_max = 0, work_sum = 0;
    for (auto& gr : groups) {
      int64_t w = 0;
      for (int v : gr) w += size[v];
      work_max = std::max(work_max, w), work_sum += w;
    }
    {
      std::vector<int> ord_nt(S, -1);
      int cnt2 = 0;
      for (int k = 0; k < p.NN; ++k)
        if (g.cls[p.NL + k] != NC_TINY && g.cls[p.NL + k] != NC_ALIAS) ord_nt[p.NL + k] = cnt2++;
      std::vector<std::pair<int64_t, int>> gc;
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        int64_t w = 0;
        for (int v : groups[gi]) w += size[v] + 32;
        gc.push_back({w, (int)gi});
      }
      std::sort(gc.rbegin(), gc.rend());
      std::fprintf(stderr, "tiny heavy groups (cost, consumer ordinal of %d):", cnt2);
      for (size_t q = 0; q < gc.size() && q < 24; ++q) {
        int par = p.parent[groups[gc[q].second].back()];
        while (par >= 0 && g.cls[par] == NC_ALIAS) par = p.parent[par];
        std::fprintf(stderr, " (%lld,%d)", (long long)gc[q].first, par >= 0 ? ord_nt[par] : -1);
      }
      std::fprintf(stderr, "\n");
    }
    std::fprintf(stderr, "tiny: %zu groups, %d levels, nodes top:", groups.size(), nlevels);
    for (size_t q = 0; q < sz.size() && q < 12; ++q) std::fprintf(stderr, " %zu", sz[q]);
    std::fprintf(stderr, "  out-entries max %lld sum %lld smem max %d doubles\n", (long long)work_max,
                 (long long)work_sum, groups.empty() ? 0 : *std::max_element(group_smem.begin(), group_smem.end()));
  }

  tmark("steps + arena");
  // ---- steps + arena --------------------------------------------------------
  Alloc arena;
  {
    // Arena policy.  Reusing freed memory adds write-after-read edges that
    // serialise the launch DAG; when every intermediate fits in the HBM the
    // caller grants (no_reuse_limit), give each buffer its own memory so
    // independent branches of the tree run concurrently.
    int64_t total = 0;
    for (int k = 0; k < p.NN; ++k) {
      int v = p.NL + k;
      if (g.cls[v] != NC_TINY || p.parent[v] < 0 || g.cls[p.parent[v]] != NC_TINY)
        total += (size[v] * 8 + kAlign - 1) / kAlign * kAlign;
    }
    total += total / 8 + ((int64_t)1 << 20);  // split-K workspaces, alignment
    const char* env = std::getenv("TC_ARENA_REUSE");
    arena.no_reuse = env ? std::atoi(env) == 0 : total <= no_reuse_limit;
  }
  std::vector<int> producer(S, -1);
  int sel_step = -1;
  if (!g.sel_ent.empty()) {
    Step st;
    st.kind = ST_SELECT;
    sel_step = (int)g.steps.size();
    g.steps.push_back(st);
    for (int l = 0; l < p.NL; ++l)
      if (g.loc[l].kind == LOC_SLICED) producer[l] = sel_step;
  }
  std::vector<int64_t> bytes(S);
  for (int s = 0; s < S; ++s) bytes[s] = size[s] * 8;
  if (hoist) {  // the pinned region: boundary tensors that live in the arena
    std::vector<char> groot(S, 0);
    for (auto& gr : groups) groot[gr.back()] = 1;
    // a forced root is read by its consumer's GROUP launch, which runs per
    // slice whenever the group's root is variant (even if the consuming node
    // itself is invariant)
    for (auto& gr : groups) {
      const int r = gr.back(), u = p.parent[r];
      if (u >= 0 && is_tiny(u) && !var_[r]) boundary[r] = var_[groups[group_of[u]].back()];
    }
    // the same for every arena tensor a tiny node reads (a group root or a
    // non-tiny node): the reading launch is the reader's group launch, whose
    // category (prologue / block / per slice) is its root's
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      if (g.cls[v] == NC_ALIAS || (is_tiny(v) && !groot[v])) continue;
      int cur = v, u = p.parent[v];
      while (u >= 0 && g.cls[u] == NC_ALIAS && alias_src[u] == cur) cur = u, u = p.parent[u];
      if (u < 0 || g.cls[u] == NC_ALIAS || !is_tiny(u)) continue;
      const int gr = groups[group_of[u]].back();
      if (!var_[v] && var_[gr]) boundary[v] = 1;
      if (blk_[v] && !blk_[gr]) blkb[v] = 1;
    }
    int64_t pin = 0;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      if (boundary[v] && (g.cls[v] != NC_TINY || groot[v])) pin += (bytes[v] + kAlign - 1) / kAlign * kAlign;
    }
    arena.reserve_pinned(pin);
    arena.split_classes();
    g.pinned_bytes = pin;
  }
  // tiny roots: arena outputs allocated up front
  std::vector<int> haz;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    int r = groups[gi].back();
    haz.clear();
    g.loc[r] = Loc{LOC_ARENA, boundary[r] ? arena.alloc_pinned(bytes[r]) : arena.alloc(bytes[r], haz, mcl(r))};
  }
  // one tiny launch per level, split by variance when hoisting (key = 2*level + variant)
  // key = H * level + category (0 prologue, 1 block, 2 per slice) when hoisting
  const int H = hoist ? 3 : 1;
  const int nkeys = H * nlevels;
  auto gkey = [&](size_t gi) {
    const int r = groups[gi].back();
    return hoist ? 3 * glevel[gi] + (!var_[r] ? 0 : blk_[r] ? 1 : 2) : glevel[gi];
  };
  std::vector<int> key_groups(nkeys, 0);
  for (size_t gi = 0; gi < groups.size(); ++gi) key_groups[gkey(gi)]++;
  std::vector<int> tiny_step(nkeys, -1);
  for (int kk = 0; kk < nkeys; ++kk) {
    if (!key_groups[kk]) continue;
    const int lv = kk / H, cat = kk % H;
    Step st;
    st.kind = ST_TINY;
    st.inv = hoist && cat == 0;
    st.blk = hoist && cat == 1;
    if (sel_step >= 0 && !st.inv) st.deps.push_back(sel_step);
    if (lv >= nbuckets)  // a later level reads forced roots of any level-0 launch
      for (int b = 0; b < kk; ++b) {
        if (tiny_step[b] < 0 || (hoist && (b / H >= lv || b % H > cat))) continue;
        st.deps.push_back(tiny_step[b]);
      }
    tiny_step[kk] = (int)g.steps.size();
    g.steps.push_back(st);
  }
  tmark("tiny descriptors");
  // tiny descriptors, ordered by level then group.  Digit strides are sums
  // over a component's variables (a diagonal read has two address bits).
  std::vector<int64_t> str_a(p.NI, 0), str_b(p.NI, 0);  // variable -> stride (0: absent)
  auto comp_strides = [&](const Comp* c, int64_t& sa, int64_t& sb) {
    sa = sb = 0;
    for (int t = 0; t < c->na; ++t) sa += str_a[c->a[t]];
    for (int t = 0; t < c->nb; ++t) sb += str_b[c->b[t]];
  };
  auto load_strides = [&](const std::vector<int>& La, const std::vector<int>& Lb) {
    int64_t st2 = 1;
    for (int i : La) {
      str_a[i] = st2;
      st2 *= p.dom[i];
    }
    st2 = 1;
    for (int i : Lb) {
      str_b[i] = st2;
      st2 *= p.dom[i];
    }
  };
  // Groups are independent: descriptors are built on worker threads over
  // contiguous ranges of the level-major group order and concatenated.
  std::vector<int> gorder;
  std::vector<std::pair<int32_t, int32_t>> level_range(nkeys);
  {
    std::vector<std::vector<int>> level_groups(nkeys);
    for (size_t gi = 0; gi < groups.size(); ++gi) level_groups[gkey(gi)].push_back((int)gi);
    // heaviest groups first (the block scheduler hands out CTAs in order, so
    // the long subtrees start at once on their own SMs); cost ~ outputs written
    // plus a per-node overhead
    std::vector<int64_t> gcost(groups.size(), 0);
    for (size_t gi = 0; gi < groups.size(); ++gi)
      for (int v : groups[gi]) gcost[gi] += size[v] + 32;
    for (auto& lg : level_groups)
      std::stable_sort(lg.begin(), lg.end(), [&](int x, int y) { return gcost[x] > gcost[y]; });
    for (int lv = 0; lv < nkeys; ++lv) {
      level_range[lv].first = (int32_t)gorder.size();
      for (int gi : level_groups[lv]) gorder.push_back(gi);
      level_range[lv].second = (int32_t)gorder.size();
    }
  }
  struct TinyOut {
    std::vector<TinyNode> nodes;
    std::vector<TinyDigit> digs;
    std::vector<Loc> ga, gb, go;
    std::vector<TinyGroup> grp;
    int32_t stage = 0, digmax = 0;
  };
  auto build_groups = [&](int q0, int q1, TinyOut& out) {
    std::vector<int64_t> sa_(p.NI, 0), sb_(p.NI, 0);
    std::vector<const Comp*> cc(p.NI, nullptr);
    // layout of a slot: materialised (leaves, group roots under big parents)
    // or the natural order, computed here for nodes inside tiny subtrees
    // computed layouts are cached for the group (a node's layout as output is
    // reused when its parent reads it as an operand)
    std::deque<std::vector<int>> natc;  // stable references across growth
    std::vector<int> nat_of(S, -1);
    std::vector<int> nat_used;
    auto lay = [&](int sl, int) -> const std::vector<int>& {
      if (!g.layout[sl].empty() || varsv(sl).size() == 0) return g.layout[sl];
      if (nat_of[sl] >= 0) return natc[nat_of[sl]];
      nat_of[sl] = (int)nat_used.size();
      nat_used.push_back(sl);
      if (natc.size() < nat_used.size()) natc.emplace_back();
      auto& o = natc[nat_of[sl]];
      o.clear();
      const auto ro = p.ref_order[sl];
      if (varsv(sl).size() == ro.size()) {  // untied, nothing sliced: variables are the indices
        for (auto it = ro.rbegin(); it != ro.rend(); ++it) o.push_back(*it);
        return o;
      }
      for (auto it = ro.rbegin(); it != ro.rend(); ++it) {
        if (pdrop[*it]) continue;
        const int var = var_of(sl, *it);
        if (std::find(o.begin(), o.end(), var) == o.end()) o.push_back(var);
      }
      return o;
    };
    auto strides2 = [&](const Comp* c, int64_t& sa, int64_t& sb) {
      sa = sb = 0;
      for (int t = 0; t < c->na; ++t) sa += sa_[c->a[t]];
      for (int t = 0; t < c->nb; ++t) sb += sb_[c->b[t]];
    };
    std::vector<int> slot;
    for (int q = q0; q < q1; ++q) {
      const int gi = gorder[q];
      const auto& nodes = groups[gi];
      const int r = nodes.back();
      TinyGroup tg;
      tg.beg = (int32_t)out.nodes.size();
      // wave bookkeeping: per-warp load of the current wave (least loaded
      // warp takes the next single-warp node)
      int cur_h = -1;
      double wload[(1 << kTinyThreadsLog) / 32] = {};
      for (int v : nodes) {
        int hv = 0;
        for (int c : {p.kid_l(v), p.kid_r(v)})
          if (c != r && group_of[c] == gi && soff[c] >= 0) hv = std::max(hv, hgt[c] + 1);
        if (hv != cur_h) {
          cur_h = hv;
          for (double& x : wload) x = 0;
        }
        const int a = p.kid_l(v), b = p.kid_r(v);
        TinyNode tn{};
        Loc la{LOC_SMEM, 0}, lb{LOC_SMEM, 0}, lo{LOC_SMEM, 0};
        auto opnd = [&](int c, Loc& l, int32_t& so) {
          if (c != r && group_of[c] == gi && soff[c] >= 0) {
            so = soff[c];
          } else {
            l = g.loc[c];  // leaf / sliced leaf / forced root in arena
            so = 0;
          }
        };
        opnd(a, la, tn.sa);
        opnd(b, lb, tn.sb);
        if (v == r) lo = g.loc[r];
        else tn.sout = soff[v];
        // digits: output variables in C's layout order, then the summed ones
        const auto& La = lay(a, 0);
        const auto& Lb = lay(b, 1);
        const auto& Lc = lay(v, 2);
        int64_t st2 = 1;
        for (int i : La) sa_[i] = st2, st2 *= p.dom[i];
        st2 = 1;
        for (int i : Lb) sb_[i] = st2, st2 *= p.dom[i];
        auto [c0, c1] = comps(v);
        for (const Comp* c = c0; c != c1; ++c)
          if (c->c >= 0) cc[c->c] = c;
        tn.dig = (int32_t)out.digs.size();
        bool p2 = true;
        for (int i : Lc) {
          int64_t sa, sb;
          strides2(cc[i], sa, sb);
          out.digs.push_back(TinyDigit{p.dom[i], (int32_t)sa, (int32_t)sb, 0});
          p2 &= (p.dom[i] == 2);
        }
        int64_t ssz = 1;
        int ns = 0;
        for (const Comp* c = c0; c != c1; ++c) {  // sorted by smallest variable
          if (c->c >= 0) {
            cc[c->c] = nullptr;
            continue;
          }
          int64_t sa, sb;
          strides2(c, sa, sb);
          const int d = p.dom[c->a[0]];
          out.digs.push_back(TinyDigit{d, (int32_t)sa, (int32_t)sb, 0});
          p2 &= (d == 2);
          ssz *= d;
          ++ns;
        }
        for (int i : La) sa_[i] = 0;
        for (int i : Lb) sb_[i] = 0;
        tn.nc = (int32_t)Lc.size();
        tn.ns = ns;
        tn.c_size = (int32_t)size[v];
        tn.s_size = (int32_t)ssz;
        tn.pow2 = p2 ? 1 : 0;
        // single-warp nodes (few outputs, short sums) run beside the other
        // nodes of their wave on their own warp; the rest use the whole CTA
        const bool single = waves_on && tn.c_size <= 32 && (p2 || ssz < 64) && (int64_t)tn.c_size * ssz <= 2048;
        const int tlog = single ? 5 : kTinyThreadsLog;
        // lanes per output: fill the node's threads, at most a warp, at most
        // the number of summed terms
        tn.lw = 0;
        while (tn.lw < 5 && (tn.c_size << (tn.lw + 1)) <= (1 << tlog) && (1 << (tn.lw + 1)) <= ssz) ++tn.lw;
        tn.wofs = -1;
        {
          const double cost = 24.0 + (double)tn.c_size * (double)ssz / (single ? 32.0 : 256.0);
          if (single) {
            int best = 0;
            for (int w = 1; w < (1 << kTinyThreadsLog) / 32; ++w)
              if (wload[w] < wload[best]) best = w;
            tn.wofs = best;
            wload[best] += cost;
          } else {
            double mx = 0;
            for (double x : wload) mx = std::max(mx, x);
            for (double& x : wload) x = mx + cost;
          }
        }
        out.nodes.push_back(tn);
        slot.push_back(v);
        out.ga.push_back(la);
        out.gb.push_back(lb);
        out.go.push_back(lo);
      }
      tg.end = (int32_t)out.nodes.size();
      // barriers: a node waits for the CTA only when it reads smem written,
      // or overwrites smem read or written, since the last barrier (batch
      // starts are barriers); nodes on the cooperative-reduce path are fenced
      {
        std::vector<std::pair<int32_t, int32_t>> ew, er;
        auto hit = [](const std::vector<std::pair<int32_t, int32_t>>& rs, int32_t b, int32_t e) {
          for (auto& x : rs)
            if (b < x.second && x.first < e) return true;
          return false;
        };
        bool prev_red = false, epoch_w0 = true;
        for (int q2 = tg.beg; q2 < tg.end; ++q2) {
          TinyNode& t = out.nodes[q2];
          const int v = slot[q2];
          const bool red = tiny_uses_reduce(t);
          // executed by warp 0 alone (its threads are the node's only active ones)
          const bool w0 = !waves_on && !red &&
                          ((t.pow2 && t.ns - t.lw <= kTinyMaxSum) ? (t.c_size << t.lw) <= 32 : t.c_size <= 32);
          std::pair<int32_t, int32_t> rd[2];
          int nr = 0;
          if (out.ga[q2].kind == LOC_SMEM) rd[nr++] = {t.sa, t.sa + (int32_t)size[p.kid_l(v)]};
          if (out.gb[q2].kind == LOC_SMEM) rd[nr++] = {t.sb, t.sb + (int32_t)size[p.kid_r(v)]};
          const bool wr = v != r;
          const int32_t wb = t.sout, we = t.sout + (int32_t)size[v];
          const bool batch0 = (q2 - tg.beg) % kTinyBatch == 0;
          bool need = red || prev_red || batch0;
          for (int k = 0; k < nr && !need; ++k) need = hit(ew, rd[k].first, rd[k].second);
          if (wr && !need) need = hit(ew, wb, we) || hit(er, wb, we);
          // a hazard among warp-0-only nodes needs only warp 0 to sync
          // (__syncwarp orders its shared-memory accesses); the CTA epoch
          // keeps running for the other warps
          if (need && !red && !prev_red && !batch0 && w0 && epoch_w0) {
            t.sync = 2;
          } else {
            if (need) ew.clear(), er.clear(), epoch_w0 = true;
            t.sync = need ? 1 : 0;
          }
          epoch_w0 = epoch_w0 && w0;
          for (int k = 0; k < nr; ++k) er.push_back(rd[k]);
          if (wr) ew.push_back({wb, we});
          prev_red = red;
        }
      }
      for (int x : nat_used) nat_of[x] = -1;
      nat_used.clear();
      // batches of kTinyBatch nodes: staging offsets of small global operands
      // (leaves, sliced leaves, small forced roots) and the digit block size
      for (int b0 = tg.beg; b0 < tg.end; b0 += kTinyBatch) {
        const int b1 = std::min(tg.end, b0 + kTinyBatch);
        int32_t cur = 0;
        auto stage = [&](const Loc& l, int64_t n, int32_t& st, int32_t& cnt) {
          st = -1;
          cnt = 0;
          if (l.kind == LOC_SMEM || n > kTinyStageMax) return;
          st = cur;
          cnt = (int32_t)n;
          cur += (int32_t)((n + 1) & ~1);
        };
        for (int q2 = b0; q2 < b1; ++q2) {
          TinyNode& t = out.nodes[q2];
          const int v = slot[q2];
          stage(out.ga[q2], size[p.kid_l(v)], t.sta, t.na);
          stage(out.gb[q2], size[p.kid_r(v)], t.stb, t.nb);
        }
        out.stage = std::max(out.stage, cur);
        const TinyNode& l = out.nodes[b1 - 1];
        out.digmax = std::max(out.digmax, l.dig + l.nc + l.ns - out.nodes[b0].dig);
      }
      out.grp.push_back(tg);
    }
  };
  {
    // split the group order into ranges of about equal node counts
    int64_t total = 0;
    for (int gi : gorder) total += (int64_t)groups[gi].size();
    static const int tmax = std::getenv("TC_TINY_THREADS") ? std::atoi(std::getenv("TC_TINY_THREADS")) : 4;
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(tmax, total / 2048));
    std::vector<int> cut{0};
    int64_t acc = 0;
    for (size_t q = 0; q < gorder.size(); ++q) {
      acc += (int64_t)groups[gorder[q]].size();
      if ((int)cut.size() < T && acc * T >= total * (int64_t)cut.size()) cut.push_back((int)q + 1);
    }
    while ((int)cut.size() <= T) cut.push_back((int)gorder.size());
    std::vector<TinyOut> outs(T);
    std::vector<std::thread> th;
    std::vector<double> wms(T, 0.0);
    auto timed = [&](int w) {
      const auto t0 = std::chrono::steady_clock::now();
      build_groups(cut[w], cut[w + 1], outs[w]);
      wms[w] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    for (int w = 1; w < T; ++w) th.emplace_back(timed, w);
    timed(0);
    for (auto& x : th) x.join();
    if (timing) {
      std::fprintf(stderr, "[compile]   tiny workers:");
      for (int w = 0; w < T; ++w) std::fprintf(stderr, " %.2f", wms[w]);
      std::fprintf(stderr, " ms\n");
      tmark("tiny: merge");
    }
    // concatenate the workers' outputs: sizes first, then each worker's part
    // copied to its offset on its own thread (no reallocation, page faults spread)
    std::vector<size_t> nb(T + 1, 0), db(T + 1, 0), gb(T + 1, 0);
    for (int w = 0; w < T; ++w) {
      nb[w + 1] = nb[w] + outs[w].nodes.size();
      db[w + 1] = db[w] + outs[w].digs.size();
      gb[w + 1] = gb[w] + outs[w].grp.size();
      g.tiny_stage_doubles = std::max(g.tiny_stage_doubles, outs[w].stage);
      g.tiny_dig_max = std::max(g.tiny_dig_max, outs[w].digmax);
    }
    g.tiny_nodes.resize(nb[T]);
    g.tiny_digits.resize(db[T]);
    g.tiny_ga.resize(nb[T]);
    g.tiny_gb.resize(nb[T]);
    g.tiny_gout.resize(nb[T]);
    g.tiny_groups.resize(gb[T]);
    auto place = [&](int w) {
      const TinyOut& o = outs[w];
      for (size_t i = 0; i < o.nodes.size(); ++i) {
        TinyNode tn = o.nodes[i];
        tn.dig += (int32_t)db[w];
        g.tiny_nodes[nb[w] + i] = tn;
      }
      std::copy(o.digs.begin(), o.digs.end(), g.tiny_digits.begin() + db[w]);
      std::copy(o.ga.begin(), o.ga.end(), g.tiny_ga.begin() + nb[w]);
      std::copy(o.gb.begin(), o.gb.end(), g.tiny_gb.begin() + nb[w]);
      std::copy(o.go.begin(), o.go.end(), g.tiny_gout.begin() + nb[w]);
      for (size_t i = 0; i < o.grp.size(); ++i)
        g.tiny_groups[gb[w] + i] = TinyGroup{o.grp[i].beg + (int32_t)nb[w], o.grp[i].end + (int32_t)nb[w]};
    };
    th.clear();
    for (int w = 1; w < T; ++w) th.emplace_back(place, w);
    place(0);
    for (auto& x : th) x.join();
    g.n_tiny = (int)g.tiny_nodes.size();
    tmark("tiny: resolve");
    if (std::getenv("TC_TINY_DEBUG")) {
      // crude per-group cost: per node, serial iterations of one thread
      double best = -1;
      size_t bg = 0;
      std::vector<double> cost(g.tiny_groups.size());
      for (size_t q = 0; q < g.tiny_groups.size(); ++q) {
        double c = 0;
        for (int i = g.tiny_groups[q].beg; i < g.tiny_groups[q].end; ++i) {
          const TinyNode& t = g.tiny_nodes[i];
          const int per = (1 << kTinyThreadsLog) >> t.lw;
          c += 20 + (double)((t.c_size + per - 1) / per) * ((t.s_size >> t.lw) + t.nc);
        }
        cost[q] = c;
        if (c > best) best = c, bg = q;
      }
      std::sort(cost.rbegin(), cost.rend());
      int nsync = 0;
      for (auto& t : g.tiny_nodes) nsync += t.sync;
      std::fprintf(stderr, "tiny barriers %d of %zu nodes; cost top:", nsync, g.tiny_nodes.size());
      for (size_t q = 0; q < cost.size() && q < 8; ++q) std::fprintf(stderr, " %.0f", cost[q]);
      std::fprintf(stderr, "\n");
      for (int i = g.tiny_groups[bg].beg; i < g.tiny_groups[bg].end; ++i) {
        const TinyNode& t = g.tiny_nodes[i];
        const int per = (1 << kTinyThreadsLog) >> t.lw;
        std::fprintf(stderr, "  c=%d s=%d nc=%d ns=%d lw=%d pow2=%d glob=%d%d%d cost=%d\n", t.c_size, t.s_size,
                     t.nc, t.ns, t.lw, t.pow2, t.ga != nullptr, t.gb != nullptr, t.gout != nullptr,
                     20 + ((t.c_size + per - 1) / per) * ((t.s_size >> t.lw) + t.nc));
      }
    }
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      g.tiny_smem_doubles = std::max(g.tiny_smem_doubles, group_smem[gi]);
      producer[groups[gi].back()] = tiny_step[gkey(gi)];
    }
    // resolve operand / output places for the kernel: sa / sb / sout become
    // offsets from the start of dynamic smem (staged operands included), -1
    // for a global operand or output (one select per operand on the device)
    const int32_t stage0 = g.tiny_smem_doubles + (1 << kTinyThreadsLog);
    for (size_t i = 0; i < g.tiny_nodes.size(); ++i) {
      TinyNode& t = g.tiny_nodes[i];
      t.sa = t.sta >= 0 ? stage0 + t.sta : (g.tiny_ga[i].kind == LOC_SMEM ? t.sa : -1);
      t.sb = t.stb >= 0 ? stage0 + t.stb : (g.tiny_gb[i].kind == LOC_SMEM ? t.sb : -1);
      t.sout = g.tiny_gout[i].kind == LOC_SMEM ? t.sout : -1;
    }
  }
  tmark("tiny: release");
  // forced roots consumed inside a tiny level: release with that level as reader
  for (size_t gi = 0; gi < groups.size(); ++gi)
    for (int v : groups[gi])
      for (int c : {p.kid_l(v), p.kid_r(v)})
        if (is_tiny(c) && group_of[c] != (int)gi)
          if (!kept(c)) arena.release(g.loc[c].off, bytes[c], tiny_step[gkey(gi)], mcl(c));
  // store level ranges in the TINY steps (reuse `work` / gdig_off fields)
  for (int lv = 0; lv < nkeys; ++lv) {
    if (tiny_step[lv] < 0) continue;
    g.steps[tiny_step[lv]].gdig_off = level_range[lv].first;
    g.steps[tiny_step[lv]].work = level_range[lv].second - level_range[lv].first;
  }

  tmark("node work");
  // physical (executed) work per node: operands and output once, 2*prod of
  // the component domains flops
  std::vector<double> node_bytes(S, 0.0), node_flops(S, 0.0);
  for (int k = 0; k < p.NN; ++k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    double fl = 2;
    for (auto [c, ce] = comps(v); c != ce; ++c) fl *= p.dom[c->na ? c->a[0] : c->b[0]];
    node_bytes[v] = 8.0 * (double)(size[a] + size[b] + size[v]);
    node_flops[v] = fl;
    if (g.cls[v] != NC_ALIAS) {
      g.phys_bytes += (u128)(8 * (size[a] + size[b] + size[v]));
      g.phys_flops += (u128)fl;
      if (hoist && !var_[v]) {
        g.phys_bytes_inv += (u128)(8 * (size[a] + size[b] + size[v]));
        g.phys_flops_inv += (u128)fl;
      } else if (blk_[v]) {
        g.phys_bytes_blk += (u128)(8 * (size[a] + size[b] + size[v]));
        g.phys_flops_blk += (u128)fl;
      }
    }
  }

  if (hoist && std::getenv("TC_DEP_STATS")) {
    // diagnostics: per variant node, the fastest chosen index it depends on
    // (kmax): in lexicographic slice order its tensor changes only every
    // prod(dims after kmax) slices -- the work a prefix-level hoist would run
    const int nc = (int)g.chosen.size();
    std::vector<int> kmax(S, -1);
    std::vector<int> chosen_pos(p.NI, -1);
    for (int j = 0; j < nc; ++j) chosen_pos[g.chosen[j]] = j;
    for (int l = 0; l < p.NL; ++l)
      for (int i : p.ref_order[l])
        if (pdrop[i]) kmax[l] = std::max(kmax[l], chosen_pos[drop[i] ? i : implied_src[i]]);
    std::vector<double> by(nc + 1, 0.0);
    std::vector<int> cnt_by(nc + 1, 0);
    double now = 0, pre = 0;
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k;
      kmax[v] = g.cls[v] == NC_ALIAS ? kmax[alias_src[v]] : std::max(kmax[p.left[k]], kmax[p.right[k]]);
      if (g.cls[v] == NC_ALIAS || !var_[v]) continue;
      double reps = 1;
      for (int j = 0; j <= kmax[v]; ++j) reps *= g.chosen_dim[j];
      by[kmax[v] + 1] += node_bytes[v];
      cnt_by[kmax[v] + 1]++;
      now += node_bytes[v] * (double)g.num_slices;
      pre += node_bytes[v] * reps;
    }
    if (nc <= 62) {  // per dependence mask (bit j = chosen[j]): node count, per-slice bytes
      std::vector<uint64_t> mask(S, 0);
      for (int l = 0; l < p.NL; ++l)
        for (int i : p.ref_order[l])
          if (pdrop[i]) mask[l] |= 1ull << chosen_pos[drop[i] ? i : implied_src[i]];
      std::map<uint64_t, std::pair<int, double>> bym;
      for (int k = 0; k < p.NN; ++k) {
        const int v = p.NL + k;
        mask[v] = g.cls[v] == NC_ALIAS ? mask[alias_src[v]] : (mask[p.left[k]] | mask[p.right[k]]);
        if (g.cls[v] == NC_ALIAS || !var_[v]) continue;
        bym[mask[v]].first++;
        bym[mask[v]].second += node_bytes[v];
      }
      for (auto& [m, cb] : bym) std::fprintf(stderr, "[depmask] %llx %d %.0f\n", (unsigned long long)m, cb.first, cb.second);
    }
    std::fprintf(stderr, "[deps] per-slice bytes by fastest chosen index (0 = slowest):");
    for (int j = 1; j <= nc; ++j) std::fprintf(stderr, " k%d:%d nodes %.2f GB", j - 1, cnt_by[j], by[j] / 1e9);
    std::fprintf(stderr, "\n[deps] variant bytes per pass: per slice %.1f GB, prefix-level hoist %.1f GB\n", now / 1e9,
                 pre / 1e9);
  }

  tmark("emit nodes");
  struct Pending {
    int64_t off, bytes;
    int reader, cl;
  };
  std::vector<Pending> pending;
  auto flush_pending = [&]() {
    for (auto& q : pending) arena.release(q.off, q.bytes, q.reader, q.cl);
    pending.clear();
  };
  struct StreamOut {
    StreamParams sp{};
    int ns = 0, nf = 0, big = -1, sm = -1;
  };
  // stream-kernel parameters of node v (false: the shape does not fit k_stream)
  auto build_stream = [&](int v, StreamOut& o) -> bool {
    const int k = v - p.NL, a = p.left[k], b = p.right[k];
    const auto& Lc = g.layout[v];
    auto [c0, c1] = comps(v);
    try {
      const bool b_small = eff[b].size() <= eff[a].size();
      const int big = b_small ? a : b, sm = b_small ? b : a;
      const auto& Lg = g.layout[big];
      const auto& Lq = g.layout[sm];
      auto bigv = [&](const Comp* c) { return b_small ? c->a : c->b; };
      auto nbig = [&](const Comp* c) { return b_small ? c->na : c->nb; };
      auto smv = [&](const Comp* c) { return b_small ? c->b : c->a; };
      auto nsm = [&](const Comp* c) { return b_small ? c->nb : c->na; };
      SmallMap<int> pg, pc, pq;
      for (size_t q = 0; q < Lg.size(); ++q) pg[Lg[q]] = (int)q;
      for (size_t q = 0; q < Lc.size(); ++q) pc[Lc[q]] = (int)q;
      for (size_t q = 0; q < Lq.size(); ++q) pq[Lq[q]] = (int)q;
      K.clear();
      N.clear();
      for (const Comp* c = c0; c != c1; ++c) {
        if (c->c >= 0) ccomp[c->c] = c;
        if (c->c < 0) K.push_back(c);
        else if (nbig(c) == 0) N.push_back(c);
      }
      auto small_off = [&](const Comp* c) {
        int64_t o = 0;
        for (int t = 0; t < nsm(c); ++t) o += (int64_t)1 << pq[smv(c)[t]];
        return o;
      };
      // x bits: C variables with a big-side variable, in C address order
      std::vector<std::pair<int, int>> xa, xa2, xc;
      StreamParams sp{};
      int j = 0;
      bool bad = false;
      for (size_t q = 0; q < Lc.size(); ++q) {
        const Comp* c = ccomp[Lc[q]];
        if (nbig(c) == 0) continue;
        xc.push_back({j, (int)q});
        xa.push_back({j, pg[bigv(c)[0]]});
        if (nbig(c) == 2) xa2.push_back({j, pg[bigv(c)[1]]});
        if (nsm(c) > 0) {  // batch variable: also indexes the small operand
          if (sp.nbt == kStreamMaxBatch) bad = true;
          else {
            sp.bt_xbit[sp.nbt] = j;
            sp.bt_poff[sp.nbt] = small_off(c);
            sp.nbt++;
            if (j < kStreamChunkBits) sp.nlb++;
          }
        }
        j++;
      }
      std::sort(K.begin(), K.end(), [&](const Comp* x, const Comp* y) { return pg[bigv(x)[0]] < pg[bigv(y)[0]]; });
      for (const Comp* c = c0; c != c1; ++c)
        if (c->c >= 0) ccomp[c->c] = nullptr;
      if (bad) throw Error{-1, "batch"};
      sp.xa = make_runs(xa);
      sp.xa2 = make_runs(xa2);
      sp.xc = make_runs(xc);
      sp.nx = (int64_t)1 << j;
      const int ns = (int)K.size(), nf = (int)N.size();
      // N by C position, K by big-operand position
      std::sort(N.begin(), N.end(), [&](const Comp* x, const Comp* y) { return pc[x->c] < pc[y->c]; });
      for (int s = 0; s < (1 << ns); ++s) {
        int64_t o = 0, oq = 0;
        for (int t = 0; t < ns; ++t)
          if (s >> t & 1) {
            for (int u = 0; u < nbig(K[t]); ++u) o += (int64_t)1 << pg[bigv(K[t])[u]];
            oq += small_off(K[t]);
          }
        sp.offA[s] = o;
        for (int f = 0; f < (1 << nf); ++f) {
          int64_t of = 0;
          for (int t = 0; t < nf; ++t)
            if (f >> t & 1) of += small_off(N[t]);
          sp.offP[s * (1 << nf) + f] = (int32_t)(oq + of);
        }
      }
      for (int f = 0; f < (1 << nf); ++f) {
        int64_t o = 0;
        for (int t = 0; t < nf; ++t)
          if (f >> t & 1) o += (int64_t)1 << pc[N[t]->c];
        sp.offC[f] = o;
      }
      sp.stage_all = ((1 << sp.nbt) << (ns + nf)) <= kStreamStageMax;
      if (j > kStreamXBits) throw Error{-1, "x bits"};
      for (int jb = 0; jb < kStreamXBits; ++jb) {
        sp.bitA[jb] = deposit((uint64_t)1 << jb, sp.xa) + deposit((uint64_t)1 << jb, sp.xa2);
        sp.bitC[jb] = deposit((uint64_t)1 << jb, sp.xc);
        sp.bitP[jb] = 0;
        sp.bitPo[jb] = 0;
        for (int t = 0; t < sp.nbt; ++t)
          if (sp.bt_xbit[t] == jb) {
            sp.bitP[jb] = 1 << t;
            sp.bitPo[jb] = sp.bt_poff[t];
          }
      }
      o.sp = sp;
      o.ns = ns;
      o.nf = nf;
      o.big = big;
      o.sm = sm;
      return true;
    } catch (const Error& e) {
      if (e.status != -1) throw;
    }
    return false;
  };
  auto emit_node = [&](int v) {
    const int k = v - p.NL, a = p.left[k], b = p.right[k];
    Step st;
    st.slot = v;
    st.inv = hoist && !var_[v];
    st.blk = blk_[v];
    st.alg_bytes = node_bytes[v];
    st.alg_flops = node_flops[v];
    st.la = g.loc[a];
    st.lb = g.loc[b];
    for (int c : {a, b})
      if (producer[c] >= 0) st.deps.push_back(producer[c]);
    haz.clear();
    g.loc[v] = Loc{LOC_ARENA, boundary[v] ? arena.alloc_pinned(bytes[v]) : arena.alloc(bytes[v], haz, mcl(v))};
    for (int h : haz) st.deps.push_back(h);
    st.lc = g.loc[v];
    flush_pending();  // the previous node's inputs: free only now (see below)
    const auto& La = g.layout[a];
    const auto& Lb = g.layout[b];
    const auto& Lc = g.layout[v];
    auto [c0, c1] = comps(v);
    bool done = false;
    if (g.cls[v] == NC_STREAM) {
      StreamOut so;
      if (build_stream(v, so)) {
        st.kind = ST_STREAM;
        st.sp = so.sp;
        st.ns = so.ns;
        st.nf = so.nf;
        st.la = g.loc[so.big];
        st.lb = g.loc[so.sm];
        st.la_bytes = bytes[so.big];
        st.lb_bytes = bytes[so.sm];
        st.lc_bytes = bytes[v];
        st.work = so.sp.nx;
        g.n_stream++;
        done = true;
        if (std::getenv("TC_STREAM_STATS")) {  // diagnostics: low address bits of the stream shapes
          auto lowbit = [](int64_t v) { return v ? __builtin_ctzll((unsigned long long)v) : -1; };
          std::fprintf(stderr, "[stream] inv=%d nx=2^%d ns=%d nf=%d sbit0=%d fbit0=%d abit0=%d cbit0=%d nbt=%d stage=%d\n",
                       (int)st.inv, 63 - __builtin_clzll((unsigned long long)so.sp.nx), so.ns, so.nf,
                       so.ns ? lowbit(so.sp.offA[1]) : -1, so.nf ? lowbit(so.sp.offC[1]) : -1, lowbit(so.sp.bitA[0]),
                       lowbit(so.sp.bitC[0]), so.sp.nbt, so.sp.stage_all);
        }
      }
    }
    bool diag = false;
    for (const Comp* c = c0; c != c1; ++c) diag |= c->na > 1 || c->nb > 1;
    // GEMM: its own class, or a stream node whose shape the stream kernel
    // cannot stage (any layout works: the tile tables gather)
    if (!done && !diag && (g.cls[v] == NC_GEMM || g.cls[v] == NC_STREAM)) {
      try {
        K.clear();
        M.clear();
        N.clear();
        Bt.clear();
        for (const Comp* c = c0; c != c1; ++c) {
          if (c->c < 0) K.push_back(c);
          else if (c->na && c->nb) Bt.push_back(c);
          else if (c->na) M.push_back(c);
          else N.push_back(c);
        }
        SmallMap<int> pa, pb, pc;
        for (size_t q = 0; q < La.size(); ++q) pa[La[q]] = (int)q;
        for (size_t q = 0; q < Lb.size(); ++q) pb[Lb[q]] = (int)q;
        for (size_t q = 0; q < Lc.size(); ++q) pc[Lc[q]] = (int)q;
        auto by_c = [&](const Comp* x, const Comp* y) { return pc[x->c] < pc[y->c]; };
        std::sort(M.begin(), M.end(), by_c);
        std::sort(N.begin(), N.end(), by_c);
        std::sort(Bt.begin(), Bt.end(), by_c);
        std::sort(K.begin(), K.end(), [&](const Comp* x, const Comp* y) { return pa[x->a[0]] < pa[y->a[0]]; });
        const int m = (int)M.size(), n = (int)N.size(), kk = (int)K.size(), nbt = (int)Bt.size();
        // 128x64 CTA tiles (8 warps) for large GEMMs, 64x64 and below otherwise
        static const int big_tiles = std::getenv("TC_GEMM_BIG") ? std::atoi(std::getenv("TC_GEMM_BIG")) : 1;
        static const int big_k = std::getenv("TC_GEMM_BIG_K") ? std::atoi(std::getenv("TC_GEMM_BIG_K")) : 4;
        const bool big = big_tiles && m >= 7 && n >= 6 && kk >= big_k;
        // small-K GEMMs (K <= 2^smallk) are latency-bound on their prologue /
        // epilogue: tiles of at most 2^small_tile per side give more CTAs
        static const int smallk = std::getenv("TC_GEMM_SMALLK") ? std::atoi(std::getenv("TC_GEMM_SMALLK")) : -1;
        static const int small_tile = std::getenv("TC_GEMM_SMALLK_TILE") ? std::atoi(std::getenv("TC_GEMM_SMALLK_TILE")) : 5;
        const int tcap = (!big && kk <= smallk) ? small_tile : 6;
        const int MT = big ? 7 : std::max(3, std::min(tcap, m)), NT = std::max(3, std::min(tcap, n)), KT = 4;
        GemmParams gp{};
        gp.m_hi = std::max(0, m - MT);
        gp.n_hi = std::max(0, n - NT);
        gp.k_tiles = (int64_t)1 << std::max(0, kk - KT);
        gp.bt_bits = nbt;
        std::vector<std::pair<int, int>> r;
        auto runs = [&](const std::vector<const Comp*>& V, int from, auto var, SmallMap<int>& P) {
          r.clear();
          for (int t = from; t < (int)V.size(); ++t) r.push_back({t - from, P[var(V[t])]});
          return make_runs(r);
        };
        auto va = [](const Comp* c) { return c->a[0]; };
        auto vb = [](const Comp* c) { return c->b[0]; };
        auto vc = [](const Comp* c) { return c->c; };
        gp.a_m = runs(M, MT, va, pa);
        gp.a_k = runs(K, KT, va, pa);
        gp.b_n = runs(N, NT, vb, pb);
        gp.b_k = runs(K, KT, vb, pb);
        gp.c_m = runs(M, MT, vc, pc);
        gp.c_n = runs(N, NT, vc, pc);
        gp.a_bt = runs(Bt, 0, va, pa);
        gp.b_bt = runs(Bt, 0, vb, pb);
        gp.c_bt = runs(Bt, 0, vc, pc);
        auto tmap = [&](SmallMap<int>& P, const std::vector<const Comp*>& R1, auto v1, int n1,
                        const std::vector<const Comp*>& R2, auto v2, int n2) {
          // R1 tile bits -> kind 0, R2 tile bits -> kind 1; bits past the
          // shape are virtual (pos -1), placed after the real ones
          std::vector<std::tuple<int, int, int>> bits, virt;  // pos, kind, sub
          for (int t = 0; t < n1; ++t) {
            if (t < (int)R1.size()) bits.emplace_back(P[v1(R1[t])], 0, t);
            else virt.emplace_back(-1, 0, t);
          }
          for (int t = 0; t < n2; ++t) {
            if (t < (int)R2.size()) bits.emplace_back(P[v2(R2[t])], 1, t);
            else virt.emplace_back(-1, 1, t);
          }
          std::sort(bits.begin(), bits.end());
          bits.insert(bits.end(), virt.begin(), virt.end());
          TileMap tm{};
          tm.nbits = (int)bits.size();
          for (size_t q = 0; q < bits.size(); ++q) {
            tm.pos[q] = (int8_t)std::get<0>(bits[q]);
            tm.kind[q] = (int8_t)std::get<1>(bits[q]);
            tm.sub[q] = (int8_t)std::get<2>(bits[q]);
          }
          return tm;
        };
        gp.ta = tmap(pa, M, va, MT, K, va, KT);
        gp.tb = tmap(pb, N, vb, NT, K, vb, KT);
        gp.tc = tmap(pc, M, vc, MT, N, vc, NT);
        gp.grid_swizzle_log = std::min(gp.m_hi, 3);
        // split-K when the output tiles cannot fill the machine; skinny
        // memory-bound GEMMs (few 8x8 tiles, one warp per CTA) want many CTAs:
        // target 16 per SM (TC_SPLITK_MULT; C2 0.93 -> 0.89 ms, C3 unchanged)
        // The target is one wave of resident CTAs: 2 per SM for 128x64 tiles (8
        // warps), 4 for the 4-warp tiles, 16 for the skinny 1-2-warp ones (C3's
        // 1024x1024x4096 GEMM: 19 splits -> 3).
        const int64_t tiles = (int64_t)1 << (gp.m_hi + gp.n_hi + nbt);
        int64_t splits = 1;
        static const int64_t mult = std::getenv("TC_SPLITK_MULT") ? std::max(1, std::atoi(std::getenv("TC_SPLITK_MULT"))) : 0;
        const int64_t ctas = kSMs * (mult ? mult : (MT + NT >= 13 ? 2 : MT + NT >= 10 ? 4 : 16));
        // (at most one wave: a second, mostly idle wave costs more than the splits save)
        if (tiles < ctas && gp.k_tiles >= 8) splits = std::min<int64_t>(gp.k_tiles / 4, ctas / tiles);
        splits = std::max<int64_t>(1, splits);
        gp.k_per_split = (gp.k_tiles + splits - 1) / splits;
        gp.splits = (int32_t)((gp.k_tiles + gp.k_per_split - 1) / gp.k_per_split);
        st.kind = ST_GEMM;
        st.gp = gp;
        st.bm = MT;
        st.bn = NT;
        st.work = tiles;
        g.n_gemm++;
        done = true;
        if (std::getenv("TC_GEMM_STATS")) {  // diagnostics: GEMM shapes (log2), tiling, C's low address bits
          char cl[9] = "........";
          auto mark = [&](const std::vector<const Comp*>& V, char ch, int lim) {
            for (int t = 0; t < (int)V.size(); ++t) {
              const int q = pc[V[t]->c];
              if (q < 8) cl[q] = t < lim ? (char)(ch - 32) : ch;  // upper case: inside the CTA tile
            }
          };
          mark(M, 'm', MT);
          mark(N, 'n', NT);
          mark(Bt, 'b', 0);
          std::fprintf(stderr, "[gemm] inv=%d m=%d n=%d k=%d bt=%d tile=%dx%d tiles=%lld splits=%d clow=%s\n",
                       (int)st.inv, m, n, kk, nbt, MT, NT, (long long)tiles, gp.splits, cl);
        }
      } catch (const Error& e) {
        if (e.status != -1) throw;
      }
    }
    if (!done) {
      load_strides(La, Lb);
      for (const Comp* c = c0; c != c1; ++c)
        if (c->c >= 0) ccomp[c->c] = c;
      GenericParams np{};
      st.gdig_off = (int64_t)g.gdigits.size();
      for (int i : Lc) {
        int64_t sa, sb;
        comp_strides(ccomp[i], sa, sb);
        g.gdigits.push_back(GDigit{p.dom[i], sa, sb});
      }
      int64_t ssz = 1;
      int ns = 0;
      for (const Comp* c = c0; c != c1; ++c) {
        if (c->c >= 0) {
          ccomp[c->c] = nullptr;
          continue;
        }
        int64_t sa, sb;
        comp_strides(c, sa, sb);
        const int d = p.dom[c->a[0]];
        g.gdigits.push_back(GDigit{d, sa, sb});
        ssz *= d;
        ++ns;
      }
      for (int i : La) str_a[i] = 0;
      for (int i : Lb) str_b[i] = 0;
      np.c_size = size[v];
      np.s_size = ssz;
      np.nc = (int32_t)Lc.size();
      np.ns = ns;
      st.kind = ST_GENERIC;
      st.np = np;
      st.work = size[v];
      g.cls[v] = NC_GENERIC;
      g.n_generic++;
    }
    int me = (int)g.steps.size();
    if (st.kind == ST_GEMM && st.gp.splits > 1) {
      // split-K workspace: [splits][tiles][BM*BN] partial tiles, reduced in split order
      const int64_t ws_bytes = (int64_t)st.gp.splits * st.work * ((int64_t)1 << (st.bm + st.bn)) * 8;
      haz.clear();
      st.lws = Loc{LOC_ARENA, arena.alloc(ws_bytes, haz, mcl(v))};
      for (int h : haz) st.deps.push_back(h);
      g.steps.push_back(st);
      Step rd;
      rd.kind = ST_GEMM_REDUCE;
      rd.slot = v;
      rd.inv = st.inv;
      rd.blk = st.blk;
      rd.gp = st.gp;
      rd.bm = st.bm;
      rd.bn = st.bn;
      rd.la = st.la;
      rd.lb = st.lb;
      rd.lc = st.lc;
      rd.lws = st.lws;
      rd.work = st.work;
      rd.deps.push_back(me);
      producer[v] = me + 1;
      g.steps.push_back(rd);
      arena.release(st.lws.off, ws_bytes, me + 1, mcl(v));
    } else {
      producer[v] = me;
      g.steps.push_back(st);
    }
    // Inputs are released one node late: the next node's output never reuses
    // them, so a chain link (stream -> stream) may run fused in one kernel
    // that reads this node's inputs while writing the next node's output.
    // (only for a stream node whose parent is a stream node reading it as the
    // big operand: elsewhere the late release would only raise the peak)
    // (relabel aliases in between are the same buffer: look through them)
    int cur = v, par = p.parent[v];
    while (par >= 0 && g.cls[par] == NC_ALIAS) cur = par, par = p.parent[par];
    bool link = g.cls[v] == NC_STREAM && par >= 0 && g.cls[par] == NC_STREAM;
    if (link) {
      const int pk = par - p.NL, pa = p.left[pk], pb = p.right[pk];
      link = (eff[pb].size() <= eff[pa].size() ? pa : pb) == cur;
    }
    for (int c : {a, b})
      if (g.loc[c].kind == LOC_ARENA && !kept(c)) {
        if (link && bytes[c] <= kLateReleaseMax) pending.push_back({g.loc[c].off, bytes[c], me, mcl(c)});
        else arena.release(g.loc[c].off, bytes[c], me, mcl(c));
      }
  };

  for (int k = 0; k < p.NN; ++k) {
    const int v = p.NL + k;
    if (g.cls[v] == NC_TINY) {
      int gi = group_of[v];
      int ts = tiny_step[gkey(gi)];
      g.steps[ts].alg_bytes += node_bytes[v];
      g.steps[ts].alg_flops += node_flops[v];
      continue;
    }
    if (g.cls[v] == NC_ALIAS) {  // same buffer, same bits: ownership moves to v
      const int src = alias_src[v];
      g.loc[v] = g.loc[src];
      bytes[v] = bytes[src];
      producer[v] = producer[src];
      continue;
    }
    emit_node(v);
  }

  flush_pending();
  tmark("root copy");
  accounting.get();  // rethrows TC_OVERFLOW from the accounting thread
  g.mem_estimate = mem_est;
  g.peak_observed = peak_obs;
  g.alg_bytes = dense_bytes;
  g.alg_flops = dense_flops;
  // root copy into the per-slice result slot, then advance the slice counter.
  // The result is dense over the root's kept indices in the reference's
  // row-major order; a root with tied indices is expanded through root_map.
  g.R = (int64_t)dsize[p.root];
  g.root_loc = g.loc[p.root];
  if (g.R != size[p.root]) {
    const auto& ro = p.ref_order[p.root];
    const auto& Lr = g.layout[p.root];
    std::vector<int> kept;
    for (int i : ro)
      if (!pdrop[i]) kept.push_back(i);
    std::vector<int64_t> vstride(p.NI, 0);
    int64_t st2 = 1;
    for (int i : Lr) {
      vstride[i] = st2;
      st2 *= p.dom[i];
    }
    std::vector<int> var_digit(p.NI, -1);
    g.root_map.resize((size_t)g.R);
    for (int64_t r = 0; r < g.R; ++r) {
      int64_t rem = r, off = 0;
      bool ok = true;
      for (int q = (int)kept.size() - 1; q >= 0; --q) {
        const int d = (int)(rem % p.dom[kept[q]]);
        rem /= p.dom[kept[q]];
        const int var = var_of(p.root, kept[q]);
        if (var_digit[var] < 0) {
          var_digit[var] = d;
          off += d * vstride[var];
        } else if (var_digit[var] != d) {
          ok = false;
        }
      }
      for (int i : kept) var_digit[var_of(p.root, i)] = -1;
      g.root_map[r] = ok ? off : -1;
    }
  }
  Step rc;
  rc.kind = ST_ROOTCOPY;
  if (producer[p.root] >= 0) rc.deps.push_back(producer[p.root]);
  rc.work = g.R;
  int rcs = (int)g.steps.size();
  g.steps.push_back(rc);
  Step et;
  et.kind = ST_ETA;
  et.deps.push_back(rcs);
  if (sel_step >= 0) et.deps.push_back(sel_step);
  g.steps.push_back(et);
  tmark("end");
  // final arena layout [pinned | slice-invariant | per-slice]: relocate the
  // per-slice class's tagged offsets; a slice lane's private copy holds the
  // per-slice region only (the prologue's tensors are lane 0's)
  auto reloc = [&](Loc& l) {
    if (l.kind == LOC_ARENA) l.off = arena.relocate(l.off);
  };
  for (auto& l : g.loc) reloc(l);
  for (auto& st : g.steps) reloc(st.la), reloc(st.lb), reloc(st.lc), reloc(st.lws);
  for (auto* v : {&g.tiny_ga, &g.tiny_gb, &g.tiny_gout})
    for (auto& l : *v) reloc(l);
  reloc(g.root_loc);
  g.lane_base = arena.region0_base();
  g.arena_bytes = std::max<int64_t>(arena.arena_end(), kAlign);
  g.lane_arena_bytes = std::max<int64_t>(g.arena_bytes - g.lane_base, kAlign);
  if (timing)
    std::fprintf(stderr, "[compile] arena %.3f GB (pinned %.3f GB), lane copy %.3f GB\n", g.arena_bytes / 1e9,
                 arena.pin_end / 1e9, g.lane_arena_bytes / 1e9);
  for (auto& s : g.steps) {
    std::sort(s.deps.begin(), s.deps.end());
    s.deps.erase(std::unique(s.deps.begin(), s.deps.end()), s.deps.end());
  }
  return g;
}

}  // namespace tc
