// Host program compiler (see compile.hpp).
//
// What it decides, per internal node of the (sliced) contraction tree:
//   * kernel class — TINY (whole small subtrees evaluated in one CTA's shared
//     memory, many subtrees per launch), STREAM (big tensor x <=64-entry
//     operand, HBM-bound), GEMM (FP64 DMMA), GENERIC (mixed radix fallback);
//   * the memory layout of every intermediate.  The reference always emits
//     kept_a ++ kept_b (tensor.py:108) and numpy pays a transpose copy per
//     tensordot (60-70% of CPU time).  Here layouts are chosen
//     top-down so that a STREAM node's output is an in-place relabel of its
//     big input (shared bits of the input and free bits of the small operand
//     share address bits) and a GEMM's operands are K-lowest matrices; the
//     permutation is folded into the producing kernel's addressing and no
//     separate transpose pass exists;
//   * a static arena: offsets from a first-fit simulation in postorder, with
//     write-after-read edges added to the launch DAG wherever a buffer reuses
//     memory, so independent branches may run concurrently in the CUDA graph.
#include "compile.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <set>

namespace tc {

namespace {

constexpr int64_t kTinyMax = 4096;           // entries per tiny tensor
constexpr int32_t kTinySmemCap = 20 * 1024;  // doubles of smem per tiny CTA (160 KB)
constexpr int64_t kAlign = 256;
constexpr int64_t kSMs = 148;                // B200 SM count (split-K sizing)

[[noreturn]] void fail(int st, const std::string& m) { throw Error{st, m}; }

struct Alloc {
  std::map<int64_t, int64_t> free_;                   // off -> size
  std::map<int64_t, std::pair<int64_t, int>> seg;     // off -> (end, last reader step)
  int64_t top = 0;

  bool no_reuse = false;  // every buffer gets fresh memory: no WAR edges at all

  int64_t alloc(int64_t size, std::vector<int>& hazards) {
    size = (size + kAlign - 1) / kAlign * kAlign;
    if (no_reuse) {
      int64_t o = top;
      top += size;
      return o;
    }
    int64_t off = -1;
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second >= size) {
        off = it->first;
        int64_t rest = it->second - size;
        free_.erase(it);
        if (rest > 0) free_[off + size] = rest;
        break;
      }
    }
    if (off < 0) {
      // extend: reuse a free block touching the top
      if (!free_.empty()) {
        auto last = std::prev(free_.end());
        if (last->first + last->second == top) {
          off = last->first;
          free_.erase(last);
          top = off + size;
        }
      }
      if (off < 0) {
        off = top;
        top += size;
      }
    }
    // hazards: previous readers of any byte we are about to overwrite
    int64_t end = off + size;
    auto it = seg.upper_bound(off);
    if (it != seg.begin()) --it;
    while (it != seg.end() && it->first < end) {
      int64_t s0 = it->first, s1 = it->second.first;
      int rd = it->second.second;
      if (s1 <= off) {
        ++it;
        continue;
      }
      hazards.push_back(rd);
      it = seg.erase(it);
      if (s0 < off) seg[s0] = {off, rd};
      if (s1 > end) seg[end] = {s1, rd};
      it = seg.lower_bound(std::min(s1, end));
    }
    return off;
  }

  void release(int64_t off, int64_t size, int reader) {
    if (no_reuse) return;
    size = (size + kAlign - 1) / kAlign * kAlign;
    seg[off] = {off + size, reader};
    auto nx = free_.lower_bound(off);
    int64_t o = off, s = size;
    if (nx != free_.end() && nx->first == off + size) {
      s += nx->second;
      nx = free_.erase(nx);
    }
    if (nx != free_.begin()) {
      auto pv = std::prev(nx);
      if (pv->first + pv->second == o) {
        o = pv->first;
        s += pv->second;
        free_.erase(pv);
      }
    }
    free_[o] = s;
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
  size_t count(int k) const {
    for (auto& e : kv)
      if (e.first == k) return 1;
    return 0;
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
  g.mem_estimate = mem_cost(p, drop);
  g.peak_observed = tracked_peak(p, drop);

  tmark("effective sets / siz");
  // ---- effective sets / sizes ------------------------------------------------
  // eff[s]: the slot's index set without the sliced indices (a view of
  // p.sets when the slot holds none of them)
  std::vector<std::vector<int>> eff_own;
  std::vector<const std::vector<int>*> effp(S);
  {
    std::vector<int> own_of(S, -1);
    for (int s = 0; s < S; ++s) {
      bool any = false;
      for (int i : p.sets[s]) any |= (bool)drop[i];
      if (any) own_of[s] = (int)eff_own.size(), eff_own.emplace_back();
    }
    for (int s = 0; s < S; ++s) {
      if (own_of[s] < 0) {
        effp[s] = &p.sets[s];
        continue;
      }
      auto& e = eff_own[own_of[s]];
      for (int i : p.sets[s])
        if (!drop[i]) e.push_back(i);
      effp[s] = &e;
    }
  }
  struct EffView {
    const std::vector<const std::vector<int>*>* v;
    const std::vector<int>& operator[](int s) const { return *(*v)[s]; }
  } eff{&effp};
  std::vector<int64_t> size(S);
  for (int s = 0; s < S; ++s) {
    u128 z = set_bytes(p, eff[s], drop) / 8;
    if (z > ((u128)1 << 50)) fail(TC_OOM, "intermediate tensor larger than 2^50 entries");
    size[s] = (int64_t)z;
  }
  auto natural = [&](int s) {
    std::vector<int> o;
    const auto& ro = p.ref_order[s];
    o.reserve(ro.size());
    for (auto it = ro.rbegin(); it != ro.rend(); ++it)
      if (!drop[*it]) o.push_back(*it);
    return o;
  };
  auto inter = [](const std::vector<int>& a, const std::vector<int>& b) {
    std::vector<int> o;
    std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
    return o;
  };
  auto minus = [](const std::vector<int>& a, const std::vector<int>& b) {
    std::vector<int> o;
    std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
    return o;
  };
  auto has = [](const std::vector<int>& s, int i) { return std::binary_search(s.begin(), s.end(), i); };

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
      int ks = (int)inter(eff[a], eff[b]).size();
      int ra = (int)eff[a].size() - ks, rb = (int)eff[b].size() - ks;
      int f = (eff[b].size() <= eff[a].size()) ? rb : ra;  // free bits of the smaller operand
      (void)ra;
      (void)rb;
      if (ks <= 4 && f <= 4 && ks + f <= 6)
        c = NC_STREAM;
      else
        c = NC_GEMM;  // any m, n, k: tile bits beyond the shape are virtual
    } else {
      c = NC_GENERIC;
    }
    g.cls[v] = c;
  }

  tmark("layouts (top-down)");
  // ---- layouts (top-down) ----------------------------------------------------
  g.layout.assign(S, {});
  std::vector<char> have(S, 0);
  for (int l = 0; l < p.NL; ++l) {
    g.layout[l] = natural(l);
    have[l] = 1;
  }
  std::vector<int> pos(p.NI, -1);
  auto set_pos = [&](const std::vector<int>& L) {
    for (size_t q = 0; q < L.size(); ++q) pos[L[q]] = (int)q;
  };
  auto clr_pos = [&](const std::vector<int>& L) {
    for (int i : L) pos[i] = -1;
  };
  if (!p.is_leaf(p.root)) {
    g.layout[p.root] = natural(p.root);
    have[p.root] = 1;
  }
  auto want = [&](int child, std::vector<int> L) {
    if (p.is_leaf(child)) return;
    g.layout[child] = std::move(L);
    have[child] = 1;
  };
  for (int k = p.NN - 1; k >= 0; --k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    const std::vector<int>& L = g.layout[v];
    switch (g.cls[v]) {
      case NC_STREAM: {
        bool b_small = eff[b].size() <= eff[a].size();
        int big = b_small ? a : b, sm = b_small ? b : a;
        std::vector<int> Sh = inter(eff[a], eff[b]);
        std::vector<int> F = minus(eff[sm], Sh);
        std::vector<int> Lg;
        size_t si = 0;
        for (int i : L) {
          if (has(F, i)) {
            if (si < Sh.size()) Lg.push_back(Sh[si++]);
          } else {
            Lg.push_back(i);
          }
        }
        while (si < Sh.size()) Lg.push_back(Sh[si++]);
        want(big, Lg);
        if (!p.is_leaf(sm)) want(sm, natural(sm));
        break;
      }
      case NC_GEMM: {
        std::vector<int> K = inter(eff[a], eff[b]);
        std::vector<int> M = minus(eff[a], K), N = minus(eff[b], K);
        // K order: follow a fixed-layout (leaf) operand when there is one
        int ref = p.is_leaf(a) ? a : (p.is_leaf(b) ? b : -1);
        if (ref >= 0) {
          set_pos(g.layout[ref]);
          std::sort(K.begin(), K.end(), [&](int x, int y) { return pos[x] < pos[y]; });
          clr_pos(g.layout[ref]);
        }
        set_pos(L);
        std::sort(M.begin(), M.end(), [&](int x, int y) { return pos[x] < pos[y]; });
        std::sort(N.begin(), N.end(), [&](int x, int y) { return pos[x] < pos[y]; });
        clr_pos(L);
        std::vector<int> La = K, Lb = K;
        La.insert(La.end(), M.begin(), M.end());
        Lb.insert(Lb.end(), N.begin(), N.end());
        want(a, La);
        want(b, Lb);
        break;
      }
      default:
        if (!p.is_leaf(a)) want(a, natural(a));
        if (!p.is_leaf(b)) want(b, natural(b));
    }
  }

  tmark("exact relabels");
  // ---- exact relabels ---------------------------------------------------------
  // big x (2x2 identity) piece: C[.., f, ..] = sum_s A[.., s, ..] I[s, f] is A
  // with index s renamed f (x*1 + y*0 == x for finite y, bit for bit).  The
  // layout pass put f at s's address bit, so C IS A's buffer: no launch, no
  // traffic.  (In C2 these are 2004 of 2783 big x piece nodes: the
  // non-carrier pieces of factored copy tensors, factoring.py:194-206.)
  std::vector<int> alias_src(S, -1);
  if (!std::getenv("TC_NO_ALIAS")) {
    for (int k = 0; k < p.NN; ++k) {
      const int v = p.NL + k, a = p.left[k], b = p.right[k];
      if (g.cls[v] != NC_STREAM) continue;
      const bool b_small = eff[b].size() <= eff[a].size();
      const int big = b_small ? a : b, sm = b_small ? b : a;
      if (p.is_leaf(big) || !p.is_leaf(sm) || p.sets[sm].size() != 2 || eff[sm].size() != 2) continue;
      std::vector<int> Sh = inter(eff[a], eff[b]);
      std::vector<int> F = minus(eff[sm], Sh);
      if (Sh.size() != 1 || F.size() != 1) continue;
      const double* q = p.lval.data() + p.lval_off[sm];
      if (!(q[0] == 1.0 && q[3] == 1.0 && q[1] == 0.0 && q[2] == 0.0)) continue;
      const auto& Lv = g.layout[v];
      const auto& Lg = g.layout[big];
      bool same = Lv.size() == Lg.size();
      for (size_t i = 0; same && i < Lv.size(); ++i)
        same = Lv[i] == Lg[i] || (Lg[i] == Sh[0] && Lv[i] == F[0]);
      if (!same) continue;
      g.cls[v] = NC_ALIAS;
      alias_src[v] = big;
      g.n_alias++;
    }
  }

  tmark("chain segments");
  // ---- chain segments: runs of STREAM nodes fused into one launch -----------
  // v_{i+1}'s big operand is v_i.  Inner bits = every index of the input the
  // segment touches plus the ones it creates; all must fit kChainU at every
  // step (touching a new input index widens every earlier step too).
  struct Seg {
    std::vector<int> nodes, big, small;
    std::vector<int> u0;     // inner indices loaded with the input tile
    std::vector<int> inner;  // inner indices of the current output (sorted)
    std::vector<int> w;      // inner width before step 0 and after each step
  };
  std::vector<Seg> segs;
  std::vector<int> seg_of(S, -1);
  // smem chain fusion is opt-in (TC_CHAIN=1): measured slower than graph-
  // concurrent k_stream launches on C2/C1b
  const bool fuse_chains = std::getenv("TC_CHAIN") != nullptr;
  // fusion pays where launches dominate (small tensors); big tensors stream at
  // HBM speed through k_stream with L2 reuse between consecutive steps
  int chain_max_bits = 20;
  if (const char* e = std::getenv("TC_CHAIN_MAX_BITS")) chain_max_bits = std::atoi(e);
  for (int k = 0; k < p.NN && fuse_chains; ++k) {
    const int v = p.NL + k, a = p.left[k], b = p.right[k];
    if (g.cls[v] != NC_STREAM) continue;
    if ((int)std::max(eff[a].size(), eff[b].size()) > chain_max_bits || (int)eff[v].size() > chain_max_bits) continue;
    const bool b_small = eff[b].size() <= eff[a].size();
    const int big = b_small ? a : b, sm = b_small ? b : a;
    std::vector<int> Sh = inter(eff[a], eff[b]);
    std::vector<int> F = minus(eff[sm], Sh);
    if (!p.is_leaf(big) && seg_of[big] >= 0) {
      Seg& sg = segs[seg_of[big]];
      if (sg.nodes.back() == big && (int)sg.nodes.size() < kChainMax) {
        std::vector<int> s_orig = minus(Sh, sg.inner);
        std::vector<int> un;
        std::set_union(sg.inner.begin(), sg.inner.end(), Sh.begin(), Sh.end(), std::back_inserter(un));
        std::vector<int> nin = minus(un, Sh);
        std::vector<int> nin2;
        std::set_union(nin.begin(), nin.end(), F.begin(), F.end(), std::back_inserter(nin2));
        int mx = (int)nin2.size();
        for (int x : sg.w) mx = std::max(mx, x + (int)s_orig.size());
        if (mx <= kChainU) {
          for (int& x : sg.w) x += (int)s_orig.size();
          sg.w.push_back((int)nin2.size());
          for (int x : s_orig) sg.u0.push_back(x);
          sg.inner = nin2;
          sg.nodes.push_back(v);
          sg.big.push_back(big);
          sg.small.push_back(sm);
          seg_of[v] = seg_of[big];
          continue;
        }
      }
    }
    Seg sg;
    sg.nodes = {v};
    sg.big = {big};
    sg.small = {sm};
    sg.u0 = Sh;
    sg.inner = F;
    sg.w = {(int)Sh.size(), (int)F.size()};
    seg_of[v] = (int)segs.size();
    segs.push_back(sg);
  }

  tmark("leaves");
  // ---- leaves: plain or per-slice selected ----------------------------------
  g.loc.assign(S, Loc{LOC_LEAF, 0});
  std::vector<int64_t> pv(g.chosen.size(), 1);
  for (int j = (int)g.chosen.size() - 2; j >= 0; --j) pv[j] = pv[j + 1] * g.chosen_dim[j + 1];
  std::vector<int> chosen_slot(p.NI, -1);
  for (size_t j = 0; j < g.chosen.size(); ++j) chosen_slot[g.chosen[j]] = (int)j;
  for (int l = 0; l < p.NL; ++l) {
    const auto& ro = p.ref_order[l];
    bool sl = false;
    for (int i : ro) sl |= (bool)drop[i];
    if (!sl) {
      g.loc[l] = Loc{LOC_LEAF, p.lval_off[l]};
      continue;
    }
    g.loc[l] = Loc{LOC_SLICED, g.sliced_doubles};
    std::vector<int64_t> stride(ro.size());
    int64_t st = 1;
    for (int q = (int)ro.size() - 1; q >= 0; --q) {
      stride[q] = st;
      st *= p.dom[ro[q]];
    }
    int32_t t0 = (int32_t)g.sel_terms.size();
    for (size_t q = 0; q < ro.size(); ++q)
      if (drop[ro[q]]) {
        int j = chosen_slot[ro[q]];
        g.sel_terms.push_back(SelTerm{pv[j], g.chosen_dim[j], stride[q]});
      }
    int32_t nt = (int32_t)g.sel_terms.size() - t0;
    // effective entries in effective layout order (LSB-first = reversed ref order)
    std::vector<int> kq;  // positions in ro of kept indices, row-major order
    for (size_t q = 0; q < ro.size(); ++q)
      if (!drop[ro[q]]) kq.push_back((int)q);
    for (int64_t e = 0; e < size[l]; ++e) {
      int64_t rem = e, src = p.lval_off[l];
      for (int q = (int)kq.size() - 1; q >= 0; --q) {
        int64_t d = p.dom[ro[kq[q]]];
        src += (rem % d) * stride[kq[q]];
        rem /= d;
      }
      g.sel_ent.push_back(SelEntry{g.sliced_doubles + e, src, t0, nt});
    }
    g.sliced_doubles += size[l];
  }

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
  // Each group root r collects its tiny subtree (stopping at other roots) and
  // simulates first-fit smem in postorder; a group over the smem cap forces
  // r's tiny children to be roots and is re-collected (a group's node set
  // changes only through its own overflow, so a worklist reaches the same
  // fixpoint as re-grouping the whole forest).  Offsets are kept for the
  // descriptor pass below.
  std::vector<int32_t> soff(S, -1);  // smem offset of a non-root tiny node
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
        for (int v : nodes) {
          if (v != r) {
            soff[v] = fit.alloc((int32_t)size[v]);
            peak = std::max(peak, fit.top);
          }
          for (int c : {p.kid_l(v), p.kid_r(v)})
            if (c != r && is_tiny(c) && !is_troot(c)) fit.free(soff[c], (int32_t)size[c]);
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
  tmark("arena policy");
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
  // tiny roots: arena outputs allocated up front
  std::vector<int64_t> bytes(S);
  for (int s = 0; s < S; ++s) bytes[s] = size[s] * 8;
  std::vector<int> haz;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    int r = groups[gi].back();
    haz.clear();
    g.loc[r] = Loc{LOC_ARENA, arena.alloc(bytes[r], haz)};
  }
  std::vector<int> tiny_step(nlevels, -1);
  for (int lv = 0; lv < nlevels; ++lv) {
    Step st;
    st.kind = ST_TINY;
    if (sel_step >= 0) st.deps.push_back(sel_step);
    if (lv > 0) st.deps.push_back(tiny_step[lv - 1]);
    tiny_step[lv] = (int)g.steps.size();
    g.steps.push_back(st);
  }
  tmark("tiny descriptors");
  // tiny descriptors, ordered by level then group
  std::vector<int64_t> str_a(p.NI, 0), str_b(p.NI, 0);  // index -> stride (0: absent)
  std::vector<std::vector<int>> level_groups(nlevels);
  for (size_t gi = 0; gi < groups.size(); ++gi) level_groups[glevel[gi]].push_back((int)gi);
  std::vector<std::pair<int32_t, int32_t>> level_range(nlevels);
  for (int lv = 0; lv < nlevels; ++lv) {
    level_range[lv].first = (int32_t)g.tiny_groups.size();
    for (int gi : level_groups[lv]) {
      const auto& nodes = groups[gi];
      int r = nodes.back();
      TinyGroup tg;
      tg.beg = (int32_t)g.tiny_nodes.size();
      for (int v : nodes) {
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
        // digits: output indices in C's layout order, then the shared ones
        const auto& La = g.layout[a];
        const auto& Lb = g.layout[b];
        const auto& Lc = g.layout[v];
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
        tn.dig = (int32_t)g.tiny_digits.size();
        bool p2 = true;
        for (int i : Lc) {
          g.tiny_digits.push_back(TinyDigit{p.dom[i], (int32_t)str_a[i], (int32_t)str_b[i], 0});
          p2 &= (p.dom[i] == 2);
        }
        int64_t ssz = 1;
        int ns = 0;
        const auto& Ea = eff[a];
        const auto& Eb = eff[b];
        for (size_t x = 0, y = 0; x < Ea.size() && y < Eb.size();) {
          if (Ea[x] < Eb[y]) ++x;
          else if (Eb[y] < Ea[x]) ++y;
          else {
            const int i = Ea[x];
            g.tiny_digits.push_back(TinyDigit{p.dom[i], (int32_t)str_a[i], (int32_t)str_b[i], 0});
            p2 &= (p.dom[i] == 2);
            ssz *= p.dom[i];
            ++ns;
            ++x;
            ++y;
          }
        }
        for (int i : La) str_a[i] = 0;
        for (int i : Lb) str_b[i] = 0;
        tn.nc = (int32_t)Lc.size();
        tn.ns = ns;
        tn.c_size = (int32_t)size[v];
        tn.s_size = (int32_t)ssz;
        tn.pow2 = p2 ? 1 : 0;
        g.tiny_nodes.push_back(tn);
        g.tiny_ga.push_back(la);
        g.tiny_gb.push_back(lb);
        g.tiny_gout.push_back(lo);
        g.n_tiny++;
      }
      tg.end = (int32_t)g.tiny_nodes.size();
      g.tiny_groups.push_back(tg);
      g.tiny_smem_doubles = std::max(g.tiny_smem_doubles, group_smem[gi]);
      for (int v : nodes)
        if (v == r) producer[v] = tiny_step[lv];
    }
    level_range[lv].second = (int32_t)g.tiny_groups.size();
  }
  // forced roots consumed inside a tiny level: release with that level as reader
  for (size_t gi = 0; gi < groups.size(); ++gi)
    for (int v : groups[gi])
      for (int c : {p.kid_l(v), p.kid_r(v)})
        if (is_tiny(c) && group_of[c] != (int)gi) arena.release(g.loc[c].off, bytes[c], tiny_step[glevel[gi]]);
  // store level ranges in the TINY steps (reuse `work` / gdig_off fields)
  for (int lv = 0; lv < nlevels; ++lv) {
    g.steps[tiny_step[lv]].gdig_off = level_range[lv].first;
    g.steps[tiny_step[lv]].work = level_range[lv].second - level_range[lv].first;
  }

  tmark("big nodes in postord");
  // big nodes in postorder
  auto stride_map = [&](const std::vector<int>& L) {
    SmallMap<int64_t> m;
    int64_t st2 = 1;
    for (int i : L) {
      m[i] = st2;
      st2 *= p.dom[i];
    }
    return m;
  };
  std::vector<double> node_bytes(S, 0.0), node_flops(S, 0.0);
  for (int k = 0; k < p.NN; ++k) {
    int v = p.NL + k, a = p.left[k], b = p.right[k];
    // 2 * prod of the union's domains (eff sets are sorted, drop-free)
    u128 un = 1;
    {
      const auto& Ea = eff[a];
      const auto& Eb = eff[b];
      size_t x = 0, y = 0;
      while (x < Ea.size() || y < Eb.size()) {
        int i;
        if (y == Eb.size() || (x < Ea.size() && Ea[x] < Eb[y])) i = Ea[x++];
        else if (x == Ea.size() || Eb[y] < Ea[x]) i = Eb[y++];
        else i = Ea[x++], ++y;
        un *= (u128)p.dom[i];
        if (un > ((u128)1 << 100)) fail(TC_OVERFLOW, "contraction size overflows 2^100");
      }
    }
    const u128 fl = 2 * un;
    g.alg_flops += fl;
    g.alg_bytes += (u128)8 * (u128)(size[a] + size[b] + size[v]);
    node_bytes[v] = 8.0 * (double)(size[a] + size[b] + size[v]);
    node_flops[v] = (double)fl;
  }
  tmark("emit nodes");
  auto emit_node = [&](int v) {
    const int k = v - p.NL, a = p.left[k], b = p.right[k];
    Step st;
    st.slot = v;
    st.alg_bytes = node_bytes[v];
    st.alg_flops = node_flops[v];
    st.la = g.loc[a];
    st.lb = g.loc[b];
    for (int c : {a, b})
      if (producer[c] >= 0) st.deps.push_back(producer[c]);
    haz.clear();
    g.loc[v] = Loc{LOC_ARENA, arena.alloc(bytes[v], haz)};
    for (int h : haz) st.deps.push_back(h);
    st.lc = g.loc[v];
    const auto& La = g.layout[a];
    const auto& Lb = g.layout[b];
    const auto& Lc = g.layout[v];
    bool done = false;
    if (g.cls[v] == NC_STREAM) {
      try {
        bool b_small = eff[b].size() <= eff[a].size();
        int big = b_small ? a : b, sm = b_small ? b : a;
        const auto& Lg = g.layout[big];
        const auto& Lq = g.layout[sm];
        std::vector<int> Sh = inter(eff[a], eff[b]);
        std::vector<int> F = minus(eff[sm], Sh);
        SmallMap<int> pg, pc, pq;
        for (size_t q = 0; q < Lg.size(); ++q) pg[Lg[q]] = (int)q;
        for (size_t q = 0; q < Lc.size(); ++q) pc[Lc[q]] = (int)q;
        for (size_t q = 0; q < Lq.size(); ++q) pq[Lq[q]] = (int)q;
        // x bits: kept indices of big, in C address order
        std::vector<std::pair<int, int>> xa, xc;
        int j = 0;
        for (size_t q = 0; q < Lc.size(); ++q) {
          int i = Lc[q];
          if (has(F, i)) continue;
          xc.push_back({j, (int)q});
          j++;
        }
        // xa needs src ascending: same j order, dst = position in big
        j = 0;
        for (size_t q = 0; q < Lc.size(); ++q) {
          int i = Lc[q];
          if (has(F, i)) continue;
          xa.push_back({j, pg[i]});
          j++;
        }
        StreamParams sp{};
        sp.xa = make_runs(xa);
        sp.xc = make_runs(xc);
        sp.nx = (int64_t)1 << j;
        int ns = (int)Sh.size(), nf = (int)F.size();
        // order F by C position, S by big-operand position
        std::sort(F.begin(), F.end(), [&](int x, int y) { return pc[x] < pc[y]; });
        std::sort(Sh.begin(), Sh.end(), [&](int x, int y) { return pg[x] < pg[y]; });
        for (int s = 0; s < (1 << ns); ++s) {
          int64_t o = 0, oq = 0;
          for (int t = 0; t < ns; ++t)
            if (s >> t & 1) {
              o += (int64_t)1 << pg[Sh[t]];
              oq += (int64_t)1 << pq[Sh[t]];
            }
          sp.offA[s] = o;
          for (int f = 0; f < (1 << nf); ++f) {
            int64_t of = 0;
            for (int t = 0; t < nf; ++t)
              if (f >> t & 1) of += (int64_t)1 << pq[F[t]];
            sp.offP[s * (1 << nf) + f] = (int32_t)(oq + of);
          }
        }
        for (int f = 0; f < (1 << nf); ++f) {
          int64_t o = 0;
          for (int t = 0; t < nf; ++t)
            if (f >> t & 1) o += (int64_t)1 << pc[F[t]];
          sp.offC[f] = o;
        }
        st.kind = ST_STREAM;
        st.sp = sp;
        st.ns = ns;
        st.nf = nf;
        st.la = g.loc[big];
        st.lb = g.loc[sm];
        st.work = sp.nx;
        g.n_stream++;
        done = true;
      } catch (const Error& e) {
        if (e.status != -1) throw;
      }
    } else if (g.cls[v] == NC_GEMM) {
      try {
        std::vector<int> K = inter(eff[a], eff[b]);
        std::vector<int> M = minus(eff[a], K), N = minus(eff[b], K);
        SmallMap<int> pa, pb, pc;
        for (size_t q = 0; q < La.size(); ++q) pa[La[q]] = (int)q;
        for (size_t q = 0; q < Lb.size(); ++q) pb[Lb[q]] = (int)q;
        for (size_t q = 0; q < Lc.size(); ++q) pc[Lc[q]] = (int)q;
        std::sort(M.begin(), M.end(), [&](int x, int y) { return pc[x] < pc[y]; });
        std::sort(N.begin(), N.end(), [&](int x, int y) { return pc[x] < pc[y]; });
        std::sort(K.begin(), K.end(), [&](int x, int y) { return pa[x] < pa[y]; });
        const int m = (int)M.size(), n = (int)N.size(), kk = (int)K.size();
        // 128x64 CTA tiles (8 warps) for large GEMMs, 64x64 and below otherwise
        static const int big_tiles = std::getenv("TC_GEMM_BIG") ? std::atoi(std::getenv("TC_GEMM_BIG")) : 1;
        static const int big_k = std::getenv("TC_GEMM_BIG_K") ? std::atoi(std::getenv("TC_GEMM_BIG_K")) : 4;
        const bool big = big_tiles && m >= 7 && n >= 6 && kk >= big_k;
        const int MT = big ? 7 : std::max(3, std::min(6, m)), NT = std::max(3, std::min(6, n)), KT = 4;
        GemmParams gp{};
        gp.m_hi = std::max(0, m - MT);
        gp.n_hi = std::max(0, n - NT);
        gp.k_tiles = (int64_t)1 << std::max(0, kk - KT);
        std::vector<std::pair<int, int>> r;
        r.clear();
        for (int t = MT; t < (int)M.size(); ++t) r.push_back({t - MT, pa[M[t]]});
        gp.a_m = make_runs(r);
        r.clear();
        for (int t = KT; t < (int)K.size(); ++t) r.push_back({t - KT, pa[K[t]]});
        gp.a_k = make_runs(r);
        r.clear();
        for (int t = NT; t < (int)N.size(); ++t) r.push_back({t - NT, pb[N[t]]});
        gp.b_n = make_runs(r);
        r.clear();
        for (int t = KT; t < (int)K.size(); ++t) r.push_back({t - KT, pb[K[t]]});
        gp.b_k = make_runs(r);
        r.clear();
        for (int t = MT; t < (int)M.size(); ++t) r.push_back({t - MT, pc[M[t]]});
        gp.c_m = make_runs(r);
        r.clear();
        for (int t = NT; t < (int)N.size(); ++t) r.push_back({t - NT, pc[N[t]]});
        gp.c_n = make_runs(r);
        auto tmap = [&](SmallMap<int>& P, const std::vector<int>& R1, int n1,
                        const std::vector<int>& R2, int n2) {
          // R1 tile bits -> kind 0, R2 tile bits -> kind 1; bits past the
          // shape are virtual (pos -1), placed after the real ones
          std::vector<std::tuple<int, int, int>> bits, virt;  // pos, kind, sub
          for (int t = 0; t < n1; ++t) {
            if (t < (int)R1.size()) bits.emplace_back(P[R1[t]], 0, t);
            else virt.emplace_back(-1, 0, t);
          }
          for (int t = 0; t < n2; ++t) {
            if (t < (int)R2.size()) bits.emplace_back(P[R2[t]], 1, t);
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
        gp.ta = tmap(pa, M, MT, K, KT);
        gp.tb = tmap(pb, N, NT, K, KT);
        gp.tc = tmap(pc, M, MT, N, NT);
        gp.grid_swizzle_log = std::min(gp.m_hi, 3);
        // split-K when the output tiles cannot fill the machine
        const int64_t tiles = (int64_t)1 << (gp.m_hi + gp.n_hi);
        int64_t splits = 1;
        if (tiles < 2 * kSMs && gp.k_tiles >= 8)
          splits = std::min<int64_t>(gp.k_tiles / 4, (2 * kSMs + tiles - 1) / tiles);
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
      } catch (const Error& e) {
        if (e.status != -1) throw;
      }
    }
    if (!done) {
      auto ma = stride_map(La), mb = stride_map(Lb);
      GenericParams np{};
      st.gdig_off = (int64_t)g.gdigits.size();
      for (int i : Lc) g.gdigits.push_back(GDigit{p.dom[i], ma.count(i) ? ma[i] : 0, mb.count(i) ? mb[i] : 0});
      std::vector<int> Sh = inter(eff[a], eff[b]);
      int64_t ssz = 1;
      for (int i : Sh) {
        g.gdigits.push_back(GDigit{p.dom[i], ma[i], mb[i]});
        ssz *= p.dom[i];
      }
      np.c_size = size[v];
      np.s_size = ssz;
      np.nc = (int32_t)Lc.size();
      np.ns = (int32_t)Sh.size();
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
      st.lws = Loc{LOC_ARENA, arena.alloc(ws_bytes, haz)};
      for (int h : haz) st.deps.push_back(h);
      g.steps.push_back(st);
      Step rd;
      rd.kind = ST_GEMM_REDUCE;
      rd.slot = v;
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
      arena.release(st.lws.off, ws_bytes, me + 1);
    } else {
      producer[v] = me;
      g.steps.push_back(st);
    }
    for (int c : {a, b})
      if (g.loc[c].kind == LOC_ARENA) arena.release(g.loc[c].off, bytes[c], me);
  };

  // one fused launch for a multi-step chain segment; false if the address
  // maps do not fit the kernel's run/tile limits (then: one launch per node)
  auto emit_chain = [&](const Seg& sg) -> bool {
    const int v1 = sg.nodes.front(), vk = sg.nodes.back();
    const int A = sg.big.front();
    const auto& La = g.layout[A];
    const auto& Lc = g.layout[vk];
    SmallMap<int> pa, pc;
    for (size_t q = 0; q < La.size(); ++q) pa[La[q]] = (int)q;
    for (size_t q = 0; q < Lc.size(); ++q) pc[Lc[q]] = (int)q;
    // inner bookkeeping
    std::vector<int> cur = sg.u0;  // inner bit j <-> index
    std::vector<ChainStep> cs;
    for (size_t i = 0; i < sg.nodes.size(); ++i) {
      const int u = sg.nodes[i], sm = sg.small[i], bg = sg.big[i];
      std::vector<int> Sh = inter(eff[bg], eff[sm]);
      std::vector<int> F = minus(eff[sm], Sh);
      const auto& Lq = g.layout[sm];
      SmallMap<int> pq;
      for (size_t q = 0; q < Lq.size(); ++q) pq[Lq[q]] = (int)q;
      std::vector<int> nw;
      for (int x : cur)
        if (!has(Sh, x)) nw.push_back(x);
      const int nkeep = (int)nw.size();
      for (int x : F) nw.push_back(x);
      if ((int)nw.size() > kChainU || (int)cur.size() > kChainU) return false;
      ChainStep c{};
      c.ns = (int)Sh.size();
      c.nf = (int)F.size();
      c.nnew = (int)nw.size();
      auto cpos = [&](int x) { return (int)(std::find(cur.begin(), cur.end(), x) - cur.begin()); };
      for (int s = 0; s < (1 << c.ns); ++s) {
        int sb = 0, oq = 0;
        for (int t = 0; t < c.ns; ++t)
          if (s >> t & 1) {
            sb |= 1 << cpos(Sh[t]);
            oq += 1 << pq[Sh[t]];
          }
        c.stab[s] = (uint8_t)sb;
        for (int f = 0; f < (1 << c.nf); ++f) {
          int of = 0;
          for (int t = 0; t < c.nf; ++t)
            if (f >> t & 1) of += 1 << pq[F[t]];
          c.offP[s * (1 << c.nf) + f] = oq + of;
        }
      }
      for (int un = 0; un < (1 << c.nnew); ++un) {
        int ub = 0, f = 0;
        for (int j = 0; j < c.nnew; ++j)
          if (un >> j & 1) {
            if (j < nkeep) ub |= 1 << cpos(nw[j]);
            else f |= 1 << (j - nkeep);
          }
        c.utab[un] = (uint16_t)(ub | (f << 8));
      }
      cs.push_back(c);
      cur = nw;
      (void)u;
    }
    const std::vector<int>& Uk = cur;
    std::vector<int> O = minus(eff[A], [&] {
      std::vector<int> s = sg.u0;
      std::sort(s.begin(), s.end());
      return s;
    }());
    std::sort(O.begin(), O.end(), [&](int x, int y) { return pa[x] < pa[y]; });
    int umax = (int)sg.u0.size();
    for (auto& c : cs) umax = std::max(umax, c.nnew);
    int lbuf = 0;
    while ((2 << lbuf) <= kChainBuf) ++lbuf;  // log2(kChainBuf)
    // x_lo bits: as wide as the smem tile allows, but leave >= ~2 tiles per SM
    const int xt = std::max(0, std::min({(int)O.size(), lbuf - umax, std::max(2, (int)O.size() - 9)}));
    if (lbuf - umax < 0) return false;
    ChainParams cp{};
    cp.nsteps = (int)cs.size();
    cp.xt = xt;
    cp.n_tiles = (int64_t)1 << ((int)O.size() - xt);
    std::vector<std::pair<int, int>> ra, rc;
    for (int j = xt; j < (int)O.size(); ++j) {
      ra.push_back({j - xt, pa[O[j]]});
      rc.push_back({j - xt, pc[O[j]]});
    }
    try {
      cp.a_hi = make_runs(ra);
      cp.c_hi = make_runs(rc);
    } catch (const Error& e) {
      if (e.status != -1) throw;
      return false;
    }
    auto tmap = [&](SmallMap<int>& P, const std::vector<int>& inner) {
      std::vector<std::tuple<int, int, int>> bits;
      for (int j = 0; j < xt; ++j) bits.emplace_back(P[O[j]], 0, j);
      for (size_t t = 0; t < inner.size(); ++t) bits.emplace_back(P[inner[t]], 1, (int)t);
      std::sort(bits.begin(), bits.end());
      TileMap tm{};
      tm.nbits = (int)bits.size();
      for (size_t q = 0; q < bits.size(); ++q) {
        tm.pos[q] = (int8_t)std::get<0>(bits[q]);
        tm.kind[q] = (int8_t)std::get<1>(bits[q]);
        tm.sub[q] = (int8_t)std::get<2>(bits[q]);
      }
      return tm;
    };
    cp.ta = tmap(pa, sg.u0);
    cp.tc = tmap(pc, Uk);
    Step st;
    st.kind = ST_CHAIN;
    st.slot = vk;
    st.cp = cp;
    st.la = g.loc[A];
    st.chain_off = (int64_t)g.chain_steps.size();
    for (size_t i = 0; i < cs.size(); ++i) {
      g.chain_steps.push_back(cs[i]);
      g.chain_piece.push_back(g.loc[sg.small[i]]);
    }
    st.work = cp.n_tiles;
    for (int u : sg.nodes) {
      st.alg_bytes += node_bytes[u];
      st.alg_flops += node_flops[u];
    }
    if (producer[A] >= 0) st.deps.push_back(producer[A]);
    for (int sm : sg.small)
      if (producer[sm] >= 0) st.deps.push_back(producer[sm]);
    haz.clear();
    g.loc[vk] = Loc{LOC_ARENA, arena.alloc(bytes[vk], haz)};
    for (int h : haz) st.deps.push_back(h);
    st.lc = g.loc[vk];
    const int me = (int)g.steps.size();
    g.steps.push_back(st);
    producer[vk] = me;
    if (g.loc[A].kind == LOC_ARENA) arena.release(g.loc[A].off, bytes[A], me);
    for (int sm : sg.small)
      if (g.loc[sm].kind == LOC_ARENA) arena.release(g.loc[sm].off, bytes[sm], me);
    g.n_stream += (int)sg.nodes.size();
    g.n_chain++;
    (void)v1;
    return true;
  };

  for (int k = 0; k < p.NN; ++k) {
    const int v = p.NL + k;
    if (g.cls[v] == NC_TINY) {
      int gi = group_of[v];
      int ts = tiny_step[glevel[gi]];
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
    if (g.cls[v] == NC_STREAM && seg_of[v] >= 0 && segs[seg_of[v]].nodes.size() > 1) {
      const Seg& sg = segs[seg_of[v]];
      if (v != sg.nodes.back()) continue;  // fused: no buffer, no launch
      if (emit_chain(sg)) continue;
      for (int u : sg.nodes) emit_node(u);
      continue;
    }
    emit_node(v);
  }

  tmark("root copy into the p");
  // root copy into the per-slice result slot, then advance the slice counter
  g.R = size[p.root];
  g.root_loc = g.loc[p.root];
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
  g.arena_bytes = std::max<int64_t>(arena.top, kAlign);
  for (auto& s : g.steps) {
    std::sort(s.deps.begin(), s.deps.end());
    s.deps.erase(std::unique(s.deps.begin(), s.deps.end()), s.deps.end());
  }
  return g;
}

}  // namespace tc
