// libtc runtime: the C-ABI of include/tc.h.
//
//  * tc_plan_*              symbolic plan (plan.cpp)
//  * tc_exec_create         compile (compile.cpp) -> bind device pointers ->
//                           one CUDA graph per device whose kernel nodes mirror
//                           the contraction DAG (independent branches run
//                           concurrently; arena reuse adds WAR edges)
//  * tc_exec_run            replay the graph once per slice; per-slice result
//                           slots stay in HBM
//  * tc_sliced_execute      Algorithm 3 end to end, multi-device with one
//                           NCCL all-reduce over the zero-padded per-slice
//                           vector (exact: one non-zero contributor per slot),
//                           then the lexicographic fold on device.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <exception>
#include <thread>
#include <vector>

#include "compile.hpp"
#include "kernels.cuh"
#include "plan.hpp"
#include "tc.h"

using namespace tc;

struct tc_plan {
  Plan p;
};

namespace {

thread_local std::string g_err;

int set_err(int st, const std::string& m) {
  g_err = m;
  return st;
}

#define CU(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      int st_ = (e_ == cudaErrorMemoryAllocation) ? TC_OOM : TC_CUDA;                     \
      throw Error{st_, std::string(#x) + ": " + cudaGetErrorString(e_)};                  \
    }                                                                                     \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return TC_OK;
  } catch (const Error& e) {
    return set_err(e.status, e.msg);
  } catch (const std::bad_alloc&) {
    return set_err(TC_OOM, "host out of memory");
  } catch (const std::exception& e) {
    return set_err(TC_BAD_ARG, e.what());
  }
}

std::string u128_str(u128 v) {
  if (v == 0) return "0";
  std::string s;
  while (v) {
    s.push_back(char('0' + (int)(v % 10)));
    v /= 10;
  }
  return std::string(s.rbegin(), s.rend());
}

// Process-wide caching device allocator: programs are built per call of the
// public API, so freed buffers go back to a per-device free list instead of
// cudaFree (a 1.6 GB cudaMalloc/cudaFree pair costs ~10-100 ms).  On OOM the
// cache of that device is released and the allocation retried once.
struct DevCache {
  std::mutex mu;
  std::vector<std::multimap<size_t, void*>> free_;
  static size_t round(size_t b) { return (std::max<size_t>(b, 256) + 511) & ~(size_t)511; }
  void* get(int dev, size_t bytes) {
    bytes = round(bytes);
    {
      std::lock_guard<std::mutex> lk(mu);
      if ((int)free_.size() > dev) {
        auto& f = free_[dev];
        auto it = f.lower_bound(bytes);
        if (it != f.end() && it->first <= 2 * bytes + ((size_t)1 << 20)) {
          void* p = it->second;
          f.erase(it);
          sizes_[p] = bytes;  // reported size: the request
          return p;
        }
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      release(dev);
      e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) {
      int st = (e == cudaErrorMemoryAllocation) ? TC_OOM : TC_CUDA;
      throw Error{st, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
    }
    std::lock_guard<std::mutex> lk(mu);
    real_[p] = bytes;
    sizes_[p] = bytes;
    return p;
  }
  void put(int dev, void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)free_.size() <= dev) free_.resize(dev + 1);
    free_[dev].emplace(real_[p], p);
  }
  void release(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    if ((int)free_.size() <= dev) return;
    for (auto& kv : free_[dev]) {
      cudaFree(kv.second);
      real_.erase(kv.second);
      sizes_.erase(kv.second);
    }
    free_[dev].clear();
  }
  std::map<void*, size_t> real_, sizes_;
};
DevCache& dcache() {
  static DevCache c;
  return c;
}

template <class T>
T* dalloc(size_t n, int64_t& total, int dev) {
  size_t b = std::max<size_t>(n * sizeof(T), 16);
  total += (int64_t)b;
  return (T*)dcache().get(dev, b);
}

using StreamFn = void (*)(StreamParams);
StreamFn stream_fn(int ns, int nf) {
#define SF(a, b) \
  if (ns == a && nf == b) return k_stream<a, b>;
  SF(0, 0) SF(0, 1) SF(0, 2) SF(0, 3) SF(0, 4) SF(0, 5)
  SF(1, 0) SF(1, 1) SF(1, 2) SF(1, 3) SF(1, 4) SF(1, 5)
  SF(2, 0) SF(2, 1) SF(2, 2) SF(2, 3) SF(2, 4) SF(2, 5)
  SF(3, 0) SF(3, 1) SF(3, 2) SF(3, 3) SF(3, 4)
  SF(4, 0) SF(4, 1) SF(4, 2) SF(4, 3)
#undef SF
  throw Error{TC_BAD_ARG, "no stream kernel for this shape"};
}

struct GemmVariant {
  void* fn;
  int threads;
  int smem;
};
template <int BM, int BN, int WGM, int WGN>
GemmVariant gv() {
  using Cfg = GemmCfg<BM, BN, WGM, WGN>;
  return GemmVariant{(void*)k_gemm<BM, BN, WGM, WGN>, Cfg::NT, Cfg::SMEM};
}
// tile bits (bm, bn) in [3, 6] -> kernel instantiation (warp grid chosen so
// every warp owns >= 8x8)
GemmVariant gemm_variant(int bm, int bn) {
  switch (bm * 8 + bn) {
    case 7 * 8 + 6: return gv<128, 64, 4, 2>();
    case 6 * 8 + 6: return gv<64, 64, 2, 2>();
    case 6 * 8 + 5: return gv<64, 32, 2, 2>();
    case 5 * 8 + 6: return gv<32, 64, 2, 2>();
    case 5 * 8 + 5: return gv<32, 32, 2, 2>();
    case 6 * 8 + 4: return gv<64, 16, 4, 1>();
    case 4 * 8 + 6: return gv<16, 64, 1, 4>();
    case 6 * 8 + 3: return gv<64, 8, 4, 1>();
    case 3 * 8 + 6: return gv<8, 64, 1, 4>();
    case 5 * 8 + 4: return gv<32, 16, 2, 2>();
    case 4 * 8 + 5: return gv<16, 32, 2, 2>();
    case 5 * 8 + 3: return gv<32, 8, 4, 1>();
    case 3 * 8 + 5: return gv<8, 32, 1, 4>();
    case 4 * 8 + 4: return gv<16, 16, 2, 2>();
    case 4 * 8 + 3: return gv<16, 8, 2, 1>();
    case 3 * 8 + 4: return gv<8, 16, 1, 2>();
    case 3 * 8 + 3: return gv<8, 8, 1, 1>();
  }
  throw Error{TC_BAD_ARG, "no GEMM variant for this tile"};
}

int sm_count(int dev) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

unsigned grid_for(int64_t work, int per_block, int dev, int max_per_sm = 8) {
  int64_t g = (work + per_block - 1) / per_block;
  int64_t cap = (int64_t)sm_count(dev) * max_per_sm;
  return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace

struct Launch {
  void* func = nullptr;
  dim3 grid, block;
  unsigned smem = 0;
  int kind = 0, slot = -1;
  bool inv = false;   // slice-invariant: in the prologue graph, once per pass
  bool blk = false;   // block tier: in the block graph, once per block of slices (compile.cpp)
  int cat() const { return inv ? 0 : blk ? 1 : 2; }
  double bytes = 0, flops = 0;
  int xbits = -1, ns = 0, nf = 0, ns2 = -1, nf2 = -1;  // stream shape (diagnostics)
  std::vector<char> blob;
  std::vector<size_t> off;
  std::vector<void*> ptrs;
  template <class T>
  void arg(const T& v) {
    size_t o = (blob.size() + 15) / 16 * 16;
    blob.resize(o + sizeof(T));
    std::memcpy(blob.data() + o, &v, sizeof(T));
    off.push_back(o);
  }
  cudaKernelNodeParams params() {
    ptrs.resize(off.size());
    for (size_t i = 0; i < off.size(); ++i) ptrs[i] = blob.data() + off[i];
    cudaKernelNodeParams kp{};
    kp.func = func;
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.sharedMemBytes = smem;
    kp.kernelParams = ptrs.data();
    return kp;
  }
};

struct tc_exec {
  std::vector<Launch> launches;
  int device = 0;
  cudaStream_t stream = nullptr;
  Program prog;
  int64_t dev_bytes = 0;
  char* arena = nullptr;
  double* leafbuf = nullptr;
  double* slicedbuf = nullptr;
  TinyNode* tnodes = nullptr;
  TinyDigit* tdigs = nullptr;
  TinyGroup* tgroups = nullptr;
  GDigit* gdig = nullptr;
  int64_t* rootmap = nullptr;
  double** results_slot = nullptr;  // device copy of `results` read by k_rootcopy
  std::vector<std::vector<int>> ldeps;  // per launch: launches it depends on
  SelEntry* sel = nullptr;
  SelTerm* selt = nullptr;
  int64_t* eta = nullptr;
  int64_t* ordbuf = nullptr;  // slice order table (compile.hpp, slice_lex); nullptr: lexicographic order
  double* results = nullptr;
  int64_t results_cap = 0;  // slices
  double* folded = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;      // per-slice graph
  cudaGraph_t graph_pro = nullptr;      // slice-invariant prologue (hoisted nodes), once per pass
  cudaGraphExec_t gexec_pro = nullptr;
  cudaGraph_t graph_blk = nullptr;      // block tier (+ the slice select), once per block of slices
  cudaGraphExec_t gexec_blk = nullptr;
  int64_t kernels_per_slice = 0;
  int64_t kernels_prologue = 0;
  int64_t kernels_block = 0;            // block-graph kernels (0: no block tier)
  int64_t last_B = 1;                   // slices per block of the last pass
  int64_t launches_per_pass(int64_t n) const {
    return kernels_prologue + kernels_per_slice * n + kernels_block * ((n + last_B - 1) / last_B);
  }
  // slices per block for a pass over [b, b + n): the program's block size when
  // the pass covers whole blocks, else 1 (the block graph runs before every slice)
  int64_t block_for(int64_t b, int64_t n) const {
    const int64_t B = prog.block_dim;
    return (kernels_block > 0 && B > 1 && b % B == 0 && n % B == 0) ? B : 1;
  }
  int64_t last_n = 0;
  double compile_ms = 0;

  // Slice lanes: slices are independent (Thm 5), so a pass
  // runs them on K concurrent streams, each lane with its own copy of the
  // per-slice arena, sliced-leaf buffer, tiny descriptors and slice counter
  // (the pinned hoisted tensors, leaves and result slots are shared).  The
  // small latency-bound launches of one slice then overlap those of others.
  // Lane 0 is the main stream and resources above.
  struct Lane {
    char* arena = nullptr;
    double* sliced = nullptr;
    TinyNode* tnodes = nullptr;
    int64_t* eta = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    std::vector<Launch> launches;
    std::vector<std::vector<int>> ldeps;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph_blk = nullptr;
    cudaGraphExec_t gexec_blk = nullptr;
  };
  std::vector<Lane> xl;  // lanes 1..K-1
  cudaEvent_t pro_done = nullptr;

  ~tc_exec() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& L : xl) {
      if (L.stream) cudaStreamSynchronize(L.stream);
      if (L.gexec) cudaGraphExecDestroy(L.gexec);
      if (L.graph) cudaGraphDestroy(L.graph);
      if (L.gexec_blk) cudaGraphExecDestroy(L.gexec_blk);
      if (L.graph_blk) cudaGraphDestroy(L.graph_blk);
      for (void* q : {(void*)L.arena, (void*)L.sliced, (void*)L.tnodes, (void*)L.eta}) dcache().put(device, q);
      if (L.done) cudaEventDestroy(L.done);
      if (L.stream) cudaStreamDestroy(L.stream);
    }
    if (pro_done) cudaEventDestroy(pro_done);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (gexec_pro) cudaGraphExecDestroy(gexec_pro);
    if (graph_pro) cudaGraphDestroy(graph_pro);
    if (gexec_blk) cudaGraphExecDestroy(gexec_blk);
    if (graph_blk) cudaGraphDestroy(graph_blk);
    if (stream) cudaStreamSynchronize(stream);
    for (void* q : {(void*)arena, (void*)leafbuf, (void*)slicedbuf, (void*)tnodes, (void*)tdigs,
                    (void*)tgroups, (void*)gdig, (void*)rootmap, (void*)results_slot, (void*)sel, (void*)selt, (void*)eta, (void*)ordbuf, (void*)results,
                    (void*)folded})
      dcache().put(device, q);
    if (stream) cudaStreamDestroy(stream);
  }

  // device address of a program location for lane k (hoisted pinned tensors
  // live in lane 0's arena prefix; per-slice buffers in the lane's copies)
  const double* ptr(const Loc& l, int k = 0) const {
    switch (l.kind) {
      case LOC_LEAF: return leafbuf + l.off;
      case LOC_SLICED: return (k ? xl[k - 1].sliced : slicedbuf) + l.off;
      case LOC_ARENA:  // a lane's copy holds the per-slice region (compile.cpp: [pinned | invariant | per-slice])
        return (const double*)(k && l.off >= prog.lane_base ? xl[k - 1].arena + (l.off - prog.lane_base)
                                                            : arena + l.off);
      default: return nullptr;
    }
  }

  std::vector<TinyNode> tiny_nodes_for(int k) const {
    const Program& g = prog;
    std::vector<TinyNode> tn = g.tiny_nodes;
    for (size_t i = 0; i < tn.size(); ++i) {
      tn[i].ga = ptr(g.tiny_ga[i], k);
      tn[i].gb = ptr(g.tiny_gb[i], k);
      tn[i].gout = (double*)ptr(g.tiny_gout[i], k);
    }
    return tn;
  }

  void build(const Plan& p, const std::vector<int>& chosen) {
    auto t0 = std::chrono::steady_clock::now();
    CU(cudaSetDevice(device));
    // Reuse-free arenas only on request (TC_ARENA_REUSE=0): the factored trees
    // are spines (C2: 2434 of 2918 launches on the critical path even without
    // write-after-read edges) and mapping a 45 GB arena costs ~200 ms per call.
    prog = compile_program(p, chosen, 0);
    auto t_prog = std::chrono::steady_clock::now();
    program_ms = std::chrono::duration<double, std::milli>(t_prog - t0).count();
    CU(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    Program& g = prog;
    arena = dalloc<char>((size_t)g.arena_bytes, dev_bytes, device);
    // raw leaf values, then the compressed (tied) leaves (compile.cpp)
    leafbuf = dalloc<double>(p.lval.size() + g.cvals.size(), dev_bytes, device);
    CU(cudaMemcpyAsync(leafbuf, p.lval.data(), p.lval.size() * 8, cudaMemcpyHostToDevice, stream));
    if (!g.cvals.empty())
      CU(cudaMemcpyAsync(leafbuf + p.lval.size(), g.cvals.data(), g.cvals.size() * 8, cudaMemcpyHostToDevice,
                         stream));
    if (!g.root_map.empty()) {
      rootmap = dalloc<int64_t>(g.root_map.size(), dev_bytes, device);
      CU(cudaMemcpyAsync(rootmap, g.root_map.data(), g.root_map.size() * 8, cudaMemcpyHostToDevice, stream));
    }
    if (g.sliced_doubles) slicedbuf = dalloc<double>((size_t)g.sliced_doubles, dev_bytes, device);
    if (!g.sel_ent.empty()) {
      sel = dalloc<SelEntry>(g.sel_ent.size(), dev_bytes, device);
      selt = dalloc<SelTerm>(std::max<size_t>(1, g.sel_terms.size()), dev_bytes, device);
      CU(cudaMemcpyAsync(sel, g.sel_ent.data(), g.sel_ent.size() * sizeof(SelEntry), cudaMemcpyHostToDevice, stream));
      if (!g.sel_terms.empty())
        CU(cudaMemcpyAsync(selt, g.sel_terms.data(), g.sel_terms.size() * sizeof(SelTerm), cudaMemcpyHostToDevice,
                           stream));
    }
    if (!g.tiny_nodes.empty()) {
      std::vector<TinyNode> tn = tiny_nodes_for(0);
      tnodes = dalloc<TinyNode>(tn.size(), dev_bytes, device);
      tdigs = dalloc<TinyDigit>(std::max<size_t>(1, g.tiny_digits.size()), dev_bytes, device);
      tgroups = dalloc<TinyGroup>(g.tiny_groups.size(), dev_bytes, device);
      CU(cudaMemcpyAsync(tnodes, tn.data(), tn.size() * sizeof(TinyNode), cudaMemcpyHostToDevice, stream));
      if (!g.tiny_digits.empty())
        CU(cudaMemcpyAsync(tdigs, g.tiny_digits.data(), g.tiny_digits.size() * sizeof(TinyDigit),
                           cudaMemcpyHostToDevice, stream));
      CU(cudaMemcpyAsync(tgroups, g.tiny_groups.data(), g.tiny_groups.size() * sizeof(TinyGroup),
                         cudaMemcpyHostToDevice, stream));
    }
    if (!g.gdigits.empty()) {
      gdig = dalloc<GDigit>(g.gdigits.size(), dev_bytes, device);
      CU(cudaMemcpyAsync(gdig, g.gdigits.data(), g.gdigits.size() * sizeof(GDigit), cudaMemcpyHostToDevice, stream));
    }
    eta = dalloc<int64_t>(6, dev_bytes, device);
    if (g.permuted) {
      std::vector<int64_t> ord{(int64_t)g.ord_dim.size()};
      for (size_t j = 0; j < g.ord_dim.size(); ++j) {
        ord.push_back(g.ord_pv_iter[j]);
        ord.push_back(g.ord_dim[j]);
        ord.push_back(g.ord_pv_lex[j]);
      }
      ord_host = ord;
      ordbuf = dalloc<int64_t>(ord.size(), dev_bytes, device);
      CU(cudaMemcpyAsync(ordbuf, ord.data(), ord.size() * 8, cudaMemcpyHostToDevice, stream));
    }
    results_slot = dalloc<double*>(1, dev_bytes, device);
    folded = dalloc<double>((size_t)g.R, dev_bytes, device);
    CU(cudaStreamSynchronize(stream));

    const int tiny_smem = (int)(g.tiny_smem_doubles + kTinyThreads + g.tiny_stage_doubles) * 8 +
                          kTinyBatch * (int)sizeof(TinyNode) + g.tiny_dig_max * (int)sizeof(TinyDigit);
    CU(cudaFuncSetAttribute(k_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, tiny_smem));
    for (int bm = 3; bm <= 7; ++bm)
      for (int bn = 3; bn <= 6; ++bn) {
        if (bm == 7 && bn != 6) continue;
        GemmVariant v = gemm_variant(bm, bn);
        CU(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem));
      }

    make_launches(0, launches, ldeps, rootcopy_launch);
    auto t_end = std::chrono::steady_clock::now();
    setup_ms = std::chrono::duration<double, std::milli>(t_end - t_prog).count();
    compile_ms = std::chrono::duration<double, std::milli>(t_end - t0).count();
    count_launches();
  }

  // launch records of lane k (one per step, then chain-link fusion)
  void make_launches(int k, std::vector<Launch>& launches, std::vector<std::vector<int>>& ldeps, int& rootcopy_launch) {
    Program& g = prog;
    double* slicedbuf = k ? xl[k - 1].sliced : this->slicedbuf;
    TinyNode* tnodes = k ? xl[k - 1].tnodes : this->tnodes;
    int64_t* eta = k ? xl[k - 1].eta : this->eta;
    const int tiny_smem = (int)(g.tiny_smem_doubles + kTinyThreads + g.tiny_stage_doubles) * 8 +
                          kTinyBatch * (int)sizeof(TinyNode) + g.tiny_dig_max * (int)sizeof(TinyDigit);
    auto ptr = [&](const Loc& l) { return this->ptr(l, k); };
    launches.clear();
    launches.reserve(g.steps.size());
    for (size_t si = 0; si < g.steps.size(); ++si) {
      Step& st = g.steps[si];
      Launch L;
      L.kind = st.kind;
      L.inv = st.inv;
      L.blk = st.blk;
      L.slot = st.slot;
      L.bytes = st.alg_bytes;
      L.flops = st.alg_flops;
      L.block = dim3(256);
      switch (st.kind) {
        case ST_SELECT: {
          SelectParams slp{leafbuf, slicedbuf, sel, selt, (int64_t)g.sel_ent.size(), eta};
          L.func = (void*)k_select;
          L.grid = dim3(grid_for(slp.n, 256, device));
          L.arg(slp);
          break;
        }
        case ST_TINY: {
          L.func = (void*)k_tiny;
          L.grid = dim3((unsigned)st.work);
          L.block = dim3(kTinyThreads);
          L.smem = tiny_smem;
          L.arg((const TinyNode*)tnodes);
          L.arg((const TinyDigit*)tdigs);
          L.arg((const TinyGroup*)(tgroups + st.gdig_off));
          L.arg((int32_t)g.tiny_smem_doubles);
          L.arg((int32_t)g.tiny_stage_doubles);
          break;
        }
        case ST_STREAM: {
          StreamParams sp = st.sp;
          sp.A = ptr(st.la);
          sp.P = ptr(st.lb);
          sp.C = (double*)ptr(st.lc);
          L.func = (void*)stream_fn(st.ns, st.nf);
          L.block = dim3(kStreamThreads);
          // 2^g CTAs, each walking 2^kchunk chunks of 2^kStreamChunkBits x
          {
            const int xb = 63 - __builtin_clzll((unsigned long long)sp.nx);  // nx is a power of two
            const int chunks_log = std::max(0, xb - kStreamChunkBits);
            int g = 0;
            while (g < chunks_log && (2 << g) <= sm_count(device) * grid_mult(chunks_log)) ++g;
            L.grid = dim3(1u << g);
            if ((1 << chunks_log) < sm_count(device) * split_mult() && split_u_on()) {  // few chunks: a quarter chunk per CTA
              sp.split_u = 1;
              L.grid = dim3(xb >= kStreamChunkBits ? 4u << chunks_log : (unsigned)((sp.nx + 255) / 256));
            } else if (persist_from() > 0 && chunks_log >= persist_from()) {  // one wave, grid-stride chunks
              sp.persist = 1;
              L.grid = dim3((unsigned)std::min<int64_t>((int64_t)1 << chunks_log, wave_ctas(L.func, 0)));
            }
            L.xbits = xb, L.ns = st.ns, L.nf = st.nf;
          }
          L.arg(sp);
          break;
        }
        case ST_GEMM: {
          GemmParams gp = st.gp;
          gp.A = ptr(st.la);
          gp.B = ptr(st.lb);
          gp.C = (double*)ptr(st.lc);
          gp.ws = (double*)ptr(st.lws);
          GemmVariant v = gemm_variant(st.bm, st.bn);
          L.func = v.fn;
          L.block = dim3(v.threads);
          L.grid = dim3((unsigned)st.work, (unsigned)gp.splits);
          L.smem = v.smem;
          L.arg(gp);
          break;
        }
        case ST_GEMM_REDUCE: {
          GemmParams gp = st.gp;
          gp.A = ptr(st.la);
          gp.B = ptr(st.lb);
          gp.C = (double*)ptr(st.lc);
          gp.ws = (double*)ptr(st.lws);
          const int te = 1 << (st.bm + st.bn);
          L.func = (void*)k_splitk_reduce;
          L.grid = dim3(grid_for(st.work * te, 256, device));
          L.arg(gp);
          L.arg((int64_t)st.work);
          L.arg(te);
          break;
        }
        case ST_GENERIC: {
          GenericParams np = st.np;
          np.A = ptr(st.la);
          np.B = ptr(st.lb);
          np.C = (double*)ptr(st.lc);
          np.dig = gdig + st.gdig_off;
          L.func = (void*)k_generic;
          L.grid = dim3(grid_for(np.c_size, 256, device));
          L.arg(np);
          break;
        }
        case ST_ROOTCOPY: {
          RootCopyParams rp{ptr(g.root_loc), results_slot, rootmap, g.R, eta, ordbuf};
          L.func = (void*)k_rootcopy;
          L.grid = dim3(grid_for(g.R, 256, device));
          L.arg(rp);
          rootcopy_launch = (int)si;
          break;
        }
        case ST_ETA: {
          L.func = (void*)k_eta;
          L.grid = dim3(1);
          L.block = dim3(1);
          L.arg(eta);
          L.arg((const int64_t*)ordbuf);
          break;
        }
      }
      launches.push_back(std::move(L));
    }
    fuse_stream_pairs(launches, ldeps, rootcopy_launch);
  }

  void count_launches() {
    kernels_prologue = kernels_per_slice = kernels_block = 0;
    for (auto& L : launches) ++(L.inv ? kernels_prologue : L.blk ? kernels_block : kernels_per_slice);
    if (kernels_block)  // the block graph also runs the slice select
      for (auto& L : launches) kernels_block += L.kind == ST_SELECT;
  }

  // Chain links: a stream step whose big operand is the previous stream step's
  // output runs with it as ONE k_stream_pair launch (the intermediate stays in
  // registers; TC_FUSE=0 disables).  Pairs are formed greedily along the step
  // order.  ldeps[i] = launches launch i depends on.
  using PairFn = void (*)(StreamPairParams);
  static PairFn pair_fn(int ni, int ns1, int nf1, int ns2, int nf2) {
#define PF(a, b, c, d, e) \
  if (ni == a && ns1 == b && nf1 == c && ns2 == d && nf2 == e) return k_stream_pair<a, b, c, d, e>;
    PF(2, 1, 1, 1, 1) PF(1, 1, 1, 0, 1) PF(2, 0, 1, 1, 1) PF(2, 2, 1, 1, 1) PF(3, 1, 1, 2, 1)
    PF(1, 0, 1, 0, 1) PF(2, 0, 2, 0, 2) PF(3, 2, 1, 2, 1) PF(1, 2, 1, 0, 1) PF(2, 1, 1, 1, 2)
    PF(3, 1, 2, 1, 1) PF(2, 0, 2, 0, 1) PF(2, 0, 1, 2, 1) PF(1, 1, 1, 1, 1) PF(1, 0, 1, 1, 1)
    // links with a batch-scaling step (weighted carrier pieces: no summed, no new variable)
    PF(1, 1, 1, 0, 0) PF(1, 0, 1, 0, 0) PF(0, 1, 0, 0, 0) PF(1, 2, 1, 0, 0) PF(0, 2, 0, 0, 0)
    PF(1, 0, 0, 1, 1) PF(1, 0, 0, 1, 0) PF(0, 0, 0, 0, 1) PF(2, 0, 0, 2, 1)
    // the next most frequent links of C2 / C4 / C5 (tools/fuse_stats.py)
    PF(1, 1, 0, 1, 1) PF(2, 1, 1, 1, 0) PF(1, 1, 0, 1, 0) PF(2, 0, 1, 1, 0) PF(3, 1, 2, 1, 2)
    PF(3, 0, 2, 1, 0) PF(3, 1, 2, 1, 0) PF(1, 1, 1, 0, 2) PF(1, 1, 0, 1, 2) PF(1, 2, 0, 1, 1)
    PF(3, 0, 1, 2, 1) PF(1, 0, 1, 0, 2) PF(0, 1, 0, 0, 1)
#undef PF
    return nullptr;
  }

  // Derive the pair parameters from the two bound steps; false if the link
  // does not fit the kernel family (then the steps launch separately).
  static bool make_pair(const StreamParams& a, int ns1, int nf1, const StreamParams& b, int ns2, int nf2,
                        StreamPairParams& o, int& ni) {
    if (ns1 > 2 || nf1 > 2 || ns2 > 2 || nf2 > 2) return false;  // the instantiated family
    if (b.A != a.C || b.xa2.n != 0) return false;
    auto bits_of = [](const BitRuns& r) {
      int n = 0;
      for (int j = 0; j < r.n; ++j) n += r.len[j];
      return n;
    };
    const int x1 = bits_of(a.xc), x2 = bits_of(b.xa);
    if (((int64_t)1 << x1) != a.nx || ((int64_t)1 << x2) != b.nx || x1 > kStreamXBits || x2 > kStreamXBits) return false;
    auto lg = [](int64_t v) { return (v > 0 && (v & (v - 1)) == 0) ? 63 - __builtin_clzll((unsigned long long)v) : -1; };
    // owners of C1 address bits: step 1 (x1 bit j -> 0..x1-1, or F1 index -> 100+t)
    int own1[64], own2[64];
    for (int c = 0; c < 64; ++c) own1[c] = own2[c] = -1;
    for (int j = 0; j < x1; ++j) {
      const int c = lg(a.bitC[j]);
      if (c < 0) return false;
      own1[c] = j;
    }
    for (int t = 0; t < nf1; ++t) {
      const int c = lg(a.offC[1 << t]);
      if (c < 0 || own1[c] >= 0) return false;
      own1[c] = 100 + t;
    }
    for (int j = 0; j < x2; ++j) {
      const int c = lg(b.bitA[j]);
      if (c < 0 || own2[c] >= 0) return false;
      own2[c] = j;
    }
    int s2bit[4];
    for (int t = 0; t < ns2; ++t) {
      const int c = lg(b.offA[1 << t]);
      if (c < 0 || own2[c] >= 0) return false;
      own2[c] = 100 + t;
      s2bit[t] = c;
    }
    const int c1bits = x1 + nf1;
    for (int c = 0; c < c1bits; ++c)
      if (own1[c] < 0 || own2[c] < 0) return false;
    // inner bits: S2 (step-2 order), then the F1 bits step 2 keeps (rest)
    int inner[8], nin = 0;
    for (int t = 0; t < ns2; ++t) inner[nin++] = s2bit[t];
    for (int c = 0; c < c1bits; ++c)
      if (own1[c] >= 100 && own2[c] < 100) {
        if (nin == 8) return false;
        inner[nin++] = c;
      }
    ni = nin;
    if (ni > 3) return false;
    o = StreamPairParams{};
    o.A = a.A;
    o.P1 = a.P;
    o.P2 = b.P;
    o.C = b.C;
    o.nq = 1 << ni;
    o.nrest = 1 << (ni - ns2);
    for (int q = 0; q < o.nq; ++q) {
      int64_t qa = 0, qp1 = 0, qp2 = 0, qc = 0;
      int f1 = 0;
      for (int t = 0; t < ni; ++t) {
        if (!((q >> t) & 1)) continue;
        const int c = inner[t];
        if (own1[c] < 100) qa += a.bitA[own1[c]], qp1 += a.bitPo[own1[c]];
        else f1 |= 1 << (own1[c] - 100);
        if (own2[c] < 100) qp2 += b.bitPo[own2[c]], qc += b.bitC[own2[c]];
      }
      o.qA[q] = qa;
      o.qP1[q] = qp1;
      o.qF1[q] = f1;
      o.qP2[q] = qp2;
      o.qC[q] = qc;
      o.q_of[q] = q;  // q = s2 | rest << ns2  ->  q_of[s2 * nrest + rest]
    }
    for (int s2 = 0; s2 < (1 << ns2); ++s2)
      for (int r = 0; r < o.nrest; ++r) o.q_of[s2 * o.nrest + r] = s2 | (r << ns2);
    // y bits: the remaining C1 bits, ascending
    int yb = 0;
    for (int c = 0; c < c1bits; ++c) {
      bool in = false;
      for (int t = 0; t < ni; ++t) in |= inner[t] == c;
      if (in) continue;
      if (own1[c] >= 100 || own2[c] >= 100 || yb >= kStreamXBits) return false;
      o.bitA[yb] = a.bitA[own1[c]];
      o.bitP1[yb] = a.bitPo[own1[c]];
      o.bitC[yb] = b.bitC[own2[c]];
      o.bitP2[yb] = b.bitPo[own2[c]];
      ++yb;
    }
    o.ybits = yb;
    for (int s = 0; s < (1 << ns1); ++s) o.offA1[s] = a.offA[s];
    for (int q = 0; q < ((1 << ns1) << nf1); ++q) o.offP1[q] = a.offP[q];
    for (int q = 0; q < ((1 << ns2) << nf2); ++q) o.offP2[q] = b.offP[q];
    for (int f = 0; f < (1 << nf2); ++f) o.offC2[f] = b.offC[f];
    return true;
  }

  void fuse_stream_pairs(std::vector<Launch>& launches, std::vector<std::vector<int>>& ldeps, int& rootcopy_launch) {
    Program& g = prog;
    const size_t S = g.steps.size();
    static const bool on = !(std::getenv("TC_FUSE") && std::atoi(std::getenv("TC_FUSE")) == 0);
    std::vector<int> lid(S, -1);
    std::vector<Launch> out;
    std::vector<std::vector<int>> odeps;
    auto bound = [&](size_t k) {
      StreamParams sp;
      std::memcpy(&sp, launches[k].blob.data() + launches[k].off[0], sizeof(sp));
      return sp;
    };
    // candidate links (i, i+1), then the set of disjoint links that saves the
    // most intermediate traffic (a chain: O(S) dynamic program) -- a greedy
    // left-to-right pairing can take a small link and block a large one
    struct Cand {
      PairFn fn = nullptr;
      StreamPairParams pp;
      int ni = 0;
      double gain = 0;
    };
    std::vector<Cand> cand(S);
    static const bool dbg = std::getenv("TC_FUSE_DEBUG") != nullptr;
    for (size_t i = 0; i + 1 < S; ++i) {
      if (dbg && g.steps[i].kind == ST_STREAM && g.steps[i + 1].kind == ST_STREAM) {
        const Step &s1 = g.steps[i], &s2 = g.steps[i + 1];
        bool dep = false;
        for (int d : s2.deps) dep |= d == (int)i;
        StreamPairParams tmp;
        int tni = 0;
        const bool mk = make_pair(bound(i), s1.ns, s1.nf, bound(i + 1), s2.ns, s2.nf, tmp, tni);
        std::fprintf(stderr, "[fuse] %zu (%d,%d)->(%d,%d) dep=%d link=%d make=%d ni=%d fn=%d inv=%d\n", i, s1.ns, s1.nf,
                     s2.ns, s2.nf, (int)dep, (int)(bound(i + 1).A == bound(i).C), (int)mk, tni,
                     (int)(mk && pair_fn(tni, s1.ns, s1.nf, s2.ns, s2.nf) != nullptr), (int)s1.inv);
      }
      if (!(on && g.steps[i].kind == ST_STREAM && g.steps[i + 1].kind == ST_STREAM &&
            g.steps[i].inv == g.steps[i + 1].inv && g.steps[i].blk == g.steps[i + 1].blk))
        continue;
      const Step &s1 = g.steps[i], &s2 = g.steps[i + 1];
      bool dep_ok = false;  // step 2 must consume step 1 (its RAW edge)
      for (int d : s2.deps) dep_ok |= d == (int)i;
      // C2 may reuse the memory step 1 read (A, P1: released after step 1);
      // fused, those reads and the C2 writes overlap in time
      auto overlaps = [](const Loc& x, int64_t xb, const Loc& y, int64_t yb) {
        return x.kind == LOC_ARENA && y.kind == LOC_ARENA && x.off < y.off + yb && y.off < x.off + xb;
      };
      if (overlaps(s1.la, s1.la_bytes, s2.lc, s2.lc_bytes) || overlaps(s1.lb, s1.lb_bytes, s2.lc, s2.lc_bytes))
        dep_ok = false;
      Cand& c = cand[i];
      if (dep_ok && make_pair(bound(i), s1.ns, s1.nf, bound(i + 1), s2.ns, s2.nf, c.pp, c.ni))
        c.fn = pair_fn(c.ni, s1.ns, s1.nf, s2.ns, s2.nf);
      if (c.fn) c.gain = 2.0 * 8.0 * (double)bound(i).nx * (double)(1 << s1.nf);
    }
    std::vector<double> best(S + 2, 0.0);
    std::vector<char> take(S + 1, 0);
    for (size_t i = S; i-- > 0;) {
      best[i] = best[i + 1];
      if (cand[i].fn && cand[i].gain + best[i + 2] > best[i]) {
        best[i] = cand[i].gain + best[i + 2];
        take[i] = 1;
      }
    }
    for (size_t i = 0; i < S;) {
      PairFn fn = take[i] ? cand[i].fn : nullptr;
      StreamPairParams pp = cand[i].pp;
      int ni = cand[i].ni;
      (void)ni;
      if (fn) {
        const Step &s1 = g.steps[i], &s2 = g.steps[i + 1];
        Launch L;
        L.kind = ST_STREAM;
        L.inv = s1.inv;
        L.blk = s1.blk;
        L.slot = s2.slot;
        L.func = (void*)fn;
        L.block = dim3(kStreamThreads);
        const int chunks_log = std::max(0, pp.ybits - kStreamChunkBits);
        int gg = 0;
        while (gg < chunks_log && (2 << gg) <= sm_count(device) * grid_mult(chunks_log)) ++gg;
        L.grid = dim3(1u << gg);
        static const int pair_mult = std::getenv("TC_SPLIT_MULT_PAIR") ? std::max(1, std::atoi(std::getenv("TC_SPLIT_MULT_PAIR"))) : split_mult();
        if ((1 << chunks_log) < sm_count(device) * pair_mult && split_u_on()) {
          pp.split_u = 1;
          L.grid = dim3(pp.ybits >= kStreamChunkBits ? 4u << chunks_log : (unsigned)((((int64_t)1 << pp.ybits) + 255) / 256));
        } else if (persist_from() > 0 && chunks_log >= persist_from()) {
          pp.persist = 1;
        }
        L.xbits = pp.ybits, L.ns = s1.ns, L.nf = s1.nf, L.ns2 = s2.ns, L.nf2 = s2.nf;
        {
          static const bool pst_on = !(std::getenv("TC_PAIR_STAGE") && std::atoi(std::getenv("TC_PAIR_STAGE")) == 0);
          pp.p1n = (int32_t)(s1.lb_bytes / 8);
          pp.p2n = (int32_t)(s2.lb_bytes / 8);
          pp.pstage = pst_on && s1.lb_bytes > 0 && s2.lb_bytes > 0 && pp.p1n + pp.p2n <= kPairStageMax;
          L.smem = pp.pstage ? (unsigned)(pp.p1n + pp.p2n) * 8 : 0;
        }
        // executed bytes: A, P1, P2 and C2 (C1 never touches memory)
        const StreamParams sp1 = bound(i);
        const double c1_bytes = 8.0 * (double)sp1.nx * (double)(1 << s1.nf);
        if (pp.persist)
          L.grid = dim3((unsigned)std::min<int64_t>((int64_t)1 << chunks_log, wave_ctas(L.func, (int)L.smem)));
        L.bytes = s1.alg_bytes + s2.alg_bytes - 2 * c1_bytes;
        L.flops = s1.alg_flops + s2.alg_flops;
        L.arg(pp);
        std::vector<int> dd;
        for (size_t k : {i, i + 1})
          for (int d : g.steps[k].deps)
            if (d < (int)i) dd.push_back(lid[d]);
        std::sort(dd.begin(), dd.end());
        dd.erase(std::unique(dd.begin(), dd.end()), dd.end());
        lid[i] = lid[i + 1] = (int)out.size();
        out.push_back(std::move(L));
        odeps.push_back(dd);
        i += 2;
        continue;
      }
      std::vector<int> dd;
      for (int d : g.steps[i].deps) dd.push_back(lid[d]);
      std::sort(dd.begin(), dd.end());
      dd.erase(std::unique(dd.begin(), dd.end()), dd.end());
      lid[i] = (int)out.size();
      if ((int)i == rootcopy_launch) rootcopy_launch = (int)out.size();
      out.push_back(std::move(launches[i]));
      odeps.push_back(dd);
      ++i;
    }
    launches = std::move(out);
    ldeps = std::move(odeps);
  }

  void launch_one(Launch& L, bool pdl) {
    auto kp = L.params();
    if (pdl) {
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = L.grid;
      cfg.blockDim = L.block;
      cfg.dynamicSmemBytes = L.smem;
      cfg.stream = stream;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CU(cudaLaunchKernelExC(&cfg, L.func, kp.kernelParams));
    } else {
      CU(cudaLaunchKernel(L.func, L.grid, L.block, kp.kernelParams, L.smem, stream));
    }
  }

  // The CUDA graphs are built on the first run that replays the program more
  // than twice; one-shot calls launch the steps eagerly on the stream (with
  // PDL: each kernel's launch and prologue overlap its predecessor's tail).
  // Two graphs from the explicit launch DAG (data + WAR edges): the prologue
  // (slice-invariant launches, once per pass over the slices) and the
  // per-slice graph.  Edges between the two are implied by stream order.
  // launches of graph category `want` (0 prologue, 1 block, 2 per slice); the
  // block graph also holds the slice select (its nodes read sliced leaves)
  static bool in_cat(const Launch& L, int want) { return L.cat() == want || (want == 1 && L.kind == ST_SELECT); }
  static void instantiate(const std::vector<Launch>& L, const std::vector<std::vector<int>>& deps, int want,
                          cudaGraph_t& gr, cudaGraphExec_t& ge) {
    gr = nullptr;
    ge = nullptr;
    if (want == 1 && std::none_of(L.begin(), L.end(), [](const Launch& x) { return x.blk; })) return;
    std::vector<cudaGraphNode_t> nodes(L.size(), nullptr);
    for (size_t si = 0; si < L.size(); ++si) {
      if (!in_cat(L[si], want)) continue;
      if (!gr) CU(cudaGraphCreate(&gr, 0));
      std::vector<cudaGraphNode_t> dd;
      for (int d : deps[si])
        if (in_cat(L[d], want)) dd.push_back(nodes[d]);
      cudaKernelNodeParams kp = const_cast<Launch&>(L[si]).params();
      CU(cudaGraphAddKernelNode(&nodes[si], gr, dd.data(), dd.size(), &kp));
    }
    if (gr) CU(cudaGraphInstantiate(&ge, gr, 0));
  }

  bool pro_built = false;
  bool kernels_prologue_hint() const {
    for (const auto& L : launches)
      if (L.inv) return true;
    return false;
  }
  void ensure_graph(bool with_prologue = true) {
    if (gexec && (pro_built || !with_prologue)) return;
    auto t_graph0 = std::chrono::steady_clock::now();
    count_launches();
    // the two graphs are independent: build them on two host threads
    std::exception_ptr err;
    std::thread th;
    if (with_prologue && !pro_built)
      th = std::thread([&] {
        try {
          CU(cudaSetDevice(device));
          instantiate(launches, ldeps, 0, graph_pro, gexec_pro);
        } catch (...) {
          err = std::current_exception();
        }
      });
    if (!gexec) {
      instantiate(launches, ldeps, 2, graph, gexec);
      instantiate(launches, ldeps, 1, graph_blk, gexec_blk);
    }
    if (th.joinable()) th.join();
    if (err) std::rethrow_exception(err);
    pro_built = pro_built || with_prologue;
    graph_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_graph0).count();
  }

  // lanes 1..K-1 (graph mode only): per-lane buffers, launch records, graph
  void ensure_lanes(int K) {
    if ((int)xl.size() + 1 >= K) return;
    const Program& g = prog;
    if (!pro_done) CU(cudaEventCreateWithFlags(&pro_done, cudaEventDisableTiming));
    while ((int)xl.size() + 1 < K) {
      xl.emplace_back();
      const int k = (int)xl.size();
      Lane& L = xl.back();
      int64_t dummy = 0;
      L.arena = dalloc<char>((size_t)g.lane_arena_bytes, dev_bytes, device);
      if (g.sliced_doubles) L.sliced = dalloc<double>((size_t)g.sliced_doubles, dev_bytes, device);
      L.eta = dalloc<int64_t>(6, dummy, device);
      CU(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
      if (!g.tiny_nodes.empty()) {
        std::vector<TinyNode> tn = tiny_nodes_for(k);
        L.tnodes = dalloc<TinyNode>(tn.size(), dev_bytes, device);
        CU(cudaMemcpy(L.tnodes, tn.data(), tn.size() * sizeof(TinyNode), cudaMemcpyHostToDevice));
      }
    }
    // launch records + graph of every new lane on its own host thread
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(xl.size());
    for (size_t q = 0; q < xl.size(); ++q) {
      if (xl[q].gexec) continue;
      th.emplace_back([this, q, &err] {
        try {
          CU(cudaSetDevice(device));
          Lane& L = xl[q];
          int rc = -1;
          make_launches((int)q + 1, L.launches, L.ldeps, rc);
          instantiate(L.launches, L.ldeps, 2, L.graph, L.gexec);
          instantiate(L.launches, L.ldeps, 1, L.graph_blk, L.gexec_blk);
        } catch (...) {
          err[q] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }

  // lanes for a pass of n slices: TC_LANES (default 4), at most n, and only
  // while the per-lane copies fit a quarter of the free HBM
  int lanes_for(int64_t n) {
    static const int want = std::getenv("TC_LANES") ? std::max(1, std::atoi(std::getenv("TC_LANES"))) : 4;
    int K = (int)std::min<int64_t>(want, n);
    if (K <= (int)xl.size() + 1) return std::max(1, K);
    size_t fr = 0, tot = 0;
    CU(cudaMemGetInfo(&fr, &tot));
    const double per = (double)prog.lane_arena_bytes + 8.0 * prog.sliced_doubles + 1e6;
    while (K > (int)xl.size() + 1 && per * (K - 1 - (int)xl.size()) > 0.25 * (double)fr) --K;
    return std::max(1, K);
  }

  // slice counters: [current slice, first slice of the pass, stride, lane's
  // first offset, slices per block]: lane k runs blocks k, k + K, ... of B
  // consecutive slices (k_eta steps +1 inside a block, then to its next block)
  // A pass over lexicographic slices [b, b + n): mode 0 when the slice order
  // maps the range onto itself (iteration ids [b, b + n), blocks of B), else
  // mode 1 (lexicographic walk, B = 1; k_eta converts through the order table).
  void set_eta(int64_t b, int K, int64_t n) {
    const bool closed = !prog.permuted || (b % prog.closed_granule == 0 && (b + n) % prog.closed_granule == 0);
    const int64_t B = closed ? block_for(b, n) : 1;
    const int64_t mode = closed ? 0 : 1;
    const int64_t* ord = ord_host.empty() ? nullptr : ord_host.data();
    last_B = B;
    for (int k = 0; k < K; ++k) {
      const int64_t t0 = mode ? slice_iter(ord, b + k) : b + k * B;
      int64_t hk[6] = {t0, b, mode ? K : K * B, mode ? k : k * B, B, mode};
      CU(cudaMemcpyAsync(k ? xl[k - 1].eta : eta, hk, sizeof(hk), cudaMemcpyHostToDevice, stream));
    }
    CU(cudaStreamSynchronize(stream));
  }
  std::vector<int64_t> ord_host;
  void reset_eta(int K) {
    k_eta_reset<<<1, 1, 0, stream>>>(eta, ordbuf);
    for (int k = 1; k < K; ++k) k_eta_reset<<<1, 1, 0, stream>>>(xl[k - 1].eta, ordbuf);
  }
  double program_ms = 0, setup_ms = 0, graph_ms = 0, lanes_ms = 0;
  std::vector<float> start_ms;  // profile_graph: launch start offset within its graph launch

  int rootcopy_launch = -1;
  // stream grids: up to this many CTAs per SM, each walking >= 1 chunk.  Large
  // launches (>= 2^12 chunks, 32 MB per operand) want more CTAs in flight (32: C4
  // -7%, C1b -16%); the small ones of C2 lose ~2% with them (measured).
  static int grid_mult(int chunks_log) {
    static const int m = std::getenv("TC_STREAM_GRID_MULT") ? std::max(1, std::atoi(std::getenv("TC_STREAM_GRID_MULT"))) : 0;
    if (m) return m;
    static const int mid = std::getenv("TC_STREAM_GRID_MID") ? std::max(1, std::atoi(std::getenv("TC_STREAM_GRID_MID"))) : 4;
    return chunks_log >= 12 ? 32 : chunks_log >= 10 ? mid : 4;
  }
  // grid-stride ("persistent") stream launches from 2^k chunks up
  // (TC_STREAM_PERSIST=k, 0: off): one wave of resident CTAs, no partial wave
  static int persist_from() {
    static const int k = std::getenv("TC_STREAM_PERSIST") ? std::atoi(std::getenv("TC_STREAM_PERSIST")) : 12;
    return k;
  }
  // resident CTAs of a kernel on the whole GPU (occupancy x SMs), cached per function
  int64_t wave_ctas(void* fn, int smem) {
    static std::mutex mu;
    static std::map<std::pair<void*, int>, int> occ;
    int o = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = occ.find({fn, smem});
      if (it != occ.end()) o = it->second;
    }
    if (!o) {
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kStreamThreads, smem));
      o = std::max(1, o);
      std::lock_guard<std::mutex> lk(mu);
      occ[{fn, smem}] = o;
    }
    return (int64_t)o * sm_count(device);
  }
  static int split_mult() {
    static const int m = std::getenv("TC_SPLIT_MULT") ? std::max(1, std::atoi(std::getenv("TC_SPLIT_MULT"))) : 1;
    return m;
  }
  static bool split_u_on() {
    static const bool on = !(std::getenv("TC_SPLIT_U") && std::atoi(std::getenv("TC_SPLIT_U")) == 0);
    return on;
  }
  static bool use_pdl() {
    static const bool on = [] {
      const char* e = std::getenv("TC_PDL");
      return !(e && std::atoi(e) == 0);
    }();
    return on;
  }

  void ensure_results(int64_t n) {
    if (n <= results_cap) return;
    int64_t bytes = 0;
    if (__builtin_mul_overflow(n, prog.R, &bytes) || __builtin_mul_overflow(bytes, (int64_t)8, &bytes) ||
        bytes > ((int64_t)1 << 40))
      throw Error{TC_OOM, "per-slice results of " + std::to_string(n) + " slices exceed device memory"};
    if (results) dcache().put(device, results);
    results = nullptr;
    int64_t dummy = 0;
    results = dalloc<double>((size_t)(n * prog.R), dummy, device);
    results_cap = n;
    // k_rootcopy reads the buffer through results_slot: graphs stay valid
    CU(cudaMemcpyAsync(results_slot, &results, sizeof(double*), cudaMemcpyHostToDevice, stream));
    CU(cudaStreamSynchronize(stream));
  }

  // the prologue (0), a block's tier (1) or one slice (2) in step order on the stream (no graph)
  void launch_eager(int cat, bool first) {
    if (cat == 1 && !kernels_block) return;
    for (size_t i = 0; i < launches.size(); ++i) {
      if (!in_cat(launches[i], cat)) continue;
      launch_one(launches[i], use_pdl() && !first);
      first = false;
    }
  }
  // one pass over n slices: prologue once, then the per-slice launches
  // (round-robin over K lanes; lane 0 is the main stream)
  void launch_pass(int64_t n, bool eager, int K = 1, bool prologue_done = false) {
    const int64_t B = last_B;  // set_eta's block size for this pass
    if (eager) {
      launch_eager(0, true);
      for (int64_t s = 0; s < n; ++s) {
        const bool first = s == 0 && kernels_prologue == 0;
        if (s % B == 0) launch_eager(1, first);
        launch_eager(2, first && !kernels_block);
      }
      return;
    }
    if (gexec_pro && !prologue_done) CU(cudaGraphLaunch(gexec_pro, stream));
    if (K > 1) {
      CU(cudaEventRecord(pro_done, stream));
      for (int k = 1; k < K; ++k) CU(cudaStreamWaitEvent(xl[k - 1].stream, pro_done, 0));
    }
    for (int64_t s = 0; s < n; ++s) {
      const int k = (int)((s / B) % K);
      if (k == 0) {
        if (gexec_blk && s % B == 0) CU(cudaGraphLaunch(gexec_blk, stream));
        CU(cudaGraphLaunch(gexec, stream));
      } else {
        if (xl[k - 1].gexec_blk && s % B == 0) CU(cudaGraphLaunch(xl[k - 1].gexec_blk, xl[k - 1].stream));
        CU(cudaGraphLaunch(xl[k - 1].gexec, xl[k - 1].stream));
      }
    }
    for (int k = 1; k < K; ++k) {
      CU(cudaEventRecord(xl[k - 1].done, xl[k - 1].stream));
      CU(cudaStreamWaitEvent(stream, xl[k - 1].done, 0));
    }
  }

  // Eager replay of one slice, one kernel at a time, timed per launch with
  // CUDA events (diagnostics: per-node-class time shares).
  void profile(int64_t slice, std::vector<float>& ms) {
    CU(cudaSetDevice(device));
    ensure_results(1);
    long long* trace = nullptr;
    if (std::getenv("TC_TINY_TRACE") && prog.n_tiny > 0) {
      CU(cudaMalloc(&trace, (prog.n_tiny + 1) * sizeof(long long)));
      CU(cudaMemset(trace, 0, (prog.n_tiny + 1) * sizeof(long long)));
      CU(cudaMemcpyToSymbol(g_tiny_trace, &trace, sizeof(trace)));
    }
    set_eta(slice, 1, 1);
    std::vector<cudaEvent_t> ev(launches.size() + 1);
    for (auto& e : ev) CU(cudaEventCreate(&e));
    CU(cudaEventRecord(ev[0], stream));
    for (size_t i = 0; i < launches.size(); ++i) {
      launch_one(launches[i], false);
      CU(cudaEventRecord(ev[i + 1], stream));
    }
    CU(cudaEventSynchronize(ev.back()));
    CU(cudaGetLastError());
    ms.resize(launches.size());
    for (size_t i = 0; i < launches.size(); ++i) CU(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
    if (trace) {
      std::vector<long long> t(prog.n_tiny + 1);
      CU(cudaMemcpy(t.data(), trace, t.size() * sizeof(long long), cudaMemcpyDeviceToHost));
      long long* null = nullptr;
      CU(cudaMemcpyToSymbol(g_tiny_trace, &null, sizeof(null)));
      cudaFree(trace);
      for (int i = 0; i < prog.n_tiny; ++i) {
        if (!t[i] || !t[i + 1]) continue;
        const TinyNode& n = prog.tiny_nodes[i];
        std::fprintf(stderr, "[tiny] %d cyc=%lld c=%d s=%d nc=%d ns=%d lw=%d sync=%d g=%d%d%d st=%d%d pow2=%d\n", i,
                     t[i + 1] - t[i], n.c_size, n.s_size, n.nc, n.ns, n.lw, n.sync, prog.tiny_ga[i].kind != LOC_SMEM,
                     prog.tiny_gb[i].kind != LOC_SMEM, prog.tiny_gout[i].kind != LOC_SMEM, n.sta >= 0, n.stb >= 0, n.pow2);
      }
    }
    if (std::getenv("TC_PROFILE_DEBUG"))
      for (size_t i = 0; i < launches.size(); ++i) {
        const Launch& L = launches[i];
        std::fprintf(stderr, "[launch] %zu kind=%d grid=%u block=%u ms=%.4f MB=%.2f xbits=%d ns=%d nf=%d ns2=%d nf2=%d\n", i,
                     L.kind, L.grid.x * L.grid.y, L.block.x, ms[i], L.bytes / 1e6, L.xbits, L.ns, L.nf, L.ns2, L.nf2);
      }
    for (auto& e : ev) cudaEventDestroy(e);
    last_n = 1;
  }

  // Per-launch device time in graph mode: the prologue and per-slice graphs
  // rebuilt with an event-record node before and after every kernel node
  // (same DAG, same concurrency as the timed graphs), one pass over slices
  // [b, e) with a synchronize after each slice to read the events.  ms[i] =
  // launch i's time summed over the pass (prologue launches once).
  void profile_graph(int64_t b, int64_t e, std::vector<float>& ms, float& pass_ms) {
    CU(cudaSetDevice(device));
    const int64_t n = e - b;
    ensure_results(n);
    ms.assign(launches.size(), 0.f);
    pass_ms = 0.f;
    struct PG {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      std::vector<int> idx;
      std::vector<cudaEvent_t> e0, e1;
      ~PG() {
        if (ge) cudaGraphExecDestroy(ge);
        if (g) cudaGraphDestroy(g);
        for (auto x : e0) cudaEventDestroy(x);
        for (auto x : e1) cudaEventDestroy(x);
      }
    } pg[3];
    for (int pass = 0; pass < 3; ++pass) {  // prologue, block tier, per slice
      PG& G = pg[pass];
      if (pass == 1 && !kernels_block) continue;
      std::vector<cudaGraphNode_t> nodes(launches.size(), nullptr);
      for (size_t si = 0; si < launches.size(); ++si) {
        if (!in_cat(launches[si], pass)) continue;
        if (!G.g) CU(cudaGraphCreate(&G.g, 0));
        std::vector<cudaGraphNode_t> deps;
        for (int d : ldeps[si])
          if (in_cat(launches[d], pass)) deps.push_back(nodes[d]);
        cudaEvent_t a, z;
        CU(cudaEventCreate(&a));
        CU(cudaEventCreate(&z));
        G.e0.push_back(a);
        G.e1.push_back(z);
        G.idx.push_back((int)si);
        cudaGraphNode_t r0, r1;
        CU(cudaGraphAddEventRecordNode(&r0, G.g, deps.data(), deps.size(), a));
        cudaKernelNodeParams kp = launches[si].params();
        CU(cudaGraphAddKernelNode(&nodes[si], G.g, &r0, 1, &kp));
        CU(cudaGraphAddEventRecordNode(&r1, G.g, &nodes[si], 1, z));
      }
      if (G.g) CU(cudaGraphInstantiate(&G.ge, G.g, 0));
    }
    set_eta(b, 1, n);
    const int64_t B = last_B;
    cudaEvent_t p0, p1;
    CU(cudaEventCreate(&p0));
    CU(cudaEventCreate(&p1));
    start_ms.assign(launches.size(), 0.f);
    auto collect = [&](PG& G) {
      for (size_t q = 0; q < G.idx.size(); ++q) {
        float t = 0, t0 = 0;
        CU(cudaEventElapsedTime(&t, G.e0[q], G.e1[q]));
        CU(cudaEventElapsedTime(&t0, p0, G.e0[q]));
        ms[G.idx[q]] += t;
        start_ms[G.idx[q]] = t0;  // of the last graph launch that ran it
      }
    };
    std::vector<int> seq;  // graph launches of the pass: prologue, then per slice (block tier first)
    seq.push_back(0);
    for (int64_t s = 0; s < n; ++s) {
      if (s % B == 0) seq.push_back(1);
      seq.push_back(2);
    }
    for (int which : seq) {
      PG& G = pg[which];
      if (!G.ge) continue;
      CU(cudaEventRecord(p0, stream));
      CU(cudaGraphLaunch(G.ge, stream));
      CU(cudaEventRecord(p1, stream));
      CU(cudaStreamSynchronize(stream));
      CU(cudaGetLastError());
      float t = 0;
      CU(cudaEventElapsedTime(&t, p0, p1));
      pass_ms += t;
      collect(G);
    }
    cudaEventDestroy(p0);
    cudaEventDestroy(p1);
    last_n = n;
  }

  double run(int64_t b, int64_t e, int64_t repeats = 1) {
    CU(cudaSetDevice(device));
    int64_t n = e - b;
    if (n <= 0) {
      last_n = 0;
      return 0.0;
    }
    ensure_results(n);
    static const bool oneshot_graph = std::getenv("TC_ONESHOT_GRAPH") && std::atoi(std::getenv("TC_ONESHOT_GRAPH")) == 1;
    const bool eager = !gexec && n * repeats <= 2 && !oneshot_graph;
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    // The first graph-mode pass of a one-shot call launches the hoisted
    // prologue eagerly and builds the per-slice graphs and lanes on the host
    // while the device runs it (the prologue graph is built only when a
    // later pass needs it); later passes replay both graphs.
    static const bool overlap_on = !(std::getenv("TC_OVERLAP_BUILD") && std::atoi(std::getenv("TC_OVERLAP_BUILD")) == 0);
    const bool overlap = overlap_on && !eager && !gexec && repeats == 1 && kernels_prologue_hint();
    auto tg0 = std::chrono::steady_clock::now();
    if (overlap) {
      CU(cudaEventRecord(e0, stream));
      launch_eager(0, true);
    }
    if (!eager) ensure_graph(!overlap);
    auto tg1 = std::chrono::steady_clock::now();
    const int K = eager ? 1 : lanes_for(n);
    if (K > 1) ensure_lanes(K);
    lanes_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg1).count();
    if (std::getenv("TC_E2E_TIMING"))
      std::fprintf(stderr, "[run] graphs %.2f ms, lanes(%d) %.2f ms%s\n",
                   std::chrono::duration<double, std::milli>(tg1 - tg0).count(), K, lanes_ms,
                   overlap ? " (overlapping the eager prologue)" : "");
    set_eta(b, K, n);
    if (!overlap) CU(cudaEventRecord(e0, stream));
    for (int64_t r = 0; r < repeats; ++r) {
      if (r > 0) reset_eta(K);
      if (r > 0 && !pro_built) ensure_graph(true);
      launch_pass(n, eager, K, overlap && r == 0);
    }
    CU(cudaEventRecord(e1, stream));
    CU(cudaEventSynchronize(e1));
    CU(cudaGetLastError());
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    last_n = n;
    return ms;
  }

  // passes timed one by one, each after an untimed L2 flush
  double run_flushed(int64_t b, int64_t e, int64_t repeats, int64_t flush_bytes) {
    CU(cudaSetDevice(device));
    const int64_t n = e - b;
    if (n <= 0) {
      last_n = 0;
      return 0.0;
    }
    ensure_results(n);
    ensure_graph();
    const int64_t n4 = std::max<int64_t>(1, flush_bytes / 32);
    int64_t scratch = 0;  // not part of the program footprint
    double4* fbuf = dalloc<double4>((size_t)n4, scratch, device);
    std::vector<cudaEvent_t> ev(2 * repeats);
    for (auto& x : ev) CU(cudaEventCreate(&x));
    const int K = lanes_for(n);
    if (K > 1) ensure_lanes(K);
    set_eta(b, K, n);
    for (int64_t r = 0; r < repeats; ++r) {
      if (r > 0) reset_eta(K);
      k_flush<<<grid_for(n4, 256, device), 256, 0, stream>>>(fbuf, n4, (double)r);
      CU(cudaEventRecord(ev[2 * r], stream));
      launch_pass(n, false, K);
      CU(cudaEventRecord(ev[2 * r + 1], stream));
    }
    CU(cudaStreamSynchronize(stream));
    CU(cudaGetLastError());
    double total = 0;
    for (int64_t r = 0; r < repeats; ++r) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]));
      total += ms;
    }
    for (auto& x : ev) cudaEventDestroy(x);
    dcache().put(device, fbuf);
    last_n = n;
    return total;
  }

  void fold(double* out_host) {
    CU(cudaSetDevice(device));
    k_fold<<<grid_for(prog.R, 256, device), 256, 0, stream>>>(results, prog.R, last_n, folded);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_host, folded, prog.R * 8, cudaMemcpyDeviceToHost, stream));
    CU(cudaStreamSynchronize(stream));
  }
};

// ---------------------------------------------------------------------------
// NCCL (single process, one communicator per device), loaded on first use.
namespace {
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.CommInitAll = (decltype(n.CommInitAll))dlsym(n.h, "ncclCommInitAll");
    n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
    n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
  });
  if (!n.h || !n.CommInitAll || !n.AllReduce) throw Error{TC_NCCL, "libnccl.so.2 not loadable"};
  return n;
}
#define NC(x)                                                                          \
  do {                                                                                 \
    ncclResult_t r_ = (x);                                                             \
    if (r_ != 0) throw Error{TC_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)}; \
  } while (0)
constexpr int kNcclFloat64 = 8, kNcclSum = 0;
}  // namespace

// One communicator set per device list, created on first use and kept for the
// process (ncclCommInitAll costs ~100 ms-1 s; a counter calls sliced_execute
// once per formula).
const std::vector<ncclComm_t>& nccl_comms(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return it->second;
  std::vector<ncclComm_t> comms(devs.size());
  NC(nccl().CommInitAll(comms.data(), (int)devs.size(), devs.data()));
  return cache.emplace(devs, std::move(comms)).first->second;
}

namespace tc {
// the error channel of tc_last_error for the host-only parts (factor.cpp)
int set_last_error(int status, const std::string& msg) { return set_err(status, msg); }
}  // namespace tc

// ---------------------------------------------------------------------------
extern "C" {

const char* tc_last_error(void) { return g_err.c_str(); }

int tc_release_cache(int32_t device) {
  return guard([&] {
    int n = 0;
    CU(cudaGetDeviceCount(&n));
    for (int d = 0; d < n; ++d)
      if (device < 0 || d == device) {
        CU(cudaSetDevice(d));
        dcache().release(d);
      }
  });
}
int32_t tc_version(void) { return 1; }
int32_t tc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int tc_plan_create(const tc_plan_desc* desc, tc_plan** out) {
  return guard([&] {
    if (!desc || !out) throw Error{TC_BAD_ARG, "null argument"};
    auto h = std::make_unique<tc_plan>();
    h->p = build_plan(*desc);
    *out = h.release();
  });
}

void tc_plan_free(tc_plan* plan) { delete plan; }

int tc_plan_info_get(const tc_plan* plan, tc_plan_info* out) {
  return guard([&] {
    const Plan& p = plan->p;
    out->num_bonds = (int32_t)p.bonds_sorted.size();
    int nf = 0;
    for (int i = 0; i < p.NI; ++i) nf += (p.occ0[i] >= 0 && p.occ1[i] < 0);
    out->num_free = nf;
    out->max_rank = max_rank(p);
    out->root_rank = (int32_t)p.sets[p.root].size();
    out->contraction_ops = to_abi(contraction_ops(p));
    std::vector<char> none(p.NI, 0);
    out->mem_cost = to_abi(mem_cost(p, none));
  });
}

int tc_mem_cost(const tc_plan* plan, const int32_t* drop, int32_t n_drop, tc_u128* out) {
  return guard([&] { *out = to_abi(mem_cost(plan->p, mask_of(plan->p, drop, n_drop))); });
}

int tc_choose_slice_index(const tc_plan* plan, const int32_t* already, int32_t n_already, int32_t* out_index) {
  return guard([&] { *out_index = choose_slice_index(plan->p, mask_of(plan->p, already, n_already)); });
}

int tc_choose_slices(const tc_plan* plan, int64_t mem_budget, int32_t* chosen, int32_t cap, int32_t* n_chosen,
                     tc_u128* needs) {
  return guard([&] {
    const Plan& p = plan->p;
    std::vector<char> mask(p.NI, 0);
    int n = 0;
    auto over = [&](u128 c) { return mem_budget < 0 || c > (u128)mem_budget; };
    while (over(mem_cost(p, mask))) {
      int pick;
      try {
        pick = choose_slice_index(p, mask);
      } catch (const Error& e) {
        if (e.status != TC_NO_CANDIDATES) throw;
        std::vector<char> all(p.NI, 0);
        for (int i : p.bonds_sorted) all[i] = 1;
        u128 need = mem_cost(p, all);
        if (needs) *needs = to_abi(need);
        *n_chosen = n;
        throw Error{TC_BUDGET_INFEASIBLE, "cannot fit in " + std::to_string(mem_budget) +
                                              " bytes even fully sliced (needs " + u128_str(need) + ")"};
      }
      if (n >= cap) throw Error{TC_BAD_ARG, "chosen buffer too small"};
      chosen[n++] = pick;
      mask[pick] = 1;
    }
    *n_chosen = n;
  });
}

int tc_choose_slices_work(const tc_plan* plan, int32_t* chosen, int32_t n_already, int32_t cap, int64_t max_entries,
                          int32_t* n_chosen) {
  return guard([&] {
    std::vector<int> already(chosen, chosen + std::max(0, n_already));
    auto picks = choose_slices_work(plan->p, already, (u128)std::max<int64_t>(1, max_entries),
                                    std::max(0, cap - n_already), 6.5517e12, 35.5e12);
    int n = n_already;
    for (int c : picks) {
      if (n >= cap) throw Error{TC_BAD_ARG, "chosen buffer too small"};
      chosen[n++] = c;
    }
    *n_chosen = n;
  });
}

int tc_compile_stats(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced, tc_stats* s) {
  return guard([&] {
    std::vector<int> ch(sliced, sliced + std::max(0, n_sliced));
    auto t0 = std::chrono::steady_clock::now();
    Program g = compile_program(plan->p, ch, 0);
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *s = tc_stats{};
    s->mem_estimate = to_abi(g.mem_estimate);
    s->peak_observed = to_abi(g.peak_observed);
    s->num_slices = g.num_slices;
    s->device_peak_bytes = g.arena_bytes;
    s->gpu_launches = (int64_t)g.steps.size();
    s->n_tiny_nodes = g.n_tiny;
    s->n_stream_nodes = g.n_stream;
    s->n_gemm_nodes = g.n_gemm;
    s->n_generic_nodes = g.n_generic;
    s->alg_bytes = to_abi(g.alg_bytes);
    s->alg_flops = to_abi(g.alg_flops);
    s->n_alias_nodes = g.n_alias;
    s->n_tied_leaves = g.n_tied_leaves;
    s->phys_bytes = to_abi(g.phys_bytes);
    s->phys_flops = to_abi(g.phys_flops);
    s->phys_bytes_hoisted = to_abi(g.phys_bytes_inv);
    s->phys_flops_hoisted = to_abi(g.phys_flops_inv);
    for (auto& st : g.steps) ++(st.inv ? s->launches_prologue : st.blk ? s->launches_block : s->launches_per_slice);
    s->pinned_bytes = g.pinned_bytes;
    s->phys_bytes_block = to_abi(g.phys_bytes_blk);
    s->phys_flops_block = to_abi(g.phys_flops_blk);
    s->slices_per_block = g.block_dim;
    s->program_ms = ms;
  });
}

int tc_result_indices(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced, int32_t* out_idx, int32_t cap,
                      int32_t* rank) {
  return guard([&] {
    const Plan& p = plan->p;
    auto m = mask_of(p, sliced, n_sliced);
    int r = 0;
    for (int i : p.ref_order[p.root])
      if (!m[i]) {
        if (r >= cap) throw Error{TC_BAD_ARG, "index buffer too small"};
        out_idx[r++] = i;
      }
    *rank = r;
  });
}

int tc_exec_create(const tc_plan* plan, const int32_t* sliced, int32_t n_sliced, int32_t device, tc_exec** out) {
  return guard([&] {
    auto ex = std::make_unique<tc_exec>();
    ex->device = device;
    std::vector<int> ch(sliced, sliced + std::max(0, n_sliced));
    ex->build(plan->p, ch);
    *out = ex.release();
  });
}

void tc_exec_free(tc_exec* ex) { delete ex; }

int64_t tc_exec_result_size(const tc_exec* ex) { return ex->prog.R; }
int64_t tc_exec_slices_per_block(const tc_exec* ex) { return ex->last_B; }

static void fill_stats(const tc_exec& ex, double ms, tc_stats* s) {
  if (!s) return;
  const Program& g = ex.prog;
  s->mem_estimate = to_abi(g.mem_estimate);
  s->peak_observed = to_abi(g.peak_observed);
  s->num_slices = g.num_slices;
  s->device_peak_bytes = ex.dev_bytes;
  s->device_ms = ms;
  s->compile_ms = ex.compile_ms;
  s->gpu_launches = ex.launches_per_pass(ex.last_n);
  s->n_tiny_nodes = g.n_tiny;
  s->n_stream_nodes = g.n_stream;
  s->n_gemm_nodes = g.n_gemm;
  s->n_generic_nodes = g.n_generic;
  s->alg_bytes = to_abi(g.alg_bytes);
  s->alg_flops = to_abi(g.alg_flops);
  s->n_alias_nodes = g.n_alias;
  s->n_tied_leaves = g.n_tied_leaves;
  s->phys_bytes = to_abi(g.phys_bytes);
  s->phys_flops = to_abi(g.phys_flops);
  s->phys_bytes_hoisted = to_abi(g.phys_bytes_inv);
  s->phys_flops_hoisted = to_abi(g.phys_flops_inv);
  s->launches_prologue = ex.kernels_prologue;
  s->launches_per_slice = ex.kernels_per_slice;
  s->pinned_bytes = g.pinned_bytes;
  s->phys_bytes_block = to_abi(g.phys_bytes_blk);
  s->phys_flops_block = to_abi(g.phys_flops_blk);
  s->launches_block = ex.kernels_block;
  s->slices_per_block = ex.last_B;
  s->program_ms = ex.program_ms;
  s->setup_ms = ex.setup_ms;
  s->graph_ms = ex.graph_ms;
}

int tc_exec_run(tc_exec* ex, int64_t slice_begin, int64_t slice_end, tc_stats* stats) {
  return tc_exec_run_repeat(ex, slice_begin, slice_end, 1, stats);
}

int tc_exec_run_repeat(tc_exec* ex, int64_t slice_begin, int64_t slice_end, int64_t repeats, tc_stats* stats) {
  return guard([&] {
    if (slice_begin < 0 || slice_end > ex->prog.num_slices || slice_begin > slice_end || repeats < 1)
      throw Error{TC_BAD_ARG, "slice range out of bounds"};
    double ms = ex->run(slice_begin, slice_end, repeats);
    fill_stats(*ex, ms, stats);
    if (stats) stats->gpu_launches = (ex->launches_per_pass(ex->last_n) + 1) * repeats - 1;
  });
}

int tc_exec_run_flushed(tc_exec* ex, int64_t slice_begin, int64_t slice_end, int64_t repeats, int64_t flush_bytes,
                        tc_stats* stats) {
  return guard([&] {
    if (slice_begin < 0 || slice_end > ex->prog.num_slices || slice_begin > slice_end || repeats < 1)
      throw Error{TC_BAD_ARG, "slice range out of bounds"};
    double ms = ex->run_flushed(slice_begin, slice_end, repeats, flush_bytes);
    fill_stats(*ex, ms, stats);
    if (stats) stats->gpu_launches = ex->launches_per_pass(ex->last_n) * repeats;
  });
}

int tc_exec_copy_results(tc_exec* ex, double* dst_device) {
  return guard([&] {
    CU(cudaSetDevice(ex->device));
    if (ex->last_n > 0)
      CU(cudaMemcpyAsync(dst_device, ex->results, ex->last_n * ex->prog.R * 8, cudaMemcpyDeviceToDevice,
                         ex->stream));
    CU(cudaStreamSynchronize(ex->stream));
  });
}

int tc_fold_device(const double* per_slice_device, int64_t R, int64_t n, double* out_device, int32_t device) {
  return guard([&] {
    if (R < 1 || n < 1) throw Error{TC_BAD_ARG, "empty fold"};
    CU(cudaSetDevice(device));
    k_fold<<<grid_for(R, 256, device), 256>>>(per_slice_device, R, n, out_device);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
  });
}

int tc_exec_profile(tc_exec* ex, int64_t slice, float* step_ms, int32_t* step_kind, int32_t* step_slot,
                    double* step_bytes, double* step_flops, int32_t cap, int32_t* n) {
  return guard([&] {
    if (slice < 0 || slice >= ex->prog.num_slices) throw Error{TC_BAD_ARG, "slice out of range"};
    std::vector<float> ms;
    ex->profile(slice, ms);
    int k = (int)std::min<size_t>(ms.size(), (size_t)std::max(0, cap));
    for (int i = 0; i < k; ++i) {
      if (step_ms) step_ms[i] = ms[i];
      if (step_kind) step_kind[i] = ex->launches[i].kind;
      if (step_slot) step_slot[i] = ex->launches[i].slot;
      if (step_bytes) step_bytes[i] = ex->launches[i].bytes;
      if (step_flops) step_flops[i] = ex->launches[i].flops;
    }
    *n = (int32_t)ms.size();
  });
}

int tc_exec_profile_graph(tc_exec* ex, int64_t slice_begin, int64_t slice_end, float* launch_ms,
                          int32_t* launch_kind, int32_t* launch_inv, double* launch_bytes, double* launch_flops,
                          int32_t cap, int32_t* n, float* pass_ms) {
  return guard([&] {
    if (slice_begin < 0 || slice_end > ex->prog.num_slices || slice_begin >= slice_end)
      throw Error{TC_BAD_ARG, "slice range out of bounds"};
    std::vector<float> ms;
    float pm = 0;
    ex->profile_graph(slice_begin, slice_end, ms, pm);
    int k = (int)std::min<size_t>(ms.size(), (size_t)std::max(0, cap));
    for (int i = 0; i < k; ++i) {
      const Launch& L = ex->launches[i];
      if (launch_ms) launch_ms[i] = ms[i];
      if (launch_kind) launch_kind[i] = L.kind;
      if (launch_inv) launch_inv[i] = (L.inv ? 1 : 0) | (L.blk ? 2 : 0) | ((int32_t)std::lround(ex->start_ms[i] * 1000.0) << 2);
      if (launch_bytes) launch_bytes[i] = L.bytes;
      if (launch_flops) launch_flops[i] = L.flops;
    }
    *n = (int32_t)ms.size();
    if (pass_ms) *pass_ms = pm;
  });
}

int tc_exec_deps(const tc_exec* ex, int32_t* dep_off, int32_t* deps, int32_t cap, int32_t* n, int32_t* m) {
  return guard([&] {
    const auto& st = ex->ldeps;  // per launch (stream runs are one launch)
    int32_t e = 0;
    for (size_t i = 0; i < st.size(); ++i) {
      if (dep_off && (int32_t)i <= cap) dep_off[i] = e;
      for (int d : st[i]) {
        if (deps && e < cap) deps[e] = d;
        ++e;
      }
    }
    if (dep_off && (int32_t)st.size() <= cap) dep_off[st.size()] = e;
    *n = (int32_t)st.size();
    *m = e;
  });
}

int tc_exec_fetch(tc_exec* ex, double* per_slice, double* folded) {
  return guard([&] {
    CU(cudaSetDevice(ex->device));
    if (per_slice && ex->last_n > 0)
      CU(cudaMemcpy(per_slice, ex->results, ex->last_n * ex->prog.R * 8, cudaMemcpyDeviceToHost));
    if (folded) {
      if (ex->last_n <= 0) throw Error{TC_BAD_ARG, "no slices were run"};
      ex->fold(folded);
    }
  });
}

int tc_sliced_execute(const tc_plan* plan, int64_t mem_budget, const int32_t* slice_ids, int32_t n_slice_ids,
                      const int32_t* devices, int32_t n_devices, double* out_val, int64_t out_cap,
                      int32_t* out_idx, int32_t idx_cap, int32_t* out_rank, int32_t* chosen, int32_t chosen_cap,
                      int32_t* n_chosen, tc_stats* stats) {
  return guard([&] {
    const Plan& p = plan->p;
    std::vector<int> ch;
    if (n_slice_ids >= 0) {
      ch.assign(slice_ids, slice_ids + n_slice_ids);
    } else if (mem_budget != INT64_MIN) {  // INT64_MIN encodes mem_budget=None
      std::vector<int32_t> buf(p.bonds_sorted.size() + 1);
      int32_t nc = 0;
      tc_u128 need{};
      int st = tc_choose_slices(plan, mem_budget, buf.data(), (int32_t)buf.size(), &nc, &need);
      if (st != TC_OK) throw Error{st, g_err};
      ch.assign(buf.begin(), buf.begin() + nc);
    }
    if ((int)ch.size() > chosen_cap) throw Error{TC_BAD_ARG, "chosen buffer too small"};
    for (size_t j = 0; j < ch.size(); ++j) chosen[j] = ch[j];
    *n_chosen = (int32_t)ch.size();
    {
      auto m = mask_of(p, ch.data(), (int)ch.size());
      int r = 0;
      for (int i : p.ref_order[p.root])
        if (!m[i]) {
          if (r >= idx_cap) throw Error{TC_BAD_ARG, "index buffer too small"};
          out_idx[r++] = i;
        }
      *out_rank = r;
    }
    std::vector<int> devs;
    if (n_devices <= 0) devs.push_back(0);
    else devs.assign(devices, devices + n_devices);
    const int G = (int)devs.size();
    std::vector<std::unique_ptr<tc_exec>> ex(G);
    std::vector<Error> errs(G, Error{TC_OK, ""});
    std::vector<double> ms(G, 0.0);
    // compile once per device (threads), then block-partition the slice ids
    int64_t NS = 1, R = 1;
    for (int i : ch) {
      if (i < 0 || i >= p.NI) throw Error{TC_BAD_ARG, "slice index id out of range"};
      if (__builtin_mul_overflow(NS, (int64_t)p.dom[i], &NS)) throw Error{TC_OVERFLOW, "too many slices"};
    }
    {
      auto m = mask_of(p, ch.data(), (int)ch.size());
      for (int i : p.sets[p.root])
        if (!m[i]) R *= p.dom[i];
    }
    if (R > out_cap) throw Error{TC_BAD_ARG, "output buffer too small"};
    const int64_t per = (NS + G - 1) / G;
    auto work = [&](int gi) {
      try {
        ex[gi] = std::make_unique<tc_exec>();
        ex[gi]->device = devs[gi];
        auto t0 = std::chrono::steady_clock::now();
        ex[gi]->build(p, ch);
        auto t1 = std::chrono::steady_clock::now();
        int64_t b = std::min<int64_t>(NS, gi * per), e = std::min<int64_t>(NS, b + per);
        ms[gi] = ex[gi]->run(b, e);
        auto t2 = std::chrono::steady_clock::now();
        if (std::getenv("TC_E2E_TIMING"))
          std::fprintf(stderr, "[sliced_execute] dev %d: build %.2f ms (program %.2f setup %.2f) run %.2f ms (device %.2f)\n",
                       devs[gi], std::chrono::duration<double, std::milli>(t1 - t0).count(), ex[gi]->program_ms,
                       ex[gi]->setup_ms, std::chrono::duration<double, std::milli>(t2 - t1).count(), ms[gi]);
      } catch (const Error& e) {
        errs[gi] = e;
      }
    };
    if (G == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int gi = 0; gi < G; ++gi) th.emplace_back(work, gi);
      for (auto& t : th) t.join();
    }
    for (auto& e : errs)
      if (e.status != TC_OK) throw e;
    if (G == 1) {
      ex[0]->fold(out_val);
    } else {
      // zero-padded [NS][R] vector on every device, one all-reduce (exact: a
      // single non-zero contributor per position), fold on device 0.  The
      // same device listed twice (tests on one GPU) gathers by peer copies
      // instead: NCCL rejects duplicate devices in one communicator.
      int64_t nbytes = 0;
      if (__builtin_mul_overflow(NS, R, &nbytes) || __builtin_mul_overflow(nbytes, (int64_t)8, &nbytes) ||
          nbytes > ((int64_t)1 << 36))
        throw Error{TC_OOM, "per-slice result vector of " + std::to_string(NS) + " x " + std::to_string(R) +
                                " entries exceeds the all-reduce cap (64 GiB)"};
      struct Full {  // returned to the cache on every exit path
        std::vector<double*> p;
        std::vector<int> dev;
        ~Full() {
          for (size_t i = 0; i < p.size(); ++i)
            if (p[i]) dcache().put(dev[i], p[i]);
        }
      } full;
      full.p.assign(G, nullptr);
      full.dev = devs;
      std::vector<int> sorted = devs;
      std::sort(sorted.begin(), sorted.end());
      const bool distinct = std::unique(sorted.begin(), sorted.end()) == sorted.end();
      for (int gi = 0; gi < G; ++gi) {
        if (!distinct && gi > 0) break;
        CU(cudaSetDevice(devs[gi]));
        int64_t dummy = 0;
        full.p[gi] = dalloc<double>((size_t)(NS * R), dummy, devs[gi]);
        CU(cudaMemsetAsync(full.p[gi], 0, NS * R * 8, ex[gi]->stream));
      }
      tc_exec& e0 = *ex[0];
      if (distinct) {
        for (int gi = 0; gi < G; ++gi) {
          CU(cudaSetDevice(devs[gi]));
          int64_t b = std::min<int64_t>(NS, gi * per);
          if (ex[gi]->last_n > 0)
            CU(cudaMemcpyAsync(full.p[gi] + b * R, ex[gi]->results, ex[gi]->last_n * R * 8,
                               cudaMemcpyDeviceToDevice, ex[gi]->stream));
        }
        auto& nc = nccl();
        const std::vector<ncclComm_t>& comms = nccl_comms(devs);
        NC(nc.GroupStart());
        for (int gi = 0; gi < G; ++gi)
          NC(nc.AllReduce(full.p[gi], full.p[gi], NS * R, kNcclFloat64, kNcclSum, comms[gi], ex[gi]->stream));
        NC(nc.GroupEnd());
        for (int gi = 0; gi < G; ++gi) {
          CU(cudaSetDevice(devs[gi]));
          CU(cudaStreamSynchronize(ex[gi]->stream));
        }
      } else {
        CU(cudaSetDevice(e0.device));
        CU(cudaStreamSynchronize(e0.stream));
        for (int gi = 0; gi < G; ++gi) {
          int64_t b = std::min<int64_t>(NS, gi * per);
          if (ex[gi]->last_n > 0)
            CU(cudaMemcpyPeerAsync(full.p[0] + b * R, devs[0], ex[gi]->results, devs[gi], ex[gi]->last_n * R * 8,
                                   e0.stream));
        }
      }
      CU(cudaSetDevice(e0.device));
      k_fold<<<grid_for(R, 256, e0.device), 256, 0, e0.stream>>>(full.p[0], R, NS, e0.folded);
      CU(cudaGetLastError());
      CU(cudaMemcpyAsync(out_val, e0.folded, R * 8, cudaMemcpyDeviceToHost, e0.stream));
      CU(cudaStreamSynchronize(e0.stream));
    }
    if (stats) {
      fill_stats(*ex[0], *std::max_element(ms.begin(), ms.end()), stats);
      int64_t launches = 0;
      for (auto& e : ex) launches += e->launches_per_pass(e->last_n);
      stats->gpu_launches = launches;
      stats->num_slices = NS;
    }
  });
}

}  // extern "C"
