// sm_100a kernels of the execution stage.  Included once, by runtime.cu.
//
//   k_select   K5  per-slice leaf selection            (slicing.py:30-41, tensor.py:118-125)
//   k_tiny     K4  tiny-subtree forest, one CTA per subtree, smem-resident
//   k_stream   K2  big x <=64-entry operand, HBM streaming, permutation folded in
//                  (batch / diagonal-read variables of tied networks)
//   k_gemm     K3  FP64 DMMA (mma.sync m8n8k4 f64) GEMM, bit-permuted operands,
//                  optional batch variables
//   k_generic      mixed-radix pairwise contraction (domains != 2, odd shapes)
//   k_rootcopy / k_eta / k_fold   per-slice result slot, slice counter, and the
//                  lexicographic left fold of the slice sum (slicing.py:139-145)
//
// Every kernel is deterministic: each output entry is produced by exactly one
// thread with a fixed summation order (no floating-point atomics), so reruns
// and different device counts give bitwise-identical results.
#pragma once
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <cstdint>

#include "program.h"

namespace tc {

namespace cg = cooperative_groups;

// Programmatic dependent launch (PDL): a kernel lets its dependent launch as
// soon as it starts (launch_dependents) and waits for its own predecessor's
// completion and memory (wait) only after the parameter-only prologue.  Both
// are no-ops for launches without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
__global__ void k_select(const SelectParams p) {
  pdl_launch();
  pdl_wait();
  const int64_t eta = p.eta[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n;
       e += (int64_t)gridDim.x * blockDim.x) {
    SelEntry en = p.ent[e];
    int64_t src = en.src;
    for (int t = 0; t < en.nt; ++t) {
      SelTerm tm = p.terms[en.t0 + t];
      src += ((eta / tm.pv) % tm.dim) * tm.stride;
    }
    p.out[en.dst] = p.lval[src];
  }
}

__global__ void k_rootcopy(const RootCopyParams p) {
  pdl_launch();
  pdl_wait();
  const int64_t slot = slice_lex(p.ord, p.eta[0]) - p.eta[1];  // the slice's lexicographic row
  double* results = *p.results;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < p.R;
       r += (int64_t)gridDim.x * blockDim.x) {
    // tied root indices: dense entries off the diagonal are structural zeros
    const int64_t m = p.map ? p.map[r] : r;
    results[slot * p.R + r] = m >= 0 ? p.src[m] : 0.0;
  }
}

// eta = [current slice (iteration id), first slice of the pass, stride K*B,
// lane's first offset k*B, slices per block B, mode].  Mode 0: a lane runs B
// consecutive iteration ids, then jumps to its next block (B = 1: every K-th
// slice).  Mode 1 (a range that the slice order does not map onto itself):
// the lane walks lexicographic ids b + k, b + k + K, ... (B = 1), held as
// their iteration ids.
__global__ void k_eta(int64_t* eta, const int64_t* ord) {
  pdl_launch();
  pdl_wait();
  if (eta[5]) {
    eta[0] = slice_iter(ord, slice_lex(ord, eta[0]) + eta[2]);
    return;
  }
  int64_t t = eta[0] + 1;
  if ((t - eta[1]) % eta[4] == 0) t += eta[2] - eta[4];
  eta[0] = t;
}
__global__ void k_eta_reset(int64_t* eta, const int64_t* ord) {
  eta[0] = eta[5] ? slice_iter(ord, eta[1] + eta[3]) : eta[1] + eta[3];
}

// L2 eviction between timed passes (benchmark only): stream a scratch buffer
__global__ void k_flush(double4* buf, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = make_double4(v, v, v, v);
}

// left fold in lexicographic slice order: ((p0 + p1) + p2) + ...  (tensor.py:111-115)
__global__ void k_fold(const double* results, int64_t R, int64_t n, double* out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = results[r];
    for (int64_t s = 1; s < n; ++s) acc = acc + results[s * R + r];
    out[r] = acc;
  }
}

// ---------------------------------------------------------------------------
// K4: one CTA walks one tiny subtree in postorder; intermediates live in smem.
constexpr int kTinyThreads = 1 << kTinyThreadsLog;
__device__ long long* g_tiny_trace = nullptr;  // diagnostics: node start clocks of block 0 (TC_TINY_TRACE)

// one dim-2 tiny node (k_tiny): thread -> output c0 + k * 2^cl, the low cl
// output bits fixed per thread, the high ones and the summed bits above lw
// stepping through carry tables.  Operands and output never overlap (the
// group's smem allocator frees a node's children after placing its output).
__device__ __forceinline__ void tiny_pow2(const double* __restrict__ A, const double* __restrict__ B,
                                          double* __restrict__ C, const TinyNode& tn, const TinyDigit* sd,
                                          const int* dAr, const int* dBr, const int* hAr, const int* hBr, int tid,
                                          int lane, int tlog) {
  // tid: the thread's index among the node's 2^tlog threads (a warp or the CTA)
  const int nc = tn.nc;
  const TinyDigit* sdS = sd + nc;
  const int lw = tn.lw, W = 1 << lw, cl = tlog - lw;
  const int r = lane & (W - 1), c0 = tid >> lw;
  const unsigned mask = (W == 32 ? 0xffffffffu : ((1u << W) - 1u) << (lane & ~(W - 1)));
  if (c0 >= tn.c_size) return;
  int xa = 0, xb = 0;
  // fixed trip counts: every digit load issues at once (no dependent chain)
#pragma unroll
  for (int j = 0; j < 5; ++j)
    if (j < lw && ((r >> j) & 1)) xa += sdS[j].sa, xb += sdS[j].sb;
#pragma unroll
  for (int j = 0; j < kTinyThreadsLog; ++j)
    if (j < cl && j < nc && ((c0 >> j) & 1)) xa += sd[j].sa, xb += sd[j].sb;
  const int nk = nc > cl ? 1 << (nc - cl) : 1;
  const int nq = tn.s_size >> lw;
  for (int k = 0; k < nk; ++k) {
    if (k) {
      const int t = __ffs(k) - 1;
      xa += hAr[t];
      xb += hBr[t];
    }
    int ya = xa, yb = xb;
    double acc0 = 0.0, acc1 = 0.0;
    for (int q = 0; q < nq; ++q) {
      if (q) {
        const int t = __ffs(q) - 1;
        ya += dAr[t];
        yb += dBr[t];
      }
      if (q & 1) acc1 = fma(A[ya], B[yb], acc1);
      else acc0 = fma(A[ya], B[yb], acc0);
    }
    double acc = acc0 + acc1;
    for (int o = W >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o);
    if (r == 0) C[c0 + (k << cl)] = acc;
  }
}

// smem: [intermediates: smem_doubles][reduce: kTinyThreads][staged operands:
// stage_doubles][kTinyBatch TinyNode][dig_max TinyDigit]
__global__ void __launch_bounds__(kTinyThreads) k_tiny(const TinyNode* __restrict__ nodes,
                                                       const TinyDigit* __restrict__ digs,
                                                       const TinyGroup* __restrict__ groups,
                                                       int32_t smem_doubles, int32_t stage_doubles) {
  extern __shared__ double sm[];
  double* red = sm + smem_doubles;  // kTinyThreads scratch for cooperative sums
  double* stg = red + kTinyThreads;
  TinyNode* bn = (TinyNode*)(stg + stage_doubles);
  TinyDigit* bd = (TinyDigit*)(bn + kTinyBatch);
  __shared__ int dA[kTinyBatch][kTinyMaxSum], dB[kTinyBatch][kTinyMaxSum];
  __shared__ int hA[kTinyBatch][kTinyMaxSum], hB[kTinyBatch][kTinyMaxSum];
  pdl_launch();
  pdl_wait();
#ifdef TC_DIAG_TINY_SKIP  // diagnostics build only: tiny launches do no work (timing bound)
  return;
#endif
  const TinyGroup G = groups[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long* const trace = (blockIdx.x == 0 && tid == 0) ? g_tiny_trace : nullptr;
  for (int b0 = G.beg; b0 < G.end; b0 += kTinyBatch) {
    const int cnt = min(kTinyBatch, G.end - b0);
    // Batch prologue: every global load of a round is issued before any of
    // its shared stores (fixed trip counts), so a round costs one round trip.
    constexpr int kWords = kTinyBatch * (int)(sizeof(TinyNode) / 4);
    constexpr int kWordIt = (kWords + kTinyThreads - 1) / kTinyThreads;
    const int words = cnt * (int)(sizeof(TinyNode) / 4);
    const int* src = (const int*)(nodes + b0);
    int wv[kWordIt];
#pragma unroll
    for (int k = 0; k < kWordIt; ++k)
      if (tid + k * kTinyThreads < words) wv[k] = src[tid + k * kTinyThreads];
    const int dig0 = nodes[b0].dig;
    const int dig1 = nodes[b0 + cnt - 1].dig + nodes[b0 + cnt - 1].nc + nodes[b0 + cnt - 1].ns;
    TinyDigit dv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (tid + k * kTinyThreads < dig1 - dig0) dv[k] = digs[dig0 + tid + k * kTinyThreads];
    __syncthreads();  // the previous batch is done with the staging buffers
#pragma unroll
    for (int k = 0; k < kWordIt; ++k)
      if (tid + k * kTinyThreads < words) ((int*)bn)[tid + k * kTinyThreads] = wv[k];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (tid + k * kTinyThreads < dig1 - dig0) bd[tid + k * kTinyThreads] = dv[k];
    for (int j = tid + 4 * kTinyThreads; j < dig1 - dig0; j += blockDim.x) bd[j] = digs[dig0 + j];
    __syncthreads();
    // small global operands (<= kTinyStageMax entries): warp w takes operands
    // w, w + 8, ...; lanes over entries
    {
      constexpr int kOpIt = 2 * kTinyBatch / (kTinyThreads / 32);
      constexpr int kEntIt = kTinyStageMax / 32;
      double v[kOpIt][kEntIt];
#pragma unroll
      for (int k = 0; k < kOpIt; ++k) {
        const int o = warp + k * (kTinyThreads / 32);
        if (o >= 2 * cnt) continue;
        const TinyNode& t = bn[o >> 1];
        const int st = (o & 1) ? t.stb : t.sta;
        const double* g = (o & 1) ? t.gb : t.ga;
        const int n = (o & 1) ? t.nb : t.na;
#pragma unroll
        for (int e = 0; e < kEntIt; ++e)
          if (st >= 0 && lane + 32 * e < n) v[k][e] = g[lane + 32 * e];
      }
#pragma unroll
      for (int k = 0; k < kOpIt; ++k) {
        const int o = warp + k * (kTinyThreads / 32);
        if (o >= 2 * cnt) continue;
        const TinyNode& t = bn[o >> 1];
        const int st = (o & 1) ? t.stb : t.sta;
        const int n = (o & 1) ? t.nb : t.na;
#pragma unroll
        for (int e = 0; e < kEntIt; ++e)
          if (st >= 0 && lane + 32 * e < n) stg[st + lane + 32 * e] = v[k][e];
      }
    }
    // dim-2 nodes: 2^lw lanes split each output's sum; lane r takes the
    // terms whose low lw summed bits equal r.  Stepping a counter q -> q+1
    // flips q's low ones to 0 and bit t = ctz(q+1) to 1, so an offset moves by
    // stride_t - sum_{i<t} stride_i: dA/dB for the summed bits above lw, hA/hB
    // for the output bits above the (kTinyThreadsLog - lw) a thread fixes.
    if (tid < cnt && bn[tid].pow2) {
      const TinyNode& t = bn[tid];
      const TinyDigit* D = bd + (t.dig - dig0);
      int pa = 0, pb = 0;
      for (int j = t.lw; j < t.ns && j - t.lw < kTinyMaxSum; ++j) {
        dA[tid][j - t.lw] = D[t.nc + j].sa - pa;
        dB[tid][j - t.lw] = D[t.nc + j].sb - pb;
        pa += D[t.nc + j].sa;
        pb += D[t.nc + j].sb;
      }
      pa = pb = 0;
      const int tl = t.wofs >= 0 ? 5 : kTinyThreadsLog;
      for (int j = tl - t.lw; j < t.nc; ++j) {
        const int k = j - (tl - t.lw);
        hA[tid][k] = D[j].sa - pa;
        hB[tid][k] = D[j].sb - pb;
        pa += D[j].sa;
        pb += D[j].sb;
      }
    }
    __syncthreads();
    for (int i = 0; i < cnt; ++i) {
      const TinyNode& tn = bn[i];
      if (trace) trace[b0 + i] = clock64();
      if (i > 0 && tn.sync) {
        if (tn.sync == 1) __syncthreads();
        else if (warp == 0) __syncwarp();  // hazard among warp-0-only nodes
      }
      // a single-warp node runs on its warp only (the other warps run the
      // other nodes of its wave); ltid / nthr index the node's threads
      if (tn.wofs >= 0 && warp != tn.wofs) continue;
      const int ltid = tn.wofs >= 0 ? lane : tid, nthr = tn.wofs >= 0 ? 32 : (int)blockDim.x;
      const int tlog = tn.wofs >= 0 ? 5 : kTinyThreadsLog;
      const TinyDigit* sd = bd + (tn.dig - dig0);
      const double* A = tn.sa >= 0 ? sm + tn.sa : tn.ga;  // (compile.cpp resolves staged / smem / global)
      const double* B = tn.sb >= 0 ? sm + tn.sb : tn.gb;
      double* C = tn.sout >= 0 ? sm + tn.sout : tn.gout;
      const int nc = tn.nc, ns = tn.ns;
      const TinyDigit* sdS = sd + nc;
      if (tn.pow2 && ns - tn.lw <= kTinyMaxSum) {
        tiny_pow2(A, B, C, tn, sd, dA[i], dB[i], hA[i], hB[i], ltid, lane, tlog);
      } else if (tn.c_size * 4 >= (int)blockDim.x || tn.s_size < 64) {
        for (int c = ltid; c < tn.c_size; c += nthr) {
          int oa = 0, ob = 0;
          if (tn.pow2) {
            for (int j = 0; j < nc; ++j) {
              int bit = (c >> j) & 1;
              oa += bit * sd[j].sa;
              ob += bit * sd[j].sb;
            }
          } else {
            int r = c;
            for (int j = 0; j < nc; ++j) {
              int q = r % sd[j].dim;
              r /= sd[j].dim;
              oa += q * sd[j].sa;
              ob += q * sd[j].sb;
            }
          }
          double acc = 0.0;
          for (int s = 0; s < tn.s_size; ++s) {
            int xa = oa, xb = ob;
            if (tn.pow2) {
              for (int j = 0; j < ns; ++j) {
                int bit = (s >> j) & 1;
                xa += bit * sdS[j].sa;
                xb += bit * sdS[j].sb;
              }
            } else {
              int r = s;
              for (int j = 0; j < ns; ++j) {
                int q = r % sdS[j].dim;
                r /= sdS[j].dim;
                xa += q * sdS[j].sa;
                xb += q * sdS[j].sb;
              }
            }
            acc = fma(A[xa], B[xb], acc);
          }
          C[c] = acc;
        }
      } else {
        // few outputs, long sums: the CTA splits each sum, fixed-shape tree reduce
        for (int c = 0; c < tn.c_size; ++c) {
          int oa = 0, ob = 0, r = c;
          for (int j = 0; j < nc; ++j) {
            int q = r % sd[j].dim;
            r /= sd[j].dim;
            oa += q * sd[j].sa;
            ob += q * sd[j].sb;
          }
          double acc = 0.0;
          for (int s = tid; s < tn.s_size; s += blockDim.x) {
            int xa = oa, xb = ob, r2 = s;
            for (int j = 0; j < ns; ++j) {
              int q = r2 % sdS[j].dim;
              r2 /= sdS[j].dim;
              xa += q * sdS[j].sa;
              xb += q * sdS[j].sb;
            }
            acc = fma(A[xa], B[xb], acc);
          }
          red[tid] = acc;
          __syncthreads();
          for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (tid < w) red[tid] = red[tid] + red[tid + w];
            __syncthreads();
          }
          if (tid == 0) C[c] = red[0];
          __syncthreads();
        }
      }
    }
  }
  if (trace) trace[G.end] = clock64();
}

// ---------------------------------------------------------------------------
// K2: streaming contraction with a <=64-entry operand held in smem.
// C[x, f] = sum_s A[x, s] P[b(x), s, f]; b(x) are the batch bits of x (tied
// variables shared by A, P and C), usually none.  A diagonal read adds a
// second A address bit per x bit (xa2).
constexpr int kStreamThreads = 256;
constexpr int kStreamUnroll = 4;

// One stream step executed by CTA `b` of 2^logG CTAs.  The 2^cl chunks split
// into 2^g CTA blocks of 2^kchunk chunks each (CTAs beyond the chunk count
// idle), or, for large launches (p.persist), a grid-stride walk over them.
template <int NS, int NF>
__device__ __forceinline__ void stream_run(const StreamParams& p, double* Ps, int b, int logG) {
  constexpr int SV = 1 << NS, FV = 1 << NF, SVFV = SV * FV;
  constexpr int CB = kStreamChunkBits;
  static_assert((kStreamThreads * kStreamUnroll) == (1 << CB), "chunk");
  static_assert(kStreamThreads == 256 && kStreamUnroll == 4, "x = base + u*256 + tid");
  const int tid = threadIdx.x;
  const int xb = 63 - __clzll((long long)p.nx);  // nx is a power of two
  const int cl = max(0, xb - CB);
  int kchunk = 0, cb = b, u0 = -1;
  if (p.persist) {
    cb = 0;  // chunks are assigned in the grid-stride loop below
  } else if (p.split_u) {  // one quarter of one chunk per CTA
    cb = b >> 2;
    u0 = b & 3;
    if (cb >= (1 << cl)) return;
    kchunk = 0;
  } else {
    const int g = min(logG, cl);
    if (b >= (1 << g)) return;
    kchunk = cl - g;
  }
  const bool staged = p.stage_all;
  // x = chunk * 2^CB + u * 256 + tid.  Every address is a sum of per-bit
  // table entries: the thread's low parts once, the CTA's chunk bits once,
  // then each step of the Gray-code chunk walk flips one bit (one add).
  int64_t ta = 0, tcc = 0, tpo = 0;
  int tp = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if ((tid >> j) & 1) {
      ta += p.bitA[j];
      tcc += p.bitC[j];
      tp += p.bitP[j];
      tpo += p.bitPo[j];
    }
  int64_t lo_a[kStreamUnroll], lo_c[kStreamUnroll], lo_p[kStreamUnroll];
#pragma unroll
  for (int u = 0; u < kStreamUnroll; ++u) {
    lo_a[u] = ta + ((u & 1) ? p.bitA[8] : 0) + ((u & 2) ? p.bitA[9] : 0);
    lo_c[u] = tcc + ((u & 1) ? p.bitC[8] : 0) + ((u & 2) ? p.bitC[9] : 0);
    lo_p[u] = staged ? (int64_t)(tp + ((u & 1) ? p.bitP[8] : 0) + ((u & 2) ? p.bitP[9] : 0)) * SVFV
                     : tpo + ((u & 1) ? p.bitPo[8] : 0) + ((u & 2) ? p.bitPo[9] : 0);
  }
  // this CTA's fixed chunk bits
  int64_t ha = 0, hc = 0, hp = 0;
  {
    uint64_t m = (uint64_t)cb << (kchunk + CB);
    while (m) {
      const int j = __ffsll((long long)m) - 1;
      m &= m - 1;
      ha += p.bitA[j];
      hc += p.bitC[j];
      hp += staged ? (int64_t)p.bitP[j] * SVFV : p.bitPo[j];
    }
  }
  // everything above reads kernel parameters only: under programmatic
  // dependencies it overlaps the predecessor; operand data is read below
  pdl_wait();
  // the first chunk's big-operand loads are issued before the small operand
  // is staged: the two global round trips overlap
  // (small summed shapes only: the early live range costs registers)
  constexpr bool kHoist = NS <= 2;
  const bool full = p.nx >= (1 << CB);
  double a[kStreamUnroll][SV];
  if (kHoist && full && !p.persist) {
#pragma unroll
    for (int u = 0; u < kStreamUnroll; ++u)
      if (u0 < 0 || u == u0)
#pragma unroll
        for (int s = 0; s < SV; ++s) a[u][s] = __ldg(p.A + ha + lo_a[u] + p.offA[s]);
  }
  if (staged) {
    for (int q = tid; q < (SVFV << p.nbt); q += blockDim.x) {
      const int bi = q / SVFV;
      int64_t off = p.offP[q % SVFV];
      for (int t = 0; t < p.nbt; ++t)
        if ((bi >> t) & 1) off += p.bt_poff[t];
      Ps[q] = p.P[off];
    }
    __syncthreads();
  }
  const double* Pbase = staged ? Ps : p.P;
  auto pv = [&](const double* Pu, int q) { return staged ? Pu[q] : __ldg(Pu + p.offP[q]); };
  if (p.persist) {
    // grid-stride over the chunks (one wave of resident CTAs: no partial
    // last wave); a chunk's address parts are summed from the tables
    const int64_t nch = (int64_t)1 << cl;
    for (int64_t c = b; c < nch; c += gridDim.x) {
      int64_t qa = 0, qc = 0, qp = 0;
      uint64_t m = (uint64_t)c << CB;
      while (m) {
        const int j = __ffsll((long long)m) - 1;
        m &= m - 1;
        qa += p.bitA[j];
        qc += p.bitC[j];
        qp += staged ? (int64_t)p.bitP[j] * SVFV : p.bitPo[j];
      }
      const double* Ab = p.A + qa;
      double* Cb = p.C + qc;
      const double* Pc = Pbase + qp;
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u)
#pragma unroll
        for (int s = 0; s < SV; ++s) a[u][s] = __ldg(Ab + lo_a[u] + p.offA[s]);
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) {
        const double* Pu = Pc + lo_p[u];
        double* Cu = Cb + lo_c[u];
#pragma unroll
        for (int f = 0; f < FV; ++f) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < SV; ++s) acc = fma(a[u][s], pv(Pu, s * FV + f), acc);
          Cu[p.offC[f]] = acc;
        }
      }
    }
    return;
  }
  const int64_t nsteps = (int64_t)1 << kchunk;
  for (int64_t i = 0; i < nsteps; ++i) {
    if (i > 0) {  // Gray code: chunk bit ctz(i) flips
      const int j = __ffsll((long long)i) - 1 + CB;
      const int64_t sg = (((i ^ (i >> 1)) >> (j - CB)) & 1) ? 1 : -1;
      ha += sg * p.bitA[j];
      hc += sg * p.bitC[j];
      hp += sg * (staged ? (int64_t)p.bitP[j] * SVFV : p.bitPo[j]);
    }
    const double* Ab = p.A + ha;
    double* Cb = p.C + hc;
    const double* Pc = Pbase + hp;
    if (full) {
      if (!kHoist || i > 0) {
#pragma unroll
        for (int u = 0; u < kStreamUnroll; ++u)
          if (u0 < 0 || u == u0)
#pragma unroll
            for (int s = 0; s < SV; ++s) a[u][s] = __ldg(Ab + lo_a[u] + p.offA[s]);
      }
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) {
        if (u0 >= 0 && u != u0) continue;
        const double* Pu = Pc + lo_p[u];
        double* Cu = Cb + lo_c[u];
#pragma unroll
        for (int f = 0; f < FV; ++f) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < SV; ++s) acc = fma(a[u][s], pv(Pu, s * FV + f), acc);
          Cu[p.offC[f]] = acc;
        }
      }
    } else {  // a single partial chunk (nx < 2^CB)
      for (int u = 0; u < kStreamUnroll; ++u) {
        if (u * kStreamThreads + tid >= p.nx || (u0 >= 0 && u != u0)) continue;
        const double* Pu = Pc + lo_p[u];
        for (int f = 0; f < FV; ++f) {
          double acc = 0.0;
          for (int s = 0; s < SV; ++s) acc = fma(Ab[lo_a[u] + p.offA[s]], pv(Pu, s * FV + f), acc);
          Cb[lo_c[u] + p.offC[f]] = acc;
        }
      }
    }
  }
}

// Resident CTAs per SM the register allocation must allow.  The streams are
// latency-hiding bound: 6 CTAs (<= 40 registers) for the common small shapes
// beat the compiler's 58-64 registers / 4 CTAs by 17% on C4 (1380 -> 1144 ms,
// measured; 8 CTAs spill and gain nothing more).
#ifndef TC_STREAM_MINB
#define TC_STREAM_MINB 6
#endif
template <int NS, int NF>
constexpr int stream_minb() { return NS + NF <= 3 ? TC_STREAM_MINB : 1; }  // larger shapes: no spills
template <int NS, int NF>
__global__ void __launch_bounds__(kStreamThreads, stream_minb<NS, NF>()) k_stream(const StreamParams p) {
  __shared__ double Ps[kStreamStageMax];  // staged small operand (stage_all)
  // operands are produced by earlier launches: stream_run waits (pdl_wait)
  // after its parameter-only address prologue
  stream_run<NS, NF>(p, Ps, blockIdx.x, 31 - __clz(gridDim.x));
  pdl_launch();  // dependents start as this CTA retires (overlap the tail only)
}

// K2p: two chained stream steps, the intermediate in registers (see program.h).
// NI inner bits, step-1 shape (NS1 summed, NF1 new), step-2 shape (NS2, NF2).
template <int NI, int NS1, int NF1, int NS2, int NF2>
__global__ void __launch_bounds__(kStreamThreads, NI <= 2 ? TC_STREAM_MINB : 1) k_stream_pair(const StreamPairParams p) {
  constexpr int NQ = 1 << NI, SV1 = 1 << NS1, FV1 = 1 << NF1, SV2 = 1 << NS2, FV2 = 1 << NF2;
  constexpr int NR = NQ / SV2;  // rest combos
  constexpr int CB = kStreamChunkBits;
  const int tid = threadIdx.x;
  // per-thread low parts of the y address tables (y = chunk * 2^CB + u * 256 + tid)
  int64_t ta = 0, tc = 0, t1 = 0, t2 = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if ((tid >> j) & 1) ta += p.bitA[j], tc += p.bitC[j], t1 += p.bitP1[j], t2 += p.bitP2[j];
  int64_t la[kStreamUnroll], lc[kStreamUnroll], l1[kStreamUnroll], l2[kStreamUnroll];
#pragma unroll
  for (int u = 0; u < kStreamUnroll; ++u) {
    la[u] = ta + ((u & 1) ? p.bitA[8] : 0) + ((u & 2) ? p.bitA[9] : 0);
    lc[u] = tc + ((u & 1) ? p.bitC[8] : 0) + ((u & 2) ? p.bitC[9] : 0);
    l1[u] = t1 + ((u & 1) ? p.bitP1[8] : 0) + ((u & 2) ? p.bitP1[9] : 0);
    l2[u] = t2 + ((u & 1) ? p.bitP2[8] : 0) + ((u & 2) ? p.bitP2[9] : 0);
  }
  const int cl = max(0, p.ybits - CB);
  const int logG = 31 - __clz(gridDim.x);
  const int b = blockIdx.x;
  int kchunk = 0, cb = b, u0 = -1;
  if (p.persist) {
    cb = 0;  // grid-stride over the chunks (walk below)
  } else if (p.split_u) {  // one quarter of one chunk per CTA
    cb = b >> 2;
    u0 = b & 3;
    if (cb >= (1 << cl)) return;
    kchunk = 0;
  } else {
    const int g = min(logG, cl);
    if (b >= (1 << g)) return;
    kchunk = cl - g;
  }
  int64_t ha = 0, hc = 0, h1 = 0, h2 = 0;
  {
    uint64_t m = (uint64_t)cb << (kchunk + CB);
    while (m) {
      const int j = __ffsll((long long)m) - 1;
      m &= m - 1;
      ha += p.bitA[j], hc += p.bitC[j], h1 += p.bitP1[j], h2 += p.bitP2[j];
    }
  }
  // parameters only so far (overlaps the predecessor under programmatic
  // dependencies); operand data is read below
  pdl_wait();
  // the chain walk, over global or smem-staged small operands (each call
  // site inlines with its own address space)
  auto walk = [&](const double* __restrict__ P1, const double* __restrict__ P2) {
    const int64_t ny = (int64_t)1 << p.ybits;
    const int64_t nsteps = p.persist ? ((((int64_t)1 << cl) - b + gridDim.x - 1) / gridDim.x) : (int64_t)1 << kchunk;
    for (int64_t i = 0; i < nsteps; ++i) {
      if (p.persist) {  // chunk b + i * grid: address parts summed from the tables
        ha = hc = h1 = h2 = 0;
        uint64_t m = (uint64_t)(b + i * (int64_t)gridDim.x) << CB;
        while (m) {
          const int j = __ffsll((long long)m) - 1;
          m &= m - 1;
          ha += p.bitA[j], hc += p.bitC[j], h1 += p.bitP1[j], h2 += p.bitP2[j];
        }
      } else if (i > 0) {
        const int j = __ffsll((long long)i) - 1 + CB;
        const int64_t sg = (((i ^ (i >> 1)) >> (j - CB)) & 1) ? 1 : -1;
        ha += sg * p.bitA[j], hc += sg * p.bitC[j], h1 += sg * p.bitP1[j], h2 += sg * p.bitP2[j];
      }
  #pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) {
        if ((ny < (1 << CB) && u * kStreamThreads + tid >= ny) || (u0 >= 0 && u != u0)) continue;
        const double* Ab = p.A + ha + la[u];
        const double* P1b = P1 + h1 + l1[u];
        const double* P2b = P2 + h2 + l2[u];
        double* Cb = p.C + hc + lc[u];
        // step 1 for every inner combo (loads shared by combos with equal A offset)
        double c1[NQ];
  #pragma unroll
        for (int q = 0; q < NQ; ++q) {
          double acc = 0.0;
  #pragma unroll
          for (int s = 0; s < SV1; ++s)
            acc = fma(__ldg(Ab + p.qA[q] + p.offA1[s]), P1b[p.qP1[q] + p.offP1[s * FV1 + p.qF1[q]]], acc);
          c1[q] = acc;
        }
        // step 2: every (rest, f2) output sums its SV2 inner combos in s2 order
  #pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int q0 = r << NS2;  // s2 = 0 combo of this rest (P2 batch / C2 offsets)
  #pragma unroll
          for (int f = 0; f < FV2; ++f) {
            double acc = 0.0;
  #pragma unroll
            for (int s = 0; s < SV2; ++s) {
              acc = fma(c1[s | (r << NS2)], P2b[p.qP2[q0] + p.offP2[s * FV2 + f]], acc);
            }
            Cb[p.qC[q0] + p.offC2[f]] = acc;
          }
        }
      }
    }
  };
  // small operands staged in smem once per CTA (p.pstage): every FMA's
  // operand then comes from a broadcast smem read instead of the L1
  if (p.pstage) {
    extern __shared__ double psm[];
    for (int i = tid; i < p.p1n; i += blockDim.x) psm[i] = __ldg(p.P1 + i);
    for (int i = tid; i < p.p2n; i += blockDim.x) psm[p.p1n + i] = __ldg(p.P2 + i);
    __syncthreads();
    walk(psm, psm + p.p1n);
  } else {
    walk(p.P1, p.P2);
  }
  pdl_launch();
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// K3: FP64 tensor-core GEMM family.  CTA tile BMxBNx16 (BM, BN in 8..64),
// WGM x WGN warps, each warp a (BM/WGM)x(BN/WGN) block of DMMA m8n8k4
// fragments; 4-stage cp.async pipeline.  Operands are gathered with
// per-thread precomputed tile offsets (any bit layout: the index permutation
// of tensordot is folded into the loads), stored k-major in smem with +4
// padding (conflict-free fragment loads).  The C tile is staged through smem
// and written in C's own address order (coalesced for any output layout).
constexpr int GBK = 16, GSTAGES = 4;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// element e of a tile -> (address offset, row coord, k coord); false if virtual
__device__ __forceinline__ bool tile_elem(const TileMap& t, int e, int64_t& off, int& r, int& k) {
  off = 0;
  r = 0;
  k = 0;
  bool real = true;
  for (int j = 0; j < t.nbits; ++j)
    if ((e >> j) & 1) {
      if (t.pos[j] < 0) real = false;
      else off += (int64_t)1 << t.pos[j];
      if (t.kind[j]) k |= 1 << t.sub[j];
      else r |= 1 << t.sub[j];
    }
  return real;
}

template <int BM, int BN, int WGM, int WGN>
struct GemmCfg {
  static constexpr int NT = 32 * WGM * WGN;
  static constexpr int LDA = BM + 4, LDB = BN + 4, LDC = BN + 4;
  static constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int ELA = (BM * GBK + NT - 1) / NT, ELB = (BN * GBK + NT - 1) / NT;
  // 3 stages for the 4-warp tiles so 4 CTAs fit an SM (occupancy over depth)
  static constexpr int ST = (WGM * WGN == 4) ? 3 : GSTAGES;
  static constexpr int SMEM = ST * GBK * (LDA + LDB) * 8 > BM * LDC * 8 ? ST * GBK * (LDA + LDB) * 8 : BM * LDC * 8;
  static_assert(FM >= 1 && FN >= 1, "warp tile below 8x8");
};

template <int BM, int BN, int WGM, int WGN>
__global__ void __launch_bounds__(32 * WGM * WGN, (WGM * WGN >= 8) ? 2 : 4)
    k_gemm(const GemmParams p) {
  using Cfg = GemmCfg<BM, BN, WGM, WGN>;
  constexpr int NT = Cfg::NT, LDA = Cfg::LDA, LDB = Cfg::LDB, LDC = Cfg::LDC;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, ELA = Cfg::ELA, ELB = Cfg::ELB;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + Cfg::ST * GBK * LDA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WGN, wn = warp % WGN;

  // tile coordinates with a grouped walk over m for L2 reuse of B; batch
  // variables (tied networks) index the grid above the tiles
  const int tbits = p.m_hi + p.n_hi;
  const int64_t bt = (int64_t)blockIdx.x >> tbits;
  const int64_t t = (int64_t)blockIdx.x & (((int64_t)1 << tbits) - 1);
  const int g = p.grid_swizzle_log;
  const int64_t gsz = (int64_t)1 << g;
  const int64_t ntn = (int64_t)1 << p.n_hi;
  const int64_t grp = t / (gsz * ntn), in = t % (gsz * ntn);
  const int64_t tm = grp * gsz + (in & (gsz - 1));
  const int64_t tn = in >> g;
  const int split = blockIdx.y;
  const int64_t kt0 = split * p.k_per_split;
  const int64_t kt1 = min(p.k_tiles, kt0 + p.k_per_split);
  const int64_t nkt = kt1 > kt0 ? kt1 - kt0 : 0;

  // tile element e = tid + i*NT decomposes additively: thread part in
  // registers + block part in a small smem table (keeps registers low)
  __shared__ int64_t ha_off[ELA], hb_off[ELB];
  __shared__ int ha_sx[ELA], hb_sx[ELB];
  __shared__ bool ha_ok[ELA], hb_ok[ELB];
  if (tid < ELA) {
    int r, k;
    ha_ok[tid] = tile_elem(p.ta, tid * NT, ha_off[tid], r, k) && tid * NT < BM * GBK;
    ha_sx[tid] = k * LDA + r;
  }
  if (tid < ELB) {
    int r, k;
    hb_ok[tid] = tile_elem(p.tb, tid * NT, hb_off[tid], r, k) && tid * NT < BN * GBK;
    hb_sx[tid] = k * LDB + r;
  }
  int64_t aoff_t, boff_t;
  int asx_t, bsx_t;
  bool aok_t, bok_t;
  {
    int r, k;
    aok_t = tile_elem(p.ta, tid, aoff_t, r, k);
    asx_t = k * LDA + r;
    bok_t = tile_elem(p.tb, tid, boff_t, r, k);
    bsx_t = k * LDB + r;
  }
  __syncthreads();
  // virtual elements are zero in every stage and never loaded
  for (int i = 0; i < ELA; ++i)
    if (tid + i * NT < BM * GBK && !(aok_t && ha_ok[i]))
      for (int s = 0; s < Cfg::ST; ++s) As[s * GBK * LDA + asx_t + ha_sx[i]] = 0.0;
  for (int i = 0; i < ELB; ++i)
    if (tid + i * NT < BN * GBK && !(bok_t && hb_ok[i]))
      for (int s = 0; s < Cfg::ST; ++s) Bs[s * GBK * LDB + bsx_t + hb_sx[i]] = 0.0;
  pdl_wait();  // operands are produced by earlier launches
  const double* Ab = p.A + deposit(tm, p.a_m) + deposit(bt, p.a_bt);
  const double* Bb = p.B + deposit(tn, p.b_n) + deposit(bt, p.b_bt);

  auto load_stage = [&](int stage, int64_t kt) {
    const double* Ag = Ab + deposit(kt, p.a_k);
    const double* Bg = Bb + deposit(kt, p.b_k);
    double* as = As + stage * GBK * LDA;
    double* bs = Bs + stage * GBK * LDB;
    if (aok_t) {
#pragma unroll
      for (int i = 0; i < ELA; ++i)
        if (ha_ok[i]) cp_async8(as + asx_t + ha_sx[i], Ag + aoff_t + ha_off[i]);
    }
    if (bok_t) {
#pragma unroll
      for (int i = 0; i < ELB; ++i)
        if (hb_ok[i]) cp_async8(bs + bsx_t + hb_sx[i], Bg + boff_t + hb_off[i]);
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < Cfg::ST - 1; ++s) {
    if (s < nkt) load_stage(s, kt0 + s);
    cp_async_commit();
  }
  for (int64_t it = 0; it < nkt; ++it) {
    cp_async_wait<Cfg::ST - 2>();
    __syncthreads();
    {
      int64_t nk = it + Cfg::ST - 1;
      if (nk < nkt) load_stage((int)(nk % Cfg::ST), kt0 + nk);
      cp_async_commit();
    }
    const double* as = As + (it % Cfg::ST) * GBK * LDA;
    const double* bs = Bs + (it % Cfg::ST) * GBK * LDB;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double af[FM], bf[FN];
      const int kr = kk * 4 + (lane & 3);
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = as[kr * LDA + wm * Cfg::WTM + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = bs[kr * LDB + wn * Cfg::WTN + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  pdl_launch();  // main loop done: dependents may start their prologue
  __syncthreads();
  double* Cs = gsm;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int row = wm * Cfg::WTM + i * 8 + (lane >> 2);
      const int col = wn * Cfg::WTN + j * 8 + (lane & 3) * 2;
      Cs[row * LDC + col] = acc[i][j][0];
      Cs[row * LDC + col + 1] = acc[i][j][1];
    }
  __syncthreads();
  if (p.splits > 1) {
    // partial tile, C-tile element order, contiguous per (split, tile)
    double* W = p.ws + ((int64_t)split * gridDim.x + blockIdx.x) * (BM * BN);
    for (int e = tid; e < BM * BN; e += NT) {
      int64_t off;
      int r, k;
      tile_elem(p.tc, e, off, r, k);
      W[e] = Cs[r * LDC + k];
    }
    return;
  }
  // C element e = tid + i*NT: offset/slot split into a thread part and a
  // block part (table), so the scatter costs one add per element
  constexpr int ELC = BM * BN / NT;
  __shared__ int64_t hc_off[ELC];
  __shared__ int hc_sx[ELC];
  __shared__ bool hc_ok[ELC];
  if (tid < ELC) {
    int r, k;
    hc_ok[tid] = tile_elem(p.tc, tid * NT, hc_off[tid], r, k);
    hc_sx[tid] = r * LDC + k;
  }
  int64_t c_off_t;
  int rt, kt_;
  const bool c_ok_t = tile_elem(p.tc, tid, c_off_t, rt, kt_);
  const int c_sx_t = rt * LDC + kt_;
  __syncthreads();
  double* Cg = p.C + deposit(tm, p.c_m) + deposit(tn, p.c_n) + deposit(bt, p.c_bt);
  if (c_ok_t) {
#pragma unroll 8
    for (int i = 0; i < ELC; ++i)
      if (hc_ok[i]) Cg[c_off_t + hc_off[i]] = Cs[c_sx_t + hc_sx[i]];
  }
}

// fixed-order split-K reduction: C = ((W0 + W1) + W2) + ...
__global__ void k_splitk_reduce(const GemmParams p, int64_t tiles, int tile_elems) {
  pdl_launch();
  pdl_wait();
  const int64_t total = tiles * tile_elems;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ta = id / tile_elems;
    const int e = (int)(id % tile_elems);
    int64_t off;
    int r, k;
    if (!tile_elem(p.tc, e, off, r, k)) continue;
    // loads batched 8 at a time ahead of the (fixed-order) additions: the
    // sum is a dependent chain, the loads need not be
    const double* w = p.ws + ta * tile_elems + e;
    const int64_t step = tiles * tile_elems;
    double acc = w[0];
    int s = 1;
    for (; s + 8 <= p.splits; s += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(w + (s + u) * step);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = acc + v[u];
    }
    for (; s < p.splits; ++s) acc = acc + __ldg(w + s * step);
    const int tbits = p.m_hi + p.n_hi;
    const int64_t bt = ta >> tbits;
    const int64_t t = ta & (((int64_t)1 << tbits) - 1);
    const int g = p.grid_swizzle_log;
    const int64_t gsz = (int64_t)1 << g;
    const int64_t ntn = (int64_t)1 << p.n_hi;
    const int64_t grp = t / (gsz * ntn), in = t % (gsz * ntn);
    const int64_t tm = grp * gsz + (in & (gsz - 1));
    const int64_t tn = in >> g;
    p.C[deposit(tm, p.c_m) + deposit(tn, p.c_n) + deposit(bt, p.c_bt) + off] = acc;
  }
}

// ---------------------------------------------------------------------------
__global__ void k_generic(const GenericParams p) {
  pdl_launch();
  pdl_wait();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < p.c_size;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t oa = 0, ob = 0, r = c;
    for (int j = 0; j < p.nc; ++j) {
      const GDigit d = p.dig[j];
      int64_t q = r % d.dim;
      r /= d.dim;
      oa += q * d.sa;
      ob += q * d.sb;
    }
    double acc = 0.0;
    for (int64_t s = 0; s < p.s_size; ++s) {
      int64_t xa = oa, xb = ob, r2 = s;
      for (int j = 0; j < p.ns; ++j) {
        const GDigit d = p.dig[p.nc + j];
        int64_t q = r2 % d.dim;
        r2 /= d.dim;
        xa += q * d.sa;
        xb += q * d.sb;
      }
      acc = fma(p.A[xa], p.B[xb], acc);
    }
    p.C[c] = acc;
  }
}


}  // namespace tc
