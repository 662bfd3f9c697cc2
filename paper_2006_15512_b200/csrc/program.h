// Device-side parameter blocks shared by the host compiler (compile.cpp) and
// the sm_100a kernels (kernels.cu).  Plain structs, no pointers to host data.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define TC_HD __host__ __device__ __forceinline__
#else
#define TC_HD inline
#endif

namespace tc {

// ---- dim-2 addressing: deposit the bits of a counter into address bits -----
// A tensor whose indices all have domain 2 is a 2^r array; "layout" = which
// index lives at address bit p.  A counter x enumerating some subset of the
// indices maps to an address by moving bit runs: (x >> src) & mask(len) << dst.
constexpr int kMaxRuns = 16;
struct BitRuns {
  int32_t n;
  uint8_t src[kMaxRuns];
  uint8_t len[kMaxRuns];
  uint8_t dst[kMaxRuns];
};

TC_HD int64_t deposit(uint64_t x, const BitRuns& r) {
  uint64_t o = 0;
#pragma unroll
  for (int j = 0; j < kMaxRuns; ++j) {
    if (j >= r.n) break;
    o |= ((x >> r.src[j]) & ((1ull << r.len[j]) - 1ull)) << r.dst[j];
  }
  return (int64_t)o;
}

// the same, as a rolled loop (setup code: fewer instructions and registers)
TC_HD int64_t deposit_rolled(uint64_t x, const BitRuns& r) {
  uint64_t o = 0;
#if defined(__CUDACC__)
#pragma unroll 1
#endif
  for (int j = 0; j < r.n; ++j) o |= ((x >> r.src[j]) & ((1ull << r.len[j]) - 1ull)) << r.dst[j];
  return (int64_t)o;
}

// ---- K2: big x small streaming contraction (dim 2) ------------------------
// C[x, f] = sum_s A[x, s] * P[s, f]; x enumerates the kept indices of the big
// operand A, s the shared ones (<= 2^4), f the small operand's free ones (<= 2^4).
// With tied (physical) variables an x bit may also read a second address
// bit of A (a diagonal read, xa2) and index the small operand (a batch
// variable: P offset bt_poff[t] when x bit bt_xbit[t] is set).  A CTA
// iteration covers 2^kStreamChunkBits consecutive x, so batch bits at or
// above that are fixed per chunk (P's slice for them is staged in smem per
// chunk) and the nlb lower ones select among the staged copies per element.
constexpr int kStreamMaxBatch = 24;
constexpr int kStreamChunkBits = 10;
constexpr int kStreamStageMax = 256;  // doubles of staged P per CTA
constexpr int kStreamXBits = 44;
struct StreamParams {
  const double* A;
  const double* P;
  double* C;
  int64_t nx;
  BitRuns xa, xa2, xc;
  int64_t offA[16];   // s -> offset in A
  int64_t offC[32];   // f -> offset in C
  int32_t offP[128];  // s * 2^NF + f -> offset in P
  int32_t nbt, nlb;   // batch bits (ascending x bit), of which nlb below the chunk
  int32_t bt_xbit[kStreamMaxBatch];
  int64_t bt_poff[kStreamMaxBatch];
  // the low kStreamChunkBits x bits: address contribution of each bit (A incl.
  // diagonal reads, C) and its weight in the staged-P batch index
  // per x bit: address contribution (A incl. diagonal reads, C), batch-index
  // weight (staged mode) and P offset (direct mode).  Deposits are additive
  // over disjoint bits, so any address is a sum of table entries.
  int64_t bitA[kStreamXBits], bitC[kStreamXBits], bitPo[kStreamXBits];
  int32_t bitP[kStreamXBits];
  int32_t stage_all;  // 1: the small operand ((SV*FV) << nbt <= kStreamStageMax entries) is staged
                      //    in smem once per CTA; 0: it is read through the L1 (direct)
  int32_t split_u;    // 1: CTA b takes chunk b >> 2 and only its quarter u = b & 3 (small tensors:
                      //    4x the CTAs, a quarter of the serial work per thread)
  int32_t persist;    // 1: grid-stride over the chunks with one wave of resident CTAs (large launches)
};

// ---- K2p: a chain link of two stream steps in registers ----------------------
// Step 1: C1[x1, f1] = sum_s1 A[x1, s1] P1[b1, s1, f1];  step 2 reads C1:
// C2[x2, f2] = sum_s2 C1[x2, s2] P2[b2, s2, f2].  Threads enumerate y = the C1
// address bits outside F1 (step 1's new bits) and S2 (step 2's summed bits);
// the NI = |F1 u S2| inner bits of C1 live in registers: C1 is never written.
// Every C1 value and every C2 sum is computed with exactly the operations and
// order of the two separate steps (bitwise-identical results).
constexpr int kPairMaxInner = 4;
struct StreamPairParams {
  const double* A;
  const double* P1;
  const double* P2;
  double* C;
  int32_t ybits;  // y counter bits
  int64_t bitA[kStreamXBits], bitC[kStreamXBits], bitP1[kStreamXBits], bitP2[kStreamXBits];
  // per inner combo q (bit t of q = inner bit t): A offset (the S2 bits that are
  // step-1 x bits), step-1 f index, P1 batch offset, step-2 s index, step-2
  // "rest" index (the F1 bits step 2 keeps), P2 batch offset, C2 offset
  int64_t qA[1 << kPairMaxInner], qP1[1 << kPairMaxInner], qP2[1 << kPairMaxInner], qC[1 << kPairMaxInner];
  int32_t qF1[1 << kPairMaxInner], qS2[1 << kPairMaxInner], qR[1 << kPairMaxInner];
  int64_t offA1[16];   // s1 -> A offset
  int32_t offP1[64];   // s1 * FV1 + f1 -> P1 offset
  int32_t offP2[64];   // s2 * FV2 + f2 -> P2 offset
  int64_t offC2[16];   // f2 -> C2 offset
  int32_t nq;          // 2^NI
  int32_t nrest;       // 2^(NI - NS2)
  int32_t q_of[1 << kPairMaxInner];  // (s2 index, rest index) -> q : q_of[s2 * nrest + r]
  int32_t split_u;                    // as StreamParams::split_u
  int32_t p1n, p2n;                   // small-operand entries
  int32_t pstage;                     // 1: both small operands staged in smem (p1n + p2n <= kPairStageMax)
  int32_t persist;                    // as StreamParams::persist
};
constexpr int kPairStageMax = 4096;

// ---- K3: FP64 DMMA GEMM with bit-permuted operands (dim 2) -----------------
// C[m, n] = sum_k A[m, k] B[k, n]. Tile bits (BM=2^6, BN=2^6, BK=2^4) are the
// lowest-ordered m/n/k bits; the remaining ("hi") bits index the CTA grid and
// the k loop.  Tile elements are enumerated in each operand's own address
// order (tpos ascending), so global loads/stores are coalesced for any layout.
constexpr int kGemmBits = 16;
struct TileMap {
  int32_t nbits;
  int8_t pos[kGemmBits];   // address bit of tile-element bit j (real bits ascending; -1 = virtual)
  int8_t kind[kGemmBits];  // 0: row-type bit (m or n), 1: k bit (for C: 0=m, 1=n)
  int8_t sub[kGemmBits];   // bit index inside the tile coordinate
};
// Shapes smaller than the tile use "virtual" tile bits (pos = -1): those
// elements are zero in smem and never stored, so one kernel family covers
// every m, n, k >= 0.  Split-K (splits > 1) writes per-split partial tiles to
// `ws` (in C-tile element order); k_splitk_reduce sums them in split order.
struct GemmParams {
  const double* A;
  const double* B;
  double* C;
  double* ws;
  int32_t m_hi, n_hi;  // grid bits
  int64_t k_tiles;
  int64_t k_per_split;
  int32_t splits;
  BitRuns a_m, a_k, b_n, b_k, c_m, c_n;  // hi-part deposits
  int32_t bt_bits;                       // batch variables (grid-major above the tiles)
  BitRuns a_bt, b_bt, c_bt;
  TileMap ta, tb, tc;
  int32_t grid_swizzle_log;  // group of 2^g m-tiles walked together (L2 reuse)
};

// ---- K4: tiny-subtree forest (any domain) ----------------------------------
struct TinyNode {
  const double* ga;  // global operand (leaf / forced root) or nullptr -> smem
  const double* gb;
  double* gout;      // global output (subtree root) or nullptr -> smem
  int32_t sa, sb, sout;  // smem offsets in doubles from the dynamic smem base (staged operands resolved), -1: global
  int32_t c_size, s_size;
  int32_t nc, ns;
  int32_t dig;   // first digit (nc C-digits then ns S-digits)
  int32_t pow2;  // all digits have dim 2
  int32_t sta, stb;  // staging offsets of small global operands within the batch (-1: read global)
  int32_t na, nb;    // entry counts of the staged operands
  int32_t lw;        // dim-2 nodes: 2^lw lanes share one output's sum (<= 32)
  int32_t sync;      // before this node: 1 CTA barrier, 2 warp-0 barrier (it reads / overwrites smem touched since)
  int32_t wofs;      // single-warp node: the warp that runs it (its wave's other nodes run beside it); -1: whole CTA
};
// k_tiny processes a group in batches of kTinyBatch nodes: descriptors,
// digits and small global operands (leaves) of a batch are copied to smem
// with one round of independent loads before the batch's nodes run.
constexpr int kTinyBatch = 32;
#ifndef TC_TINY_THREADS_LOG
#define TC_TINY_THREADS_LOG 8
#endif
constexpr int kTinyThreadsLog = TC_TINY_THREADS_LOG;  // k_tiny CTA = 2^8 threads
constexpr int kTinyMaxSum = 16;     // summed dim-2 digits with precomputed deltas
// k_tiny's cooperative path (CTA-wide reduce with internal barriers): mixed
// radix or very long sums with few outputs
inline bool tiny_uses_reduce(const TinyNode& t) {
  return !(t.pow2 && t.ns - t.lw <= kTinyMaxSum) && !(t.c_size * 4 >= (1 << kTinyThreadsLog) || t.s_size < 64);
}
constexpr int kTinyStageMax = 64;  // entries: larger global operands are read in place
struct TinyDigit {
  int32_t dim, sa, sb, pad;
};
struct TinyGroup {
  int32_t beg, end;
};

// ---- generic mixed-radix contraction (any domain, any size) ---------------
struct GDigit {
  int64_t dim, sa, sb;
};
struct GenericParams {
  const double* A;
  const double* B;
  double* C;
  int64_t c_size, s_size;
  int32_t nc, ns;
  const GDigit* dig;  // device array: nc C-digits (C layout order) then ns S-digits
};

// ---- K5: per-slice leaf selection ----------------------------------------
struct SelTerm {
  int64_t pv;      // place value of the sliced index in the slice id
  int64_t dim;
  int64_t stride;  // stride of that index in the leaf
};
struct SelEntry {
  int64_t dst, src;
  int32_t t0, nt;
};
struct SelectParams {
  const double* lval;
  double* out;
  const SelEntry* ent;
  const SelTerm* terms;
  int64_t n;
  const int64_t* eta;
};

struct RootCopyParams {
  const double* src;
  double* const* results;  // device slot holding the [n][R] results buffer (re-pointed by the runtime)
  const int64_t* map;  // dense entry -> physical offset or -1 (nullptr: identity)
  int64_t R;
  const int64_t* eta;  // [0] = current slice (iteration id), [1] = first lexicographic slice of the run
  const int64_t* ord;  // slice order table (nullptr: iteration id = lexicographic id), see slice_lex
};

// Slice order table: [n, then per chosen index (lexicographic position j):
// place value in the iteration id, dimension, place value in the lexicographic id]
#ifdef __CUDACC__
#define TC_HD __host__ __device__
#else
#define TC_HD
#endif
TC_HD inline int64_t slice_lex(const int64_t* ord, int64_t t) {
  if (!ord) return t;
  int64_t s = 0;
  for (int64_t j = 0; j < ord[0]; ++j) s += ((t / ord[1 + 3 * j]) % ord[2 + 3 * j]) * ord[3 + 3 * j];
  return s;
}
TC_HD inline int64_t slice_iter(const int64_t* ord, int64_t s) {
  if (!ord) return s;
  int64_t t = 0;
  for (int64_t j = 0; j < ord[0]; ++j) t += ((s / ord[3 + 3 * j]) % ord[2 + 3 * j]) * ord[1 + 3 * j];
  return t;
}

}  // namespace tc
