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

// ---- K2: big x small streaming contraction (dim 2) ------------------------
// C[x, f] = sum_s A[x, s] * P[s, f]; x enumerates the kept indices of the big
// operand A, s the shared ones (<= 2^4), f the small operand's free ones (<= 2^4).
struct StreamParams {
  const double* A;
  const double* P;
  double* C;
  int64_t nx;
  BitRuns xa, xc;
  int64_t offA[16];  // s -> offset in A
  int64_t offC[16];  // f -> offset in C
  int32_t offP[64];  // s * 2^NF + f -> offset in P
};

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
  TileMap ta, tb, tc;
  int32_t grid_swizzle_log;  // group of 2^g m-tiles walked together (L2 reuse)
};

// ---- K2c: fused chain of big x small contractions (dim 2) -----------------
// A chain v1..vk (v_{i+1}'s big operand is v_i) runs as ONE pass: a CTA loads
// a tile = (x_lo outer bits) x (all "inner" bits the chain touches) of the
// input, applies the k small operands in shared memory, stores the tile of
// v_k.  Intermediates v_1..v_{k-1} never touch HBM.
constexpr int kChainU = 6;       // max inner bits alive at any step (x_lo >= 6 bits)
constexpr int kChainMax = 16;    // max steps per fused segment
constexpr int kChainBuf = 4096;  // doubles per smem tile buffer (x_lo * 2^inner)
struct ChainStep {
  const double* P;         // small operand
  int32_t offP[64];        // s * 2^nf + f -> offset in P
  uint16_t utab[1 << kChainU];  // new inner u -> (cur inner base | f << 8)
  uint8_t stab[16];        // s -> cur inner bits of the shared indices
  int32_t ns, nf, nnew, pad;
};
struct ChainParams {
  const double* A;
  double* C;
  const ChainStep* steps;
  int32_t nsteps;
  int32_t xt;  // x_lo bits
  int64_t n_tiles;
  BitRuns a_hi, c_hi;  // x_hi -> offsets
  TileMap ta, tc;      // (x_lo kind 0, inner kind 1) in A / C address order
};

// ---- K4: tiny-subtree forest (any domain) ----------------------------------
struct TinyNode {
  const double* ga;  // global operand (leaf / forced root) or nullptr -> smem
  const double* gb;
  double* gout;      // global output (subtree root) or nullptr -> smem
  int32_t sa, sb, sout;  // smem offsets in doubles
  int32_t c_size, s_size;
  int32_t nc, ns;
  int32_t dig;   // first digit (nc C-digits then ns S-digits)
  int32_t pow2;  // all digits have dim 2
  int32_t pad;
};
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
  double* results;
  int64_t R;
  const int64_t* eta;  // [0] = current slice, [1] = first slice of the run
};

}  // namespace tc
