// Stream-step access-pattern probe: C[x, f] = sum_s A[x | s<<sb] P[s, f] over
// 2^n x values (the k_stream<1,1> shape with x bit 0 at address bit 0 of A and C,
// the common case in C4).  Variants:
//   0  scalar: x = chunk*1024 + u*256 + tid, 4 x per thread per chunk (today's k_stream)
//   1  vec2:   a thread owns 2 adjacent x (one 16-B load per s, one 16-B store per f)
//   2  vec2 + the next chunk's loads issued before this chunk's FMAs / stores
//   3  plain double2 copy of the same bytes (read |A|, write |C|) for reference
// grid-stride over chunks with `ctas` CTAs per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sp tools/micro/stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

__constant__ double cP[4];

__device__ __forceinline__ int64_t spread(int64_t x, int sb) {  // insert a 0 at bit sb
  const int64_t lo = x & ((1ll << sb) - 1);
  return ((x >> sb) << (sb + 1)) | lo;
}

template <int V>
__global__ void __launch_bounds__(256, 6) k_probe(const double* __restrict__ A, double* __restrict__ C, int n, int sb) {
  const int64_t nch = (int64_t)1 << (n - 10);
  const int tid = threadIdx.x;
  const int64_t S = (int64_t)1 << sb;
  if (V == 0) {
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
      double a[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t x = (c << 10) + u * 256 + tid;
        const int64_t ad = spread(x, sb);
        a[u][0] = __ldg(A + ad);
        a[u][1] = __ldg(A + ad + S);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t x = (c << 10) + u * 256 + tid;
        const int64_t ad = spread(x, sb);
#pragma unroll
        for (int f = 0; f < 2; ++f) C[ad + f * S] = fma(a[u][1], cP[2 + f], a[u][0] * cP[f]);
      }
    }
  } else if (V == 1 || V == 2) {
    // thread owns x pairs (2*tid, 2*tid+1) + w*512, w = 0, 1
    double2 a[2][2], nx[2][2];
    auto load = [&](int64_t c, double2 (&r)[2][2]) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int64_t x = (c << 10) + w * 512 + 2 * tid;
        const int64_t ad = spread(x, sb);
        r[w][0] = __ldg(reinterpret_cast<const double2*>(A + ad));
        r[w][1] = __ldg(reinterpret_cast<const double2*>(A + ad + S));
      }
    };
    int64_t c = blockIdx.x;
    if (c >= nch) return;
    load(c, a);
    for (; c < nch; c += gridDim.x) {
      const int64_t cn = c + gridDim.x;
      if (V == 2 && cn < nch) load(cn, nx);
      if (V == 1 && c != blockIdx.x) load(c, a);
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int64_t x = (c << 10) + w * 512 + 2 * tid;
        const int64_t ad = spread(x, sb);
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          double2 o;
          o.x = fma(a[w][1].x, cP[2 + f], a[w][0].x * cP[f]);
          o.y = fma(a[w][1].y, cP[2 + f], a[w][0].y * cP[f]);
          *reinterpret_cast<double2*>(C + ad + f * S) = o;
        }
      }
      if (V == 2) {
#pragma unroll
        for (int w = 0; w < 2; ++w) a[w][0] = nx[w][0], a[w][1] = nx[w][1];
      }
    }
  } else {
    const int64_t n2 = ((int64_t)1 << (n + 1)) / 2;
    const double2* A2 = reinterpret_cast<const double2*>(A);
    double2* C2 = reinterpret_cast<double2*>(C);
    for (int64_t i = (int64_t)blockIdx.x * 256 + tid; i < n2; i += (int64_t)gridDim.x * 256) C2[i] = __ldg(A2 + i);
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 26;  // x bits: |A| = |C| = 2^(n+1) doubles
  const int sb = argc > 2 ? std::atoi(argv[2]) : 5;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = sizeof(double) << (n + 1);
  double *A, *C, *F;
  CK(cudaMalloc(&A, bytes));
  CK(cudaMalloc(&C, bytes));
  const size_t fl = (size_t)512 << 20;
  CK(cudaMalloc(&F, fl));
  CK(cudaMemset(A, 0, bytes));
  double hp[4] = {0.5, 0.25, 0.125, 2.0};
  CK(cudaMemcpyToSymbol(cP, hp, sizeof(hp)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int v = 0; v < 4; ++v) {
    for (int ctas : {4, 6, 8, 16, 32}) {
      const int64_t nch = (int64_t)1 << (n - 10);
      int grid = (int)std::min<int64_t>((int64_t)sms * ctas, nch);
      float best = 1e30f;
      for (int r = 0; r < 8; ++r) {
        CK(cudaMemset(F, r, fl));  // flush L2
        CK(cudaEventRecord(e0));
        switch (v) {
          case 0: k_probe<0><<<grid, 256>>>(A, C, n, sb); break;
          case 1: k_probe<1><<<grid, 256>>>(A, C, n, sb); break;
          case 2: k_probe<2><<<grid, 256>>>(A, C, n, sb); break;
          default: k_probe<3><<<grid, 256>>>(A, C, n, sb); break;
        }
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      std::printf("n=%d sb=%d variant %d ctas/SM %2d: %8.2f us  %7.1f GB/s\n", n, sb, v, ctas, best * 1e3,
                  2.0 * bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
