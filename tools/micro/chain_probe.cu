// Dependent-step chain probe: N streaming steps (B[x] = 0.5 A[x] + 0.25 A[x^1],
// ping-pong buffers of S bytes each) run as
//   G: N kernel launches captured in one CUDA graph (today's C2 chain), or
//   P: one persistent launch (all CTAs resident) with a grid barrier between steps.
// Reports us per step for several S.  Decides whether a persistent chain
// executor can beat graph-launched steps on C2-sized (1-64 MB) tensors.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/micro/chain_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);          \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

__device__ __forceinline__ void step_body(const double* __restrict__ A, double* __restrict__ B, long n, long i0,
                                          long stride) {
  for (long i = i0; i < n; i += stride) B[i] = fma(0.25, A[i ^ 1], 0.5 * A[i]);
}

__global__ void __launch_bounds__(256) k_step(const double* A, double* B, long n) {
  step_body(A, B, n, (long)blockIdx.x * blockDim.x + threadIdx.x, (long)gridDim.x * blockDim.x);
}

// the same step with a 2.5 KB parameter block read with dynamic indices
// (like k_stream's per-bit address tables): every entry is 0
struct BigParams {
  long long t[320];
};
__global__ void __launch_bounds__(256) k_step_big(const double* A, double* B, long n, const BigParams p) {
  long long off = 0;
#pragma unroll
  for (int j = 0; j < 10; ++j)
    if ((threadIdx.x >> (j & 7)) & 1) off += p.t[j * 32 + (blockIdx.x & 31)];
  step_body(A, B, n, (long)blockIdx.x * blockDim.x + threadIdx.x + off, (long)gridDim.x * blockDim.x);
}

__device__ unsigned g_count = 0;
__device__ volatile unsigned g_gen = 0;

__device__ __forceinline__ void grid_barrier(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = gen + 1;
    } else {
      while (g_gen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_chain(double* A, double* B, long n, int steps) {
  for (int s = 0; s < steps; ++s) {
    const double* src = (s & 1) ? B : A;
    double* dst = (s & 1) ? A : B;
    step_body(src, dst, n, (long)blockIdx.x * blockDim.x + threadIdx.x, (long)gridDim.x * blockDim.x);
    grid_barrier(gridDim.x);
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chain, 256, 0));
  const int N = 100;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (long mb : {1L, 4L, 16L, 64L}) {
    const long n = mb * (1L << 20) / 8;
    double *A, *B;
    CK(cudaMalloc(&A, n * 8));
    CK(cudaMalloc(&B, n * 8));
    CK(cudaMemset(A, 0, n * 8));
    CK(cudaMemset(B, 0, n * 8));
    for (int per_sm : {1, 2, 4}) {
      // graph of N launches
      const int grid = (int)std::min<long>((long)sms * per_sm * 2, (n + 255) / 256);
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
      for (int s = 0; s < N; ++s) k_step<<<grid, 256, 0, st>>>((s & 1) ? B : A, (s & 1) ? A : B, n);
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      float best_g = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best_g = std::min(best_g, ms);
      }
      // the same graph with the big parameter block
      BigParams bp{};
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
      for (int s = 0; s < N; ++s) k_step_big<<<grid, 256, 0, st>>>((s & 1) ? B : A, (s & 1) ? A : B, n, bp);
      cudaGraph_t g2;
      cudaGraphExec_t ge2;
      CK(cudaStreamEndCapture(st, &g2));
      CK(cudaGraphInstantiate(&ge2, g2, 0));
      float best_b = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge2, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best_b = std::min(best_b, ms);
      }
      std::printf("S=%3ld MB  graph+2.5KB params grid %5d: %7.2f us/step\n", mb, grid, best_b * 1e3 / N);
      CK(cudaGraphExecDestroy(ge2));
      CK(cudaGraphDestroy(g2));
      // persistent chain (all CTAs resident)
      const int pgrid = std::min(sms * std::min(per_sm, occ), (int)((n + 255) / 256));
      float best_p = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0, st));
        k_chain<<<pgrid, 256, 0, st>>>(A, B, n, N);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best_p = std::min(best_p, ms);
      }
      std::printf("S=%3ld MB  graph grid %5d: %7.2f us/step   persistent grid %5d: %7.2f us/step  (%.1f / %.1f GB/s)\n",
                  mb, grid, best_g * 1e3 / N, pgrid, best_p * 1e3 / N, 2.0 * n * 8 / (best_g * 1e-3 / N) / 1e9,
                  2.0 * n * 8 / (best_p * 1e-3 / N) / 1e9);
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(g));
    }
    CK(cudaFree(A));
    CK(cudaFree(B));
  }
  return 0;
}
