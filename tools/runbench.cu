// Calibration: HBM throughput of a 2^12 x 2^12 transpose (the k=12 SQS of
// QAOA c12) done with short runs on one side. A tile is 2^s rows (p_lo) x TQ
// amplitudes (q); the "read-long" variant reads 2^s runs of TQ amplitudes and
// writes TQ runs of 2^s amplitudes (what a block pass holding 2^s chunks
// would store), "write-long" is the dual. Tile order: p_hi fastest (adjacent
// CTAs touch adjacent short runs) or q fastest.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o runbench tools/runbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>


template <int S, bool READ_LONG, int ORDER, int TQ = (2048 >> S)>
__global__ void __launch_bounds__(256) k_tr(const double2* __restrict__ src, double2* __restrict__ dst, int nbits) {
  __shared__ double2 sm[(1 << S) * TQ];
  const uint64_t nrest = 1ull << (nbits - 24);
  const uint64_t nph = 1ull << (12 - S);
  const uint64_t nqb = 4096 / TQ;
  const uint64_t ntiles = nrest * nph * nqb;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint64_t ph, qb, rest;
    if (ORDER == 0) {
      ph = t % nph; qb = (t / nph) % nqb; rest = t / (nph * nqb);
    } else {
      qb = t % nqb; ph = (t / nqb) % nph; rest = t / (nph * nqb);
    }
    const uint64_t base = rest << 24;
    // element (r, c): p = ph<<S | r, q = qb*TQ + c; src = base | p<<12 | q; dst = base | q<<12 | p
    constexpr int R = 1 << S;
    constexpr int N = R * TQ;
    if (READ_LONG) {
      for (int e = threadIdx.x; e < N; e += 256) {
        const int r = e / TQ, c = e % TQ;
        sm[r * TQ + (c ^ (r & 7))] = src[base | ((ph << S | r) << 12) | (qb * TQ + c)];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < N; e += 256) {
        const int c = e / R, r = e % R;
        __stcs(dst + (base | ((qb * TQ + c) << 12) | (ph << S | r)), sm[r * TQ + (c ^ (r & 7))]);
      }
      __syncthreads();
    } else {
      // dual: src rows are q (short runs of R along p), dst rows are p (long runs along q)
      for (int e = threadIdx.x; e < N; e += 256) {
        const int c = e / R, r = e % R;
        sm[r * TQ + (c ^ (r & 7))] = src[base | ((qb * TQ + c) << 12) | (ph << S | r)];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < N; e += 256) {
        const int r = e / TQ, c = e % TQ;
        __stcs(dst + (base | ((ph << S | r) << 12) | (qb * TQ + c)), sm[r * TQ + (c ^ (r & 7))]);
      }
      __syncthreads();
    }
  }
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, uint64_t n) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) __stcs(b + i, a[i]);
}

template <int S, bool RL, int ORD>
void run(const double2* a, double2* b, int nbits, int grid) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tr<S, RL, ORD><<<grid, 256>>>(a, b, nbits);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_tr<S, RL, ORD><<<grid, 256>>>(a, b, nbits);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("s=%d run=%4d B %s order=%s grid=%d: %.0f GB/s\n", S, 16 << S, RL ? "short-writes" : "short-reads ",
         ORD ? "q-fast " : "ph-fast", grid, 3 * 32.0 * (double)(1ull << nbits) / (ms * 1e-3) / 1e9);
}

int main() {
  const int nbits = 30;
  const uint64_t n = 1ull << nbits;
  double2 *a, *b;
  if (cudaMalloc(&a, n * 16) || cudaMalloc(&b, n * 16)) return 1;
  cudaMemset(a, 0, n * 16);
  cudaMemset(b, 0, n * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  k_copy<<<148 * 8, 256>>>(a, b, n);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_copy<<<148 * 8, 256>>>(a, b, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.0f GB/s\n", 3 * 32.0 * n / (ms * 1e-3) / 1e9);
  for (int g : {148 * 4, 148 * 8}) {
    run<2, true, 0>(a, b, nbits, g);
    run<3, true, 0>(a, b, nbits, g);
    run<3, true, 1>(a, b, nbits, g);
    run<3, false, 0>(a, b, nbits, g);
    run<4, true, 0>(a, b, nbits, g);
    run<4, true, 1>(a, b, nbits, g);
    run<4, false, 0>(a, b, nbits, g);
    run<5, true, 0>(a, b, nbits, g);
    run<5, false, 0>(a, b, nbits, g);
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
