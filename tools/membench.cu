// Calibration: achievable HBM bandwidth for the access patterns of the AIC path
// (in-place read+write sweep vs out-of-place copy), 16 GiB complex128.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, uint64_t n) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
    b[i] = x0; b[i + stride] = x1; b[i + 2 * stride] = x2; b[i + 3 * stride] = x3;
  }
  for (; i < n; i += stride) b[i] = a[i];
}

__global__ void k_inplace(double2* __restrict__ a, uint64_t n, double s) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
    x0.x *= s; x1.x *= s; x2.x *= s; x3.x *= s;
    a[i] = x0; a[i + stride] = x1; a[i + 2 * stride] = x2; a[i + 3 * stride] = x3;
  }
}

// chunked in-place: each CTA owns contiguous 64 KiB chunks (like a gate-block pass)
__global__ void __launch_bounds__(256) k_inplace_chunk(double2* __restrict__ a, uint64_t nchunks, double s) {
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    double2* p = a + (c << 12);
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = p[threadIdx.x + 256 * j];
#pragma unroll
    for (int j = 0; j < 16; ++j) { v[j].x *= s; p[threadIdx.x + 256 * j] = v[j]; }
  }
}

int main() {
  const uint64_t n = 1ull << 30;  // 16 GiB
  double2 *a, *b;
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16 / 2);
  cudaMemset(a, 0, n * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int blocksPerSm : {4, 8, 16}) {
    const int grid = 148 * blocksPerSm;
    for (int r = 0; r < 2; ++r) k_copy<<<grid, 256>>>(a, b, n / 2);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_copy<<<grid, 256>>>(a, b, n / 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy      grid=%5d  %.0f GB/s\n", grid, 5 * (n / 2) * 32.0 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_inplace<<<grid, 256>>>(a, n, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("inplace   grid=%5d  %.0f GB/s\n", grid, 5 * n * 32.0 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_inplace_chunk<<<grid, 256>>>(a, n >> 12, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("chunk64K  grid=%5d  %.0f GB/s\n", grid, 5 * n * 32.0 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
