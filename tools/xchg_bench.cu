// Calibration: cost of one phase transition of the gate-block pass (16
// complex128 per thread, 256 threads, a 64-KiB chunk) through shared memory
// (STS.128 + bar.sync + LDS.128 + bar.sync) against warp shuffles that swap
// two register bits with two lane bits (4 x SHFL.32 per amplitude that moves).
// One CTA per SM, persistent loop; the figure is SM cycles per transition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xchg_bench tools/xchg_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256, 1) k_smem(double2* out, int rounds) {
  extern __shared__ double2 sm[];
  double2 v[16];
  const unsigned t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = make_double2(t + j, j);
  long long c0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    // write: thread bits 0..7 -> positions 0..7, registers -> 8..11 (XOR-swizzled)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const unsigned i = t | (j << 8);
      sm[i ^ ((i >> 4) & 7)] = v[j];  // conflict-free for both access patterns
    }
    __syncthreads();
    // read: registers -> positions 0..3, thread bits -> 4..11
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const unsigned i = (j | (t << 4));
      v[j] = sm[i ^ ((i >> 4) & 7)];
      v[j].x += 1e-9;
    }
    __syncthreads();
  }
  long long c1 = clock64();
  if (t == 0) out[blockIdx.x] = make_double2((double)(c1 - c0) / rounds, 0);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += v[j].x + v[j].y;
  if (s == 12345.0) out[gridDim.x + blockIdx.x] = make_double2(s, 0);
}

__device__ __forceinline__ double shfl_d(double x, int m) {
  int lo = __double2loint(x), hi = __double2hiint(x);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return __hiloint2double(hi, lo);
}

__global__ void __launch_bounds__(256, 1) k_shfl(double2* out, int rounds) {
  double2 v[16];
  const unsigned t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = make_double2(t + j, j);
  long long c0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    // swap register bits 0,1 with lane bits 3,4: amplitude j goes to lane
    // l ^ ((j&3) ^ lanebits) ... (as a butterfly: two xor stages, half of the
    // amplitudes move at each)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int m = 8 << b;  // lane bit 3 or 4
      const bool hi = (t >> (3 + b)) & 1;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (((j >> b) & 1) == 0) {
          const int k = j | (1 << b);
          // the lane with the bit set sends v[j], the other v[k]
          double2 send = hi ? v[j] : v[k];
          double2 got;
          got.x = shfl_d(send.x, m);
          got.y = shfl_d(send.y, m);
          if (hi) v[j] = got; else v[k] = got;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j].x += 1e-9;
  }
  long long c1 = clock64();
  if (t == 0) out[blockIdx.x] = make_double2((double)(c1 - c0) / rounds, 0);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += v[j].x + v[j].y;
  if (s == 12345.0) out[gridDim.x + blockIdx.x] = make_double2(s, 0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* out;
  cudaMalloc(&out, 2 * sms * sizeof(double2));
  double2 h[1];
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int rounds = 2000;
  k_smem<<<sms, 256, 64 * 1024>>>(out, rounds);
  k_smem<<<sms, 256, 64 * 1024>>>(out, rounds);
  cudaMemcpy(h, out, sizeof(double2), cudaMemcpyDeviceToHost);
  printf("smem transition (64 KiB STS + LDS, 2 barriers): %.0f cycles\n", h[0].x);
  k_shfl<<<sms, 256>>>(out, rounds);
  k_shfl<<<sms, 256>>>(out, rounds);
  cudaMemcpy(h, out, sizeof(double2), cudaMemcpyDeviceToHost);
  printf("shuffle exchange of 2 register bits with 2 lane bits (48 KiB moved): %.0f cycles\n", h[0].x);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
