// Calibration: HBM efficiency of an in-place read+write sweep over 2^30
// complex128 amplitudes when each unit ("tile") of 2^(rb+nh) amplitudes is
// made of rows of 2^rb amplitudes (address bits 0..rb-1) whose nh row-index
// bits sit at address bits [p, p + nh): the access pattern of a strided-tile
// gate-block pass. Plain LDG/STG, 256 threads per tile, 16 amplitudes per
// thread per step. Clusters of K CTAs take K consecutive tiles (adjacent rows)
// and synchronise once per tile, so their requests to one DRAM page arrive
// together.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/strided_bench tools/strided_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t addr(uint64_t t, uint32_t e, int rb, int nh, int p) {
  const uint64_t lo = e & ((1u << rb) - 1);
  const uint64_t hi = e >> rb;
  const int nlow = p - rb;  // tile bits: [rb, p) then [p + nh, 30)
  const uint64_t tlo = t & ((1ull << nlow) - 1), thi = t >> nlow;
  return lo | (tlo << rb) | (hi << p) | (thi << (p + nh));
}

template <int K>
__global__ void __launch_bounds__(256) k_tile(double2* __restrict__ a, uint64_t ntiles, int rb, int nh, int p) {
  unsigned r = 0, nc = gridDim.x, cid = blockIdx.x;
  if (K > 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(nc));
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  }
  const uint32_t steps = 1u << (rb + nh - 12);
  for (uint64_t u = cid; u * K < ntiles; u += nc) {
    const uint64_t t = u * K + r;
    if (K > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    for (uint32_t st = 0; st < steps; ++st) {
      double2 v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = a[addr(t, st * 4096 + threadIdx.x + 256 * j, rb, nh, p)];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j].x *= 1.0000001;
        a[addr(t, st * 4096 + threadIdx.x + 256 * j, rb, nh, p)] = v[j];
      }
    }
  }
}

int main() {
  const uint64_t n = 1ull << 30;
  double2* a;
  if (cudaMalloc(&a, n * 16)) return 1;
  cudaMemset(a, 0, n * 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int rb, nh, p, K; };
  const Cfg cfgs[] = {{12, 0, 12, 1}, {3, 9, 12, 1}, {3, 9, 12, 2}, {3, 9, 15, 1}, {3, 9, 15, 2}, {3, 9, 18, 1},
                      {3, 9, 18, 2}, {3, 9, 21, 1}, {3, 9, 21, 2}, {3, 9, 21, 4}, {4, 8, 21, 1}, {4, 9, 21, 1},
                      {4, 9, 12, 1}, {3, 8, 21, 1}, {3, 8, 22, 1}, {5, 9, 21, 1}};
  for (const Cfg& c : cfgs) {
    const uint64_t ntiles = n >> (c.rb + c.nh);
    auto run = [&]() {
      const int grid = sms * 8;
      if (c.K == 1) k_tile<1><<<grid, 256>>>(a, ntiles, c.rb, c.nh, c.p);
      else if (c.K == 2) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_tile<2>, a, ntiles, c.rb, c.nh, c.p);
      } else {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_tile<4>, a, ntiles, c.rb, c.nh, c.p);
      }
    };
    run();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    int pagebits = 0;
    for (int b = c.p; b < c.p + c.nh; ++b) pagebits += b >= 17;
    printf("rows %5d B  row bits %d..%d  pages/tile %4d  cluster %d : %.3f ms  %.0f GB/s\n", 16 << c.rb, c.p,
           c.p + c.nh - 1, 1 << pagebits, c.K, ms, 2.0 * n * 16 / (ms * 1e6));
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
