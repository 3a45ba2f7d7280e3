// Calibration: HBM efficiency of an in-place read+write sweep over 2^30
// complex128 amplitudes when each 4096-amplitude unit ("tile") is made of rows
// of 2^rb amplitudes placed at address bits [p, p + 12 - rb), i.e. the access
// pattern of a strided-tile gate-block pass. Plain LDG/STG, 256 threads per
// tile, 16 amplitudes per thread, many CTAs per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sb tools/strided_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

// tile t, element e (0..4095) -> address: e's low rb bits are the row bits
// (address bits 0..rb-1), e's high 12-rb bits go to address bits p.., the
// tile index fills the remaining bits in ascending order
__device__ __forceinline__ uint64_t addr(uint64_t t, uint32_t e, int rb, int p) {
  const uint64_t lo = e & ((1u << rb) - 1);
  const uint64_t hi = e >> rb;
  const int nh = 12 - rb;
  // tile bits: [rb, p) then [p + nh, 30)
  const int nlow = p - rb;
  const uint64_t tlo = t & ((1ull << nlow) - 1), thi = t >> nlow;
  return lo | (tlo << rb) | (hi << p) | (thi << (p + nh));
}

__global__ void __launch_bounds__(256) k_tile(double2* __restrict__ a, uint64_t ntiles, int rb, int p, double s) {
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = a[addr(t, threadIdx.x + 256 * j, rb, p)];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j].x *= s;
      a[addr(t, threadIdx.x + 256 * j, rb, p)] = v[j];
    }
  }
}

// clusters of K CTAs take K consecutive tiles (adjacent 128-B rows) and
// synchronise once per tile, so their requests to one DRAM row arrive together
template <int K>
__global__ void __cluster_dims__(K, 1, 1) __launch_bounds__(256) k_tile_cl(double2* __restrict__ a, uint64_t ntiles, int rb, int p, double s) {
  unsigned r, nc, cid;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(nc));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  for (uint64_t u = cid; u * K < ntiles; u += nc) {
    const uint64_t t = u * K + r;
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = a[addr(t, threadIdx.x + 256 * j, rb, p)];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j].x *= s;
      a[addr(t, threadIdx.x + 256 * j, rb, p)] = v[j];
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
  const int rbs[] = {3, 4, 12};
  const int ps[] = {12, 21};
  for (int rb : rbs)
    for (int p : ps) {
      if (rb == 12 && p != 12) continue;
      int pp = rb == 12 ? 12 : p;
      for (int per : {4, 8}) {
        const int grid = sms * per;
        k_tile<<<grid, 256>>>(a, n >> 12, rb, pp, 1.0);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k_tile<<<grid, 256>>>(a, n >> 12, rb, pp, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        printf("rows %4d B  high bits at %2d  ctas/sm %d : %.3f ms  %.0f GB/s\n", 16 << rb, pp, per, ms,
               2.0 * n * 16 / (ms * 1e6));
      }
    }
  for (int p : {12, 21})
    for (int K : {2, 4})
      for (int per : {4, 8}) {
        const int grid = sms * per;
        auto run = [&]() {
          if (K == 2) k_tile_cl<2><<<grid, 256>>>(a, n >> 12, 3, p, 1.0);
          else k_tile_cl<4><<<grid, 256>>>(a, n >> 12, 3, p, 1.0);
        };
        run();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        printf("rows 128 B  high bits at %2d  cluster %d ctas/sm %d : %.3f ms  %.0f GB/s\n", p, K, per, ms,
               2.0 * n * 16 / (ms * 1e6));
      }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
