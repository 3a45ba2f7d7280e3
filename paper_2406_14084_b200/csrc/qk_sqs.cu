// qk_sqs.cu — persistent bulk-copy SQS pass for sm_100a.
//
// new[i] = old[bitswap(i, A, B)] in place (simulator.py:159-176; single-device
// CSQS :179-235). Same tile-pair decomposition as k_sqs (SqsDesc: tile bits V =
// the 5 low address bits + their swap partners + fillers, outer pairs map tile
// X to tile Y = pi(X)), but the loads no longer go through registers: warp 0
// streams the 512-B runs of both tiles of a pair into a ring of shared-memory
// stages with cp.async.bulk + mbarrier complete_tx, so up to ~190 KiB per SM
// are in flight. Eight consumer warps wait on the stage, read each element's
// source through the in-tile permutation, and store whole 512-B runs with
// 128-bit st.global.cs. Runs sit at a 528-B pitch in shared memory, so both the
// run-major reads and the permuted reads are bank-conflict-free.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qk_internal.h"

namespace qk {
namespace {

constexpr int kRunBytes = 512;   // 2^5 amplitudes
constexpr int kPitch = 528;      // run pitch in shared memory (+16 B)
constexpr int kConsumerWarps = 8;
constexpr int kStageMax = 6;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "QS_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra QS_WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void st_cs(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

struct Unit {
  uint64_t X, Y;
  bool same;
};

// i-th candidate tile of this CTA -> canonical unit (X <= Y, not a no-op)?
__device__ __forceinline__ bool unit_of(const SqsDesc& S, uint64_t X, Unit* u) {
  uint64_t Y = X;
  for (int p = 0; p < S.nop; ++p) {
    const uint64_t d = ((X >> S.oa[p]) ^ (X >> S.ob[p])) & 1ull;
    Y ^= (d << S.oa[p]) | (d << S.ob[p]);
  }
  if (Y < X) return false;
  if (Y == X && S.ident) return false;
  u->X = X;
  u->Y = Y;
  u->same = (X == Y);
  return true;
}

__device__ __forceinline__ uint64_t deposit_outer(const SqsDesc& S, uint64_t X) {
  uint64_t b = 0;
  for (int k = 0; k < S.nouter; ++k) b |= ((X >> k) & 1ull) << S.opos[k];
  return b;
}

__global__ void __launch_bounds__(32 * (1 + kConsumerWarps), 1)
    k_sqs_bulk(double2* __restrict__ state, const __grid_constant__ SqsDesc S, int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int nv = S.nv, w = S.w;
  const uint32_t tile = 1u << nv;
  const int nruns = 1 << (nv - w);
  const uint32_t stage_bytes = 2u * nruns * kPitch;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  const uint64_t nunits = 1ull << S.nouter;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t G = gridDim.x;
  if (warp == 0) {
    // producer: every lane issues bulk copies of whole runs
    uint64_t k = 0;
    for (uint64_t X = blockIdx.x; X < nunits; X += G) {
      Unit u;
      if (!unit_of(S, X, &u)) continue;
      const int s = (int)(k % stages);
      const uint32_t round = (uint32_t)(k / stages);
      ++k;
      if (round > 0) mbar_wait(empty + s, (round - 1) & 1u);
      if (lane == 0) mbar_expect_tx(full + s, (u.same ? 1u : 2u) * nruns * kRunBytes);
      __syncwarp();
      const uint64_t bx = deposit_outer(S, u.X), by = deposit_outer(S, u.Y);
      uint8_t* sx = smem + (size_t)s * stage_bytes;
      uint8_t* sy = sx + (size_t)nruns * kPitch;
      for (int r = lane; r < nruns; r += 32) {
        uint64_t off = 0;
        for (int b = w; b < nv; ++b) off |= (uint64_t)((r >> (b - w)) & 1) << S.vpos[b];
        bulk_load(sx + r * kPitch, state + bx + off, kRunBytes, full + s);
        if (!u.same) bulk_load(sy + r * kPitch, state + by + off, kRunBytes, full + s);
      }
    }
    return;
  }
  // consumers
  const uint32_t ct = threadIdx.x - 32;
  const uint32_t wmask = (1u << w) - 1;
  uint64_t k = 0;
  for (uint64_t X = blockIdx.x; X < nunits; X += G) {
    Unit u;
    if (!unit_of(S, X, &u)) continue;
    const int s = (int)(k % stages);
    const uint32_t round = (uint32_t)(k / stages);
    ++k;
    const uint64_t bx = deposit_outer(S, u.X), by = deposit_outer(S, u.Y);
    const uint8_t* sx = smem + (size_t)s * stage_bytes;
    const uint8_t* sy = sx + (size_t)nruns * kPitch;
    mbar_wait(full + s, round & 1u);
    for (uint32_t e = ct; e < tile; e += 32 * kConsumerWarps) {
      uint64_t off = e & wmask;
      for (int b = w; b < nv; ++b) off |= (uint64_t)((e >> b) & 1u) << S.vpos[b];
      uint32_t pe = e;
      for (int p = 0; p < S.nvp; ++p) {
        const uint32_t d = ((pe >> S.va[p]) ^ (pe >> S.vb[p])) & 1u;
        pe ^= (d << S.va[p]) | (d << S.vb[p]);
      }
      const uint32_t so = (pe >> w) * kPitch + (pe & wmask) * 16u;
      const double2 vx = *reinterpret_cast<const double2*>(sx + so);
      if (u.same) {
        st_cs(state + bx + off, vx);
      } else {
        const double2 vy = *reinterpret_cast<const double2*>(sy + so);
        st_cs(state + bx + off, vy);
        st_cs(state + by + off, vx);
      }
    }
    // all reads of this stage are consumed (the stores depend on them): order
    // them before the next bulk copy (async proxy) and release the stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
}

}  // namespace

int launch_sqs_bulk(double* state, const SqsDesc* h, int num_sms, CUstream_st* stream) {
  if (h->w != 5 || h->nv < 5 || h->nv - h->w > 5) return -2;  // not covered: caller falls back
  const int nruns = 1 << (h->nv - h->w);
  const size_t stage_bytes = 2ull * nruns * kPitch;
  int stages = (int)((200 * 1024) / stage_bytes);
  if (stages > kStageMax) stages = kStageMax;
  if (stages < 2) return -2;
  const size_t smem = stages * stage_bytes + 2 * stages * 8;
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) cudaFuncSetAttribute(k_sqs_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const uint64_t units = 1ull << h->nouter;
  const uint64_t grid = units < (uint64_t)num_sms ? units : (uint64_t)num_sms;
  k_sqs_bulk<<<(unsigned)grid, 32 * (1 + kConsumerWarps), smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(state), *h, stages);
  return (int)cudaGetLastError();
}

}  // namespace qk
