// qk_tma.cu — persistent, warp-specialised gate-block pass for sm_100a.
//
// One CTA per SM. Warp 0 (one elected lane) is the TMA producer: it streams
// 2^C-amplitude chunks of the HBM state into a ring of shared-memory stages
// with cp.async.bulk.tensor (SWIZZLE_128B tensor map, mbarrier complete_tx).
// The remaining 256 threads form NG consumer groups of 2^(C-4) threads; a
// group owns every NG-th chunk, waits on the stage's `full` mbarrier, runs the
// pass's register-tiled phases in place in shared memory (16 amplitudes per
// thread, one named barrier per phase), fences the generic->async proxy and
// writes the chunk back with a TMA bulk store, then releases the stage through
// its `empty` mbarrier once the store has read it. Loads of later chunks
// overlap the compute and the stores of earlier ones. Same op semantics as
// k_block_pass (simulator.py:338-357 per chunk).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qk_internal.h"

namespace qk {
namespace {

constexpr int kConsumers4 = 256;   // M = 4: 16 amplitudes per thread
constexpr int kConsumers3 = 512;   // M = 3: 8 amplitudes per thread
constexpr uint32_t kSmemBudget = 200 * 1024;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "QK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra QK_WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void st_g_cs(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TMA SWIZZLE_128B: 16-B slot bits [4:6] ^= bits [7:9] of the byte offset
__device__ __forceinline__ uint32_t swz128(uint32_t i) { return i ^ ((i >> 3) & 7u); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// in-place butterfly (a, b) -> (a + b, a - b) computed as s = a + b,
// d = s - 2b (one FMA): no temporaries, so no register moves
template <int M, int R>
__device__ __forceinline__ void h_slot(double2 (&v)[1 << M]) {
  constexpr int NA = 1 << M;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if (j & (1 << R)) continue;
    double2& a = v[j];
    double2& b = v[j | (1 << R)];
    a.x += b.x;
    a.y += b.y;
    b.x = fma(-2.0, b.x, a.x);
    b.y = fma(-2.0, b.y, a.y);
  }
}
template <int M, int R>
__device__ __forceinline__ void x_slot(double2 (&v)[1 << M]) {
  constexpr int NA = 1 << M;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if (j & (1 << R)) continue;
    const double2 a = v[j];
    v[j] = v[j | (1 << R)];
    v[j | (1 << R)] = a;
  }
}
template <int M, int R>
__device__ __forceinline__ void mat_slot(double2 (&v)[1 << M], const double* m) {
  constexpr int NA = 1 << M;
  const double m00r = m[0], m00i = m[1], m01r = m[2], m01i = m[3];
  const double m10r = m[4], m10i = m[5], m11r = m[6], m11i = m[7];
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if (j & (1 << R)) continue;
    const double2 a = v[j], b = v[j | (1 << R)];
    double2 n0, n1;
    n0.x = fma(m00r, a.x, fma(-m00i, a.y, fma(m01r, b.x, -m01i * b.y)));
    n0.y = fma(m00r, a.y, fma(m00i, a.x, fma(m01r, b.y, m01i * b.x)));
    n1.x = fma(m10r, a.x, fma(-m10i, a.y, fma(m11r, b.x, -m11i * b.y)));
    n1.y = fma(m10r, a.y, fma(m10i, a.x, fma(m11r, b.y, m11i * b.x)));
    v[j] = n0;
    v[j | (1 << R)] = n1;
  }
}
template <int M, int R>
__device__ __forceinline__ void cx_slot(double2 (&v)[1 << M], int creg, int rc, int tcond) {
  constexpr int NA = 1 << M;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if (j & (1 << R)) continue;
    const int cond = creg ? ((j >> rc) & 1) : tcond;
    const double2 a = v[j], b = v[j | (1 << R)];
    v[j] = cond ? b : a;
    v[j | (1 << R)] = cond ? a : b;
  }
}
template <int M, int A, int B>
__device__ __forceinline__ void swap_slots(double2 (&v)[1 << M]) {
  constexpr int NA = 1 << M;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    if (!((j >> A) & 1) || ((j >> B) & 1)) continue;
    const int k = j ^ (1 << A) ^ (1 << B);
    const double2 t = v[j];
    v[j] = v[k];
    v[k] = t;
  }
}

#define QK_SLOT4(FN, r, ...)                                       \
  switch (r) {                                                     \
    case 0: FN<M, 0>(__VA_ARGS__); break;                          \
    case 1: FN<M, 1>(__VA_ARGS__); break;                          \
    case 2: FN<M, 2>(__VA_ARGS__); break;                          \
    default: if constexpr (M > 3) FN<M, 3>(__VA_ARGS__); break;    \
  }

template <int M, int S>
__device__ __forceinline__ void slot_1q(double2 (&v)[1 << M], const TOp& op, const double* coef) {
  if constexpr (S < M) {
    const int k = op.st[S];
    if (k == 1) {
      h_slot<M, S>(v);
    } else if (k == 3) {
      mat_slot<M, S>(v, coef + op.cf[S]);
    } else if (k == 2) {
      x_slot<M, S>(v);
    }
  }
}

template <int M>
__device__ __forceinline__ void apply_ops(double2 (&v)[1 << M], const TmaParams& p, const TPhase& D, uint32_t tid,
                                          int T, uint32_t loct) {
  constexpr int NA = 1 << M;
  for (int o = D.op_begin; o < D.op_end; ++o) {
    const TOp& op = p.ops[o];
    const int code = op.code;
    if (code == STEP_1Q) {
      slot_1q<M, 0>(v, op, p.coef);
      slot_1q<M, 1>(v, op, p.coef);
      slot_1q<M, 2>(v, op, p.coef);
      slot_1q<M, 3>(v, op, p.coef);
    } else if (code == OP_DIAG) {
      uint32_t pt = 0;
      for (int k = 0; k < T; ++k)
        if ((tid >> k) & 1u) pt |= op.tcontrib[k];
      const double2* tab = reinterpret_cast<const double2*>(p.tabs) + op.table;
#pragma unroll
      for (int j = 0; j < NA; ++j) v[j] = cmul(v[j], __ldg(tab + (pt | op.pr[j])));
    } else if (code == OP_CX) {
      const int creg = op.creg;
      const int tcond = creg ? 0 : (int)((loct >> op.ctrl) & 1u);
      QK_SLOT4(cx_slot, op.r0, v, creg, (int)op.r1, tcond)
    } else if (code == OP_SWAP) {
      switch (op.r0 * 4 + op.r1) {
        case 1: swap_slots<M, 0, 1>(v); break;
        case 2: swap_slots<M, 0, 2>(v); break;
        case 6: swap_slots<M, 1, 2>(v); break;
        case 3: if constexpr (M > 3) swap_slots<M, 0, 3>(v); break;
        case 7: if constexpr (M > 3) swap_slots<M, 1, 3>(v); break;
        default: if constexpr (M > 3) swap_slots<M, 2, 3>(v); break;
      }
    } else if (code == OP_SCALE) {
      const double sr = p.coef[op.coef], si = p.coef[op.coef + 1];
#pragma unroll
      for (int j = 0; j < NA; ++j)
        v[j] = make_double2(fma(v[j].x, sr, -v[j].y * si), fma(v[j].x, si, v[j].y * sr));
    }
  }
}

template <int M, int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, 1) k_block_tma(const __grid_constant__ TmaParams p) {
  constexpr int NA = 1 << M;
  // dynamic shared memory starts 1024-B aligned (no static smem in this kernel)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw;
  const int C = p.C;
  const int T = C - M;
  const int GT = 1 << T;
  const int NG = p.ng;
  const int S = p.stages;
  const uint32_t stage_bytes = 16u << C;
  const uint32_t box_bytes = (uint32_t)p.box_rows * 128u;
  const int rows_chunk = 1 << (C - 3);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t G = gridDim.x;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.map) : "memory");
      for (uint64_t i = 0;; ++i) {
        const uint64_t chunk = blockIdx.x + i * G;
        if (chunk >= p.nchunks) break;
        const int s = (int)(i % S);
        const uint32_t round = (uint32_t)(i / S);
        if (round > 0) mbar_wait(empty + s, (round - 1) & 1u);
        mbar_expect_tx(full + s, stage_bytes);
        uint8_t* dst = base + (size_t)s * stage_bytes;
        const int row0 = (int)(chunk * rows_chunk);
        for (int t = 0; t < p.ntma; ++t) tma_load(dst + t * box_bytes, &p.map, 0, row0 + t * p.box_rows, full + s);
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  const int g = ct >> T;
  if (g >= NG) return;
  const uint32_t tid = ct & (GT - 1);
  const int bar_id = 1 + g;
  double2 v[NA];
  for (uint64_t i = g;; i += NG) {
    const uint64_t chunk = blockIdx.x + i * G;
    if (chunk >= p.nchunks) break;
    const int s = (int)(i % S);
    const uint32_t round = (uint32_t)(i / S);
    double2* sm = reinterpret_cast<double2*>(base + (size_t)s * stage_bytes);
    mbar_wait(full + s, round & 1u);
    const int last = p.nphases - 1;
    for (int ph = 0; ph <= last; ++ph) {
      const TPhase& D = p.ph[ph];
      uint32_t loct = 0;
      for (int k = 0; k < T; ++k)
        if ((tid >> k) & 1u) loct |= 1u << D.tpos[k];
#pragma unroll
      for (int j = 0; j < NA; ++j) v[j] = sm[swz128(loct | D.rloc[j])];
      if (ph == last && p.direct_store) {
        // compute first: consuming the loaded registers guarantees every shared
        // load has returned; then order them before the next TMA (async proxy)
        // write into this stage, and release it before the global stores
        apply_ops<M>(v, p, D, tid, T, loct);
        fence_async_smem();
        group_bar(bar_id, GT);
        if (tid == 0) mbar_arrive(empty + s);
        if (p.permuted) {
          // fused SQS: amplitude with source index o goes to pi(o), a bit permutation
          uint64_t dst = 0;
          const int nout = p.nbits - C;
          for (int k = 0; k < nout; ++k) dst |= ((chunk >> k) & 1ull) << p.dpos[C + k];
          for (int k = 0; k < T; ++k)
            if ((tid >> k) & 1u) dst |= p.ldst_t[k];
          double2* g = reinterpret_cast<double2*>(p.out) + dst;
#pragma unroll
          for (int j = 0; j < NA; ++j) st_g_cs(g + p.ldst_r[j], v[j]);
        } else {
          double2* g = reinterpret_cast<double2*>(p.out) + (chunk << C);
#pragma unroll
          for (int j = 0; j < NA; ++j) st_g_cs(g + (loct | D.rloc[j]), v[j]);
        }
        break;
      }
      apply_ops<M>(v, p, D, tid, T, loct);
#pragma unroll
      for (int j = 0; j < NA; ++j) sm[swz128(loct | D.rloc[j])] = v[j];
      if (ph < last) group_bar(bar_id, GT);
    }
    if (p.direct_store) continue;
    fence_async_smem();
    group_bar(bar_id, GT);
    if (tid == 0) {
      const int row0 = (int)(chunk * rows_chunk);
      for (int t = 0; t < p.ntma; ++t)
        tma_store(&p.map, 0, row0 + t * p.box_rows, reinterpret_cast<uint8_t*>(sm) + t * box_bytes);
      bulk_commit();
      bulk_wait_read0();
      mbar_arrive(empty + s);
    }
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace

static int consumers_for(int C, int M) {
  if (M == 5) return 2 << (C - 5);  // two groups (specialised kernels only)
  if (M == 4 && C == 12 && getenv("QK_NG2")) return 512;
  if (M == 4 && C <= 11 && getenv("QK_CONS")) return atoi(getenv("QK_CONS"));
  return M == 4 ? kConsumers4 : kConsumers3;
}

int tma_smem_bytes(int C, int M, int* ng, int* stages, int smax) {
  const int consumers = consumers_for(C, M);
  const int GT = 1 << (C - M);
  const int NG = GT >= consumers ? 1 : consumers / GT;
  const uint32_t stage = 16u << C;
  // each stage belongs to exactly one consumer group (S % NG == 0), so a
  // group never waits on a stage more than one mbarrier phase ahead
  int S = (int)(kSmemBudget / stage);
  // Stages are taken in chunk order by whichever group owns the chunk, so a
  // stage's barrier never runs more than one phase ahead of its waiter even
  // when S is not a multiple of NG (QK_NG2: 2 groups of 256 on 3 stages)
  // (with more stages than groups a group may wait for round r of a stage whose
  // round r - 1 has not completed yet, and the parity wait passes at once: M = 5
  // keeps one stage per group)
  if (!(NG == 2 && C == 12 && getenv("QK_NG2") && !getenv("QK_NG2_EVEN"))) S = (S / NG) * NG;
  if (S > 4 * NG) S = 4 * NG;
  if (const char* e = getenv("QK_SMAX")) smax = atoi(e);
  if (smax > 0) S = std::max(std::min(S, smax), NG);
  if (ng) *ng = NG;
  if (stages) *stages = S;
  if (S < 1 || (S < 2 && C != 13) || S < NG) return -1;  // C = 13: one 128-KiB stage
  return (int)(S * stage + 2 * S * 8);
}

int launch_block_tma(const TmaParams* p, int num_sms, CUstream_st* stream) {
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(k_block_tma<4, 32 + kConsumers4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_block_tma<3, 32 + kConsumers3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_block_tma<4, 32 + 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  if (p->M > 4) return -1;  // five register qubits: specialised kernels only
  int ng = 0, st = 0;
  const int smem = tma_smem_bytes(p->C, p->M, &ng, &st, p->smax);
  if (smem < 0) return -1;
  const uint64_t grid = p->nchunks < (uint64_t)num_sms ? p->nchunks : (uint64_t)num_sms;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (p->M == 4 && consumers_for(p->C, 4) == 512)
    k_block_tma<4, 32 + 512><<<(unsigned)grid, 32 + 512, smem, s>>>(*p);
  else if (p->M == 4)
    k_block_tma<4, 32 + kConsumers4><<<(unsigned)grid, 32 + kConsumers4, smem, s>>>(*p);
  else
    k_block_tma<3, 32 + kConsumers3><<<(unsigned)grid, 32 + kConsumers3, smem, s>>>(*p);
  return (int)cudaGetLastError();
}

}  // namespace qk
