// qk_kernels.cu — hand-written sm_100a kernels of the AIC simulation path.
//
//   k_block_pass   gate-block pass (simulator.py:338-376): one CTA
//                  per 2^C-amplitude chunk, register-tiled phases, swizzled
//                  shared-memory re-layouts between phases, 128-bit global
//                  loads/stores, diagonal runs as one table multiply.
//   k_build_tables diagonal-run phase tables (fusion of RZ/RZZ/CP/D<k> runs,
//                  the runtime counterpart of optimizer.py:184-276).
//   k_sqs          in-place bit permutation new[i] = old[bitswap(i, A, B)]
//                  (SURVEY K2/K3 single device; simulator.py:159-235) in one
//                  HBM pass over 256-B runs.
//   k_sqs_range    the reference's pair walk restricted to a thread range
//                  (simulator.py:117-176 with start/stop), for unit parity.
//   k_swap_seg     segment exchange for multi-process CSQS over NVLink P2P.
//   k_sumsq / k_gather  norm and readback (simulator.py:393-419).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qk_internal.h"

namespace qk {

bool first_on_device(unsigned long long* mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  const unsigned long long old = __atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL);
  return !(old & bit);
}

// ---------------------------------------------------------------------------
// helpers

__device__ __forceinline__ uint32_t swz(uint32_t i) {
  // XOR-fold of the 3-bit groups of i into the 16-B slot within a 128-B bank
  // row: a quarter-warp whose lane bits sit on positions distinct mod 3
  // (the planner guarantees it) hits 8 distinct slots -> conflict-free.
  return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

__device__ __forceinline__ double2 ld_g(const double2* p) {
  double2 r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_g(double2* p, double2 v) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---------------------------------------------------------------------------
// register-slot gate kernels (compile-time slots, runtime dispatch)

template <int M, int R>
__device__ __forceinline__ void h_slot(double2 (&v)[1 << M]) {
#pragma unroll
  for (int j = 0; j < (1 << M); ++j) {
    if (j & (1 << R)) continue;
    const double2 a = v[j], b = v[j | (1 << R)];
    v[j] = make_double2(a.x + b.x, a.y + b.y);
    v[j | (1 << R)] = make_double2(a.x - b.x, a.y - b.y);
  }
}

template <int M, int R>
__device__ __forceinline__ void x_slot(double2 (&v)[1 << M]) {
#pragma unroll
  for (int j = 0; j < (1 << M); ++j) {
    if (j & (1 << R)) continue;
    const double2 a = v[j];
    v[j] = v[j | (1 << R)];
    v[j | (1 << R)] = a;
  }
}

template <int M, int R>
__device__ __forceinline__ void mat_slot(double2 (&v)[1 << M], const double* __restrict__ m) {
  const double m00r = m[0], m00i = m[1], m01r = m[2], m01i = m[3];
  const double m10r = m[4], m10i = m[5], m11r = m[6], m11i = m[7];
#pragma unroll
  for (int j = 0; j < (1 << M); ++j) {
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

// controlled X, target slot R; control: register slot rc (creg) or thread flag tcond
template <int M, int R>
__device__ __forceinline__ void cx_slot(double2 (&v)[1 << M], int creg, int rc, int tcond) {
#pragma unroll
  for (int j = 0; j < (1 << M); ++j) {
    if (j & (1 << R)) continue;
    const int cond = creg ? ((j >> rc) & 1) : tcond;
    const double2 a = v[j], b = v[j | (1 << R)];
    v[j] = cond ? b : a;
    v[j | (1 << R)] = cond ? a : b;
  }
}

template <int M, int A, int B>
__device__ __forceinline__ void swap_slots(double2 (&v)[1 << M]) {
#pragma unroll
  for (int j = 0; j < (1 << M); ++j) {
    if (!((j >> A) & 1) || ((j >> B) & 1)) continue;  // bit A set, bit B clear
    const int k = j ^ (1 << A) ^ (1 << B);
    const double2 t = v[j];
    v[j] = v[k];
    v[k] = t;
  }
}

#define QK_DISPATCH_SLOT(FN, r, ...)                     \
  switch (r) {                                           \
    case 0: FN<M, 0>(__VA_ARGS__); break;                \
    case 1: if constexpr (M > 1) FN<M, 1>(__VA_ARGS__); break; \
    case 2: if constexpr (M > 2) FN<M, 2>(__VA_ARGS__); break; \
    case 3: if constexpr (M > 3) FN<M, 3>(__VA_ARGS__); break; \
    default: break;                                      \
  }

template <int M>
__device__ __forceinline__ void swap_dispatch(double2 (&v)[1 << M], int a, int b) {
  const int key = a * 4 + b;  // a < b
  switch (key) {
    case 1: if constexpr (M > 1) swap_slots<M, 0, 1>(v); break;
    case 2: if constexpr (M > 2) swap_slots<M, 0, 2>(v); break;
    case 3: if constexpr (M > 3) swap_slots<M, 0, 3>(v); break;
    case 6: if constexpr (M > 2) swap_slots<M, 1, 2>(v); break;
    case 7: if constexpr (M > 3) swap_slots<M, 1, 3>(v); break;
    case 11: if constexpr (M > 3) swap_slots<M, 2, 3>(v); break;
    default: break;
  }
}

// ---------------------------------------------------------------------------
// K1/K4: gate-block pass

template <int M, int MAXT>
__global__ void __launch_bounds__(MAXT, 512 / MAXT + 1) k_block_pass(double2* __restrict__ state,
                                                    const PassDesc* __restrict__ P,
                                                    const PhaseDesc* __restrict__ PH,
                                                    const OpDesc* __restrict__ OPS,
                                                    const double* __restrict__ coef,
                                                    const double2* __restrict__ tabs,
                                                    uint64_t cta_base) {
  extern __shared__ double2 sm[];
  constexpr int NA = 1 << M;
  const uint32_t tid = threadIdx.x;
  const uint64_t X = cta_base + blockIdx.x;
  const int nouter = P->nouter;
  uint64_t obase = 0;
  for (int k = 0; k < nouter; ++k) obase |= ((X >> k) & 1ull) << P->opos[k];

  double2 v[NA];
  const int np = P->nphases;
  const PhaseDesc* D = PH + P->phase0;
  for (int ph = 0; ph < np; ++ph, ++D) {
    const int T = D->tbits;
    uint32_t loct = 0;
    uint64_t addrt = obase;
    for (int k = 0; k < T; ++k) {
      if ((tid >> k) & 1u) {
        loct |= 1u << D->tpos[k];
        addrt += D->taddr[k];
      }
    }
    if (ph == 0) {
#pragma unroll
      for (int j = 0; j < NA; ++j) v[j] = ld_g(state + addrt + D->raddr[j]);
    } else {
#pragma unroll
      for (int j = 0; j < NA; ++j) v[j] = sm[swz(loct | D->rloc[j])];
    }
    const int oe = D->op_end;
    for (int o = D->op_begin; o < oe; ++o) {
      const OpDesc* op = OPS + o;
      const int code = op->code;
      const int r0 = op->r0;
      if (code == OP_H) {
        QK_DISPATCH_SLOT(h_slot, r0, v)
      } else if (code == OP_DIAG) {
        uint32_t pt = 0;
        for (int k = 0; k < T; ++k)
          if ((tid >> k) & 1u) pt |= op->tcontrib[k];
        const double2* tab = tabs + op->table;
#pragma unroll
        for (int j = 0; j < NA; ++j) v[j] = cmul(v[j], tab[pt | op->pr[j]]);
      } else if (code == OP_MAT) {
        const double* m = coef + op->coef;
        QK_DISPATCH_SLOT(mat_slot, r0, v, m)
      } else if (code == OP_X) {
        QK_DISPATCH_SLOT(x_slot, r0, v)
      } else if (code == OP_CX) {
        const int creg = op->ctrl_reg;
        const int rc = op->r1;
        const int tcond = creg ? 0 : (int)((loct >> op->ctrl) & 1u);
        QK_DISPATCH_SLOT(cx_slot, r0, v, creg, rc, tcond)
      } else if (code == OP_SWAP) {
        swap_dispatch<M>(v, r0, op->r1);
      } else if (code == OP_SCALE) {
        const double2 s = make_double2(coef[op->coef], coef[op->coef + 1]);
#pragma unroll
        for (int j = 0; j < NA; ++j) v[j] = cmul(v[j], s);
      }
    }
    if (ph == np - 1) {
#pragma unroll
      for (int j = 0; j < NA; ++j) st_g(state + addrt + D->raddr[j], v[j]);
    } else {
      if (ph > 0) __syncthreads();
#pragma unroll
      for (int j = 0; j < NA; ++j) sm[swz(loct | D->rloc[j])] = v[j];
      __syncthreads();
    }
  }
}

int launch_block_pass(double* state, const PassDesc* h, const PassDesc* d_pass,
                      const PhaseDesc* d_phases, const OpDesc* d_ops, const double* d_coef,
                      const double* d_tables, uint64_t first, CUstream_st* stream) {
  const int C = h->C, M = h->M;
  const unsigned threads = 1u << (C - M);
  const size_t smem = h->nphases > 1 ? ((size_t)16 << C) : 0;
  static unsigned long long attr_set = 0;
  if (first_on_device(&attr_set)) {
    const int mx = 16 << kMaxC;
    cudaFuncSetAttribute(k_block_pass<1, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_block_pass<2, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_block_pass<3, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_block_pass<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_block_pass<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  }
  const uint64_t total = h->ncta;
  const uint64_t max_grid = 1ull << 30;
  for (uint64_t base = 0; base < total; base += max_grid) {
    const unsigned grid = (unsigned)((total - base) < max_grid ? (total - base) : max_grid);
    auto* st = reinterpret_cast<double2*>(state);
    auto* tb = reinterpret_cast<const double2*>(d_tables);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t b0 = first + base;
    switch (M) {
      case 1: k_block_pass<1, 512><<<grid, threads, smem, s>>>(st, d_pass, d_phases, d_ops, d_coef, tb, b0); break;
      case 2: k_block_pass<2, 512><<<grid, threads, smem, s>>>(st, d_pass, d_phases, d_ops, d_coef, tb, b0); break;
      case 3: k_block_pass<3, 512><<<grid, threads, smem, s>>>(st, d_pass, d_phases, d_ops, d_coef, tb, b0); break;
      case 4:
        if (threads <= 256)
          k_block_pass<4, 256><<<grid, threads, smem, s>>>(st, d_pass, d_phases, d_ops, d_coef, tb, b0);
        else
          k_block_pass<4, 512><<<grid, threads, smem, s>>>(st, d_pass, d_phases, d_ops, d_coef, tb, b0);
        break;
      default: return -1;
    }
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// diagonal-run tables

__global__ void k_build_tables(const TableDesc* __restrict__ T, const TableGate* __restrict__ G,
                               const double2* __restrict__ E, double2* __restrict__ pool) {
  const TableDesc d = T[blockIdx.y];
  const uint64_t n = 1ull << d.bits;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(d.scale, d.scale_im);
    for (int g = d.g0; g < d.g0 + d.ng; ++g) {
      const TableGate& tg = G[g];
      uint32_t sub = 0;
      for (int j = 0; j < tg.nt; ++j) sub |= (uint32_t)((x >> tg.slot[j]) & 1) << (tg.nt - 1 - j);
      acc = cmul(acc, E[tg.entries + sub]);
    }
    pool[d.out + x] = acc;
  }
}

int launch_build_tables(const TableDesc* d_tables, int ntables, const TableGate* d_gates,
                        const double* d_entries, double* d_pool, CUstream_st* stream) {
  if (ntables <= 0) return 0;
  for (int base = 0; base < ntables; base += 65535) {
    const int nt = (ntables - base) < 65535 ? (ntables - base) : 65535;
    dim3 grid(16, nt);
    k_build_tables<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        d_tables + base, d_gates, reinterpret_cast<const double2*>(d_entries),
        reinterpret_cast<double2*>(d_pool));
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2/K3 (single device): in-place bit permutation new[i] = old[bitswap(i, A, B)].
// The planner splits the address bits into a tile set V (the low w bits, the
// partners of any of them, and fillers up to 2^8..2^10 amplitudes) and the
// outer bits O. Pairs inside V permute within a tile; pairs inside O map tile
// X to tile Y = pi(X). A CTA moves one canonical tile pair (X <= Y) per loop
// iteration: every thread issues all its loads (runs of 2^w amplitudes are
// contiguous across lanes), then writes the swapped/permuted values back —
// through shared memory only when the in-tile permutation is not the identity.

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

__global__ void __launch_bounds__(256) k_sqs(double2* __restrict__ state, const __grid_constant__ SqsDesc S) {
  extern __shared__ double2 sm[];
  const int nv = S.nv, w = S.w;
  const uint32_t tile = 1u << nv;
  const uint64_t nunits = 1ull << S.nouter;
  const int lane = threadIdx.x & 31;
  const uint32_t e0 = threadIdx.x;
  const int per = tile > 256 ? (int)(tile >> 8) : 1;
  const bool active = e0 < tile;
  const uint32_t wmask = (1u << w) - 1;
  uint64_t off[4];
  uint32_t pe[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const uint32_t e = e0 + 256u * m;
    uint64_t o = e & wmask;
    for (int b = w; b < nv; ++b) o |= (uint64_t)((e >> b) & 1u) << S.vpos[b];
    off[m] = o;
    uint32_t q = e;
    for (int k = 0; k < S.nvp; ++k) {
      const uint32_t d = ((q >> S.va[k]) ^ (q >> S.vb[k])) & 1u;
      q ^= (d << S.va[k]) | (d << S.vb[k]);
    }
    pe[m] = q;
  }
  for (uint64_t X = blockIdx.x; X < nunits; X += gridDim.x) {
    uint64_t c = 0;
    if (lane < S.nop) {
      const uint64_t d = ((X >> S.oa[lane]) ^ (X >> S.ob[lane])) & 1ull;
      c = (d << S.oa[lane]) | (d << S.ob[lane]);
    }
    if (lane + 32 < S.nop) {
      const uint64_t d = ((X >> S.oa[lane + 32]) ^ (X >> S.ob[lane + 32])) & 1ull;
      c |= (d << S.oa[lane + 32]) | (d << S.ob[lane + 32]);
    }
    const uint64_t Y = X ^ warp_or64(c);
    if (Y < X) continue;
    const bool same = (Y == X);
    if (same && S.ident) continue;
    uint64_t cx = 0, cy = 0;
    if (lane < S.nouter) {
      cx = ((X >> lane) & 1ull) << S.opos[lane];
      cy = ((Y >> lane) & 1ull) << S.opos[lane];
    }
    if (lane + 32 < S.nouter) {
      cx |= ((X >> (lane + 32)) & 1ull) << S.opos[lane + 32];
      cy |= ((Y >> (lane + 32)) & 1ull) << S.opos[lane + 32];
    }
    const uint64_t bx = warp_or64(cx), by = warp_or64(cy);
    double2 a[4], b[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m < per && active) {
        a[m] = ld_g(state + bx + off[m]);
        if (!same) b[m] = ld_g(state + by + off[m]);
      }
    }
    if (S.ident) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (m < per && active) {
          st_g(state + bx + off[m], b[m]);
          st_g(state + by + off[m], a[m]);
        }
      }
      continue;
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m < per && active) {
        sm[swz(e0 + 256u * m)] = a[m];
        if (!same) sm[tile + swz(e0 + 256u * m)] = b[m];
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m < per && active) {
        const uint32_t q = swz(pe[m]);
        if (same) {
          st_g(state + bx + off[m], sm[q]);
        } else {
          st_g(state + bx + off[m], sm[tile + q]);
          st_g(state + by + off[m], sm[q]);
        }
      }
    }
    __syncthreads();
  }
}

// cp.async variant: 16-B async copies land in (swizzled) shared memory without
// register staging, so several CTAs per SM keep ~100+ KiB of loads in flight.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__global__ void __launch_bounds__(256) k_sqs_async(double2* __restrict__ state, const __grid_constant__ SqsDesc S) {
  extern __shared__ double2 sm[];
  const int nv = S.nv, w = S.w;
  const uint32_t tile = 1u << nv;
  const uint64_t nunits = 1ull << S.nouter;
  const int lane = threadIdx.x & 31;
  const uint32_t e0 = threadIdx.x;
  const int per = tile > 256 ? (int)(tile >> 8) : 1;
  const bool active = e0 < tile;
  const uint32_t wmask = (1u << w) - 1;
  uint64_t off[4];
  uint32_t pe[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const uint32_t e = e0 + 256u * m;
    uint64_t o = e & wmask;
    for (int b = w; b < nv; ++b) o |= (uint64_t)((e >> b) & 1u) << S.vpos[b];
    off[m] = o;
    uint32_t q = e;
    for (int k = 0; k < S.nvp; ++k) {
      const uint32_t d = ((q >> S.va[k]) ^ (q >> S.vb[k])) & 1u;
      q ^= (d << S.va[k]) | (d << S.vb[k]);
    }
    pe[m] = swz(q);
  }
  for (uint64_t X = blockIdx.x; X < nunits; X += gridDim.x) {
    uint64_t c = 0;
    if (lane < S.nop) {
      const uint64_t d = ((X >> S.oa[lane]) ^ (X >> S.ob[lane])) & 1ull;
      c = (d << S.oa[lane]) | (d << S.ob[lane]);
    }
    if (lane + 32 < S.nop) {
      const uint64_t d = ((X >> S.oa[lane + 32]) ^ (X >> S.ob[lane + 32])) & 1ull;
      c |= (d << S.oa[lane + 32]) | (d << S.ob[lane + 32]);
    }
    const uint64_t Y = X ^ warp_or64(c);
    if (Y < X) continue;
    const bool same = (Y == X);
    if (same && S.ident) continue;
    uint64_t cx = 0, cy = 0;
    if (lane < S.nouter) {
      cx = ((X >> lane) & 1ull) << S.opos[lane];
      cy = ((Y >> lane) & 1ull) << S.opos[lane];
    }
    if (lane + 32 < S.nouter) {
      cx |= ((X >> (lane + 32)) & 1ull) << S.opos[lane + 32];
      cy |= ((Y >> (lane + 32)) & 1ull) << S.opos[lane + 32];
    }
    const uint64_t bx = warp_or64(cx), by = warp_or64(cy);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m < per && active) {
        const uint32_t e = swz(e0 + 256u * m);
        cp_async16(sm + e, state + bx + off[m]);
        if (!same) cp_async16(sm + tile + e, state + by + off[m]);
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (m < per && active) {
        if (same) {
          st_g(state + bx + off[m], sm[pe[m]]);
        } else {
          st_g(state + bx + off[m], sm[tile + pe[m]]);
          st_g(state + by + off[m], sm[pe[m]]);
        }
      }
    }
    __syncthreads();
  }
}

// Out-of-place variant (second buffer): every destination tile X takes the
// permuted source tile Y = X ^ swap once, so there are no pairs, no skipped
// units and the reads and writes go to different buffers.
__global__ void __launch_bounds__(256) k_sqs_oop(const double2* __restrict__ src, double2* __restrict__ dst,
                                                 const __grid_constant__ SqsDesc S) {
  extern __shared__ double2 sm[];
  const int nv = S.nv, w = S.w;
  const uint32_t tile = 1u << nv;
  const uint64_t nunits = 1ull << S.nouter;
  const int lane = threadIdx.x & 31;
  const uint32_t e0 = threadIdx.x;
  const int per = tile > 256 ? (int)(tile >> 8) : 1;
  const bool active = e0 < tile;
  const uint32_t wmask = (1u << w) - 1;
  uint64_t off[4];
  uint32_t pe[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const uint32_t e = e0 + 256u * m;
    uint64_t o = e & wmask;
    for (int b = w; b < nv; ++b) o |= (uint64_t)((e >> b) & 1u) << S.vpos[b];
    off[m] = o;
    uint32_t q = e;
    for (int k = 0; k < S.nvp; ++k) {
      const uint32_t d = ((q >> S.va[k]) ^ (q >> S.vb[k])) & 1u;
      q ^= (d << S.va[k]) | (d << S.vb[k]);
    }
    pe[m] = swz(q);
  }
  for (uint64_t X = blockIdx.x; X < nunits; X += gridDim.x) {
    uint64_t c = 0;
    if (lane < S.nop) {
      const uint64_t d = ((X >> S.oa[lane]) ^ (X >> S.ob[lane])) & 1ull;
      c = (d << S.oa[lane]) | (d << S.ob[lane]);
    }
    if (lane + 32 < S.nop) {
      const uint64_t d = ((X >> S.oa[lane + 32]) ^ (X >> S.ob[lane + 32])) & 1ull;
      c |= (d << S.oa[lane + 32]) | (d << S.ob[lane + 32]);
    }
    const uint64_t Y = X ^ warp_or64(c);
    uint64_t cx = 0, cy = 0;
    if (lane < S.nouter) {
      cx = ((X >> lane) & 1ull) << S.opos[lane];
      cy = ((Y >> lane) & 1ull) << S.opos[lane];
    }
    if (lane + 32 < S.nouter) {
      cx |= ((X >> (lane + 32)) & 1ull) << S.opos[lane + 32];
      cy |= ((Y >> (lane + 32)) & 1ull) << S.opos[lane + 32];
    }
    const uint64_t bx = warp_or64(cx), by = warp_or64(cy);
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (m < per && active) cp_async16(sm + swz(e0 + 256u * m), src + by + off[m]);
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (m < per && active) st_g(dst + bx + off[m], sm[pe[m]]);
    __syncthreads();
  }
}

int launch_sqs_oop(const double* src, double* dst, const SqsDesc* h, CUstream_st* stream) {
  const uint64_t units = 1ull << h->nouter;
  const size_t smem = (size_t)16u << h->nv;
  // many more CTAs than fit (8 per SM): the block scheduler balances the
  // tail better than a persistent grid (QAOA30 SQS: 60.1 ms in place,
  // 59.0 ms here at 12 per SM, 54.9 ms at 64 per SM, 67 ms with one unit each)
  static const int per_sm = getenv("QK_SQS_OOP_CTAS") ? atoi(getenv("QK_SQS_OOP_CTAS")) : 64;
  uint64_t grid = 148ull * per_sm;
  if (grid > units) grid = units;
  k_sqs_oop<<<(unsigned)grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), *h);
  return (int)cudaGetLastError();
}

int launch_sqs(double* state, const SqsDesc* h, const SqsDesc* /*d*/, CUstream_st* stream) {
  if (!getenv("QK_SQS_REG")) {
    const uint64_t units = 1ull << h->nouter;
    const size_t smem = (size_t)2 * (16u << h->nv);
    static unsigned long long attr2 = 0;
    if (first_on_device(&attr2))
      cudaFuncSetAttribute(k_sqs_async, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * (16 << 10));
    // oversubscribed like k_sqs_oop (7 fit per SM): QAOA33r3's SQS 2.48 -> 2.32 s
    static const int per_sm = getenv("QK_SQS_CTAS") ? atoi(getenv("QK_SQS_CTAS")) : 64;
    uint64_t grid = 148ull * per_sm;
    if (grid > units) grid = units;
    k_sqs_async<<<(unsigned)grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<double2*>(state), *h);
    return (int)cudaGetLastError();
  }
  const uint64_t units = 1ull << h->nouter;
  const size_t smem = h->ident ? 0 : (size_t)2 * (16u << h->nv);
  uint64_t grid = 148ull * 6;
  if (grid > units) grid = units;
  k_sqs<<<(unsigned)grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(state), *h);
  return (int)cudaGetLastError();
}

// reference pair walk over t in [start, stop): m = bitshift(t), n = bitswap(m), swap iff m > n
struct PairArgs {
  int np, k;
  int p[16], q[16];
  int a[64], b[64];
};

__global__ void k_sqs_range(double2* __restrict__ state, uint64_t start, uint64_t stop,
                            PairArgs pa) {
  for (uint64_t t = start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < stop;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = t;
    for (int i = 0; i < pa.np; ++i) {
      const uint64_t d = ((m >> pa.p[i]) ^ (m >> pa.q[i])) & 1ull;
      m ^= (d << pa.p[i]) | (d << pa.q[i]);
    }
    uint64_t n = m;
    for (int i = 0; i < pa.k; ++i) {
      const uint64_t d = ((n >> pa.a[i]) ^ (n >> pa.b[i])) & 1ull;
      n ^= (d << pa.a[i]) | (d << pa.b[i]);
    }
    if (m > n) {
      const double2 x = state[m];
      state[m] = state[n];
      state[n] = x;
    }
  }
}

int launch_sqs_range(double* state, uint64_t start, uint64_t stop, const int* p, const int* q,
                     int np, const int* a, const int* b, int k, CUstream_st* stream) {
  if (stop <= start) return 0;
  PairArgs pa{};
  pa.np = np;
  pa.k = k;
  for (int i = 0; i < np; ++i) { pa.p[i] = p[i]; pa.q[i] = q[i]; }
  for (int i = 0; i < k; ++i) { pa.a[i] = a[i]; pa.b[i] = b[i]; }
  const uint64_t n = stop - start;
  const unsigned grid = (unsigned)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  k_sqs_range<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(state), start, stop, pa);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// segment exchange (either pointer may be a peer mapping over NVLink)

// Segment exchange. Every thread keeps 4 independent 16-B loads of each side
// in flight before it stores (the remote side is NVLink peer memory, ~2 us
// away): the grid needs ~1.8 MB in flight to fill a 900 GB/s link.
constexpr int kSwapUnroll = 4;

__global__ void __launch_bounds__(256) k_swap_seg(double2* __restrict__ a, double2* __restrict__ b, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * kSwapUnroll) {
    double2 x[kSwapUnroll], y[kSwapUnroll];
#pragma unroll
    for (int u = 0; u < kSwapUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n) {
        x[u] = ld_g(a + i);
        y[u] = ld_g(b + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kSwapUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n) {
        st_g(a + i, y[u]);
        st_g(b + i, x[u]);
      }
    }
  }
}

// Device-side barrier between the shards of one exchange (no host round
// trip): shard `me` publishes `epoch` into slot `me` of every peer's flag
// array (system-scope release), then waits until each peer has published it
// into its own array. Stream order puts every earlier kernel of this shard
// before the release. A peer that never arrives (dead process) trips a 60-s
// timeout that sets *err instead of hanging the GPU.
struct PeerFlags {
  int32_t n, me;
  int32_t idx[64];
  unsigned long long* remote[64];  // peer idx[k]'s flag array (mapped over NVLink / IPC)
  unsigned long long epoch[64];    // this pair's meeting count (both sides count alike)
};

__global__ void k_peer_barrier(unsigned long long* __restrict__ mine, const __grid_constant__ PeerFlags pf,
                               int* __restrict__ err) {
  const int k = threadIdx.x;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  const unsigned long long epoch = k < pf.n ? pf.epoch[k] : 0ull;
  if (k < pf.n) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pf.remote[k] + pf.me), "l"(epoch) : "memory");
  if (k < pf.n) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + pf.idx[k]) : "memory");
      if (v >= epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60000000000ull) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

int launch_peer_barrier(unsigned long long* mine, unsigned long long* const* remote, const int* idx,
                        const unsigned long long* epochs, int n, int me, int* err, CUstream_st* stream) {
  if (n > 64 || n < 0) return -1;
  PeerFlags pf{};
  pf.n = n;
  pf.me = me;
  for (int k = 0; k < n; ++k) {
    pf.idx[k] = idx[k];
    pf.remote[k] = remote[k];
    pf.epoch[k] = epochs[k];
  }
  k_peer_barrier<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(mine, pf, err);
  return (int)cudaGetLastError();
}

// Strided segment exchange: element t of the segment sits at
// deposit(t) = sum over runs of ((t >> src) & (2^len - 1)) << dst, the same
// offsets in both shards (every shard holds the same layout).
struct SwapRuns {
  int32_t n;
  uint8_t src[24], dst[24], len[24];
};

__global__ void __launch_bounds__(256) k_swap_strided(double2* __restrict__ a, double2* __restrict__ b, uint64_t n,
                                                      const __grid_constant__ SwapRuns R) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += stride * kSwapUnroll) {
    double2 x[kSwapUnroll], y[kSwapUnroll];
    uint64_t off[kSwapUnroll];
#pragma unroll
    for (int u = 0; u < kSwapUnroll; ++u) {
      const uint64_t t = t0 + u * stride;
      off[u] = 0;
      for (int k = 0; k < R.n; ++k) off[u] |= ((t >> R.src[k]) & ((1ull << R.len[k]) - 1)) << R.dst[k];
      if (t < n) {
        x[u] = ld_g(a + off[u]);
        y[u] = ld_g(b + off[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kSwapUnroll; ++u) {
      if (t0 + u * stride < n) {
        st_g(a + off[u], y[u]);
        st_g(b + off[u], x[u]);
      }
    }
  }
}

int launch_swap_strided(double* a, double* b, uint64_t n, const int* pos, int npos, CUstream_st* stream) {
  // pos: physical positions of the free bits (ascending = thread-order bits)
  if (!n) return 0;
  SwapRuns R{};
  for (int k = 0; k < npos;) {
    int e = k + 1;
    while (e < npos && pos[e] == pos[e - 1] + 1) ++e;
    if (R.n >= 24) return -1;
    R.src[R.n] = (uint8_t)k;
    R.dst[R.n] = (uint8_t)pos[k];
    R.len[R.n] = (uint8_t)(e - k);
    ++R.n;
    k = e;
  }
  const uint64_t blocks = (n + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 148 * 8 ? blocks : 148 * 8);
  k_swap_strided<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(a), reinterpret_cast<double2*>(b), n, R);
  return (int)cudaGetLastError();
}

// With lazy module loading (the CUDA 12 default) the first launch of a kernel
// loads it, and a load may wait for the kernels running on the device. A
// member enqueueing its first swap while its own barrier kernel already spins
// for a member the host has not reached yet would then deadlock. Every kernel
// an exchange step launches is therefore loaded when the handle is created.
int preload_exchange_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)k_peer_barrier, (const void*)k_swap_seg, (const void*)k_swap_strided,
                       (const void*)k_sqs, (const void*)k_sqs_async, (const void*)k_sqs_oop};
  for (const void* f : fns)
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return (int)cudaGetLastError();
  return 0;
}

int launch_swap_segments(double* a, double* b, uint64_t n, CUstream_st* stream) {
  if (!n) return 0;
  const uint64_t blocks = (n + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 148 * 8 ? blocks : 148 * 8);
  k_swap_seg<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<double2*>(a), reinterpret_cast<double2*>(b), n);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// norm: deterministic two-level reduction of sum |a|^2

constexpr int kSumBlocks = 148 * 8;

__global__ void __launch_bounds__(256) k_sumsq(const double2* __restrict__ s, uint64_t n,
                                               double* __restrict__ partial) {
  __shared__ double red[256];
  double acc = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 v = s[i];
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_sum_final(const double* __restrict__ partial, int n, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

int launch_sum_final(const double* partial, int n, double* out, CUstream_st* stream) {
  k_sum_final<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(partial, n, out);
  return (int)cudaGetLastError();
}

int launch_sumsq(const double* state, uint64_t n, double* d_partial, double* d_out,
                 CUstream_st* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  k_sumsq<<<kSumBlocks, 256, 0, s>>>(reinterpret_cast<const double2*>(state), n, d_partial);
  k_sum_final<<<1, 256, 0, s>>>(d_partial, kSumBlocks, d_out);
  return (int)cudaGetLastError();
}

__global__ void k_gather(const double2* __restrict__ s, const uint64_t* __restrict__ idx,
                         uint64_t n, double2* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = s[idx[i]];
}

int launch_gather(const double* state, const uint64_t* d_idx, uint64_t count, double* d_out,
                  CUstream_st* stream) {
  if (!count) return 0;
  const uint64_t blocks = (count + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
  k_gather<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const double2*>(state), d_idx, count, reinterpret_cast<double2*>(d_out));
  return (int)cudaGetLastError();
}

struct PermArgs {
  int n;
  int perm[64];
};

// logical index l -> physical p: bit pos of p = bit perm[pos] of l (simulator.py:415-417)
__global__ void k_gather_logical(const double2* __restrict__ s, PermArgs pa, uint64_t start,
                                 uint64_t n, double2* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t l = start + i;
    uint64_t p = 0;
    for (int pos = 0; pos < pa.n; ++pos) p |= ((l >> pa.perm[pos]) & 1ull) << pos;
    out[i] = s[p];
  }
}

int launch_gather_logical(const double* state, const int* perm, int n, uint64_t start,
                          uint64_t count, double* d_out, CUstream_st* stream) {
  if (!count) return 0;
  PermArgs pa{};
  pa.n = n;
  for (int i = 0; i < n; ++i) pa.perm[i] = perm[i];
  const uint64_t blocks = (count + 255) / 256;
  const unsigned grid = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
  k_gather_logical<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const double2*>(state), pa, start, count, reinterpret_cast<double2*>(d_out));
  return (int)cudaGetLastError();
}

// Overlap <phi|psi> of the state with a product state (analytic parity at
// sizes beyond the CPU reference): conj(phi_j) is the product
// of four 1024-entry tables, one per 10-bit group of the memory index j
// (built on the host from the per-qubit factors and the layout). Deterministic
// two-level reduction like k_sumsq.
constexpr int kOvBlocks = 148 * 8;

__global__ void __launch_bounds__(256) k_overlap(const double2* __restrict__ s, uint64_t n,
                                                 const double2* __restrict__ tabs,
                                                 double2* __restrict__ partial) {
  extern __shared__ double2 T[];  // 4 x 1024
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) T[i] = tabs[i];
  __syncthreads();
  double re = 0.0, im = 0.0;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double2 a = T[j & 1023], b = T[1024 + ((j >> 10) & 1023)];
    const double2 c = T[2048 + ((j >> 20) & 1023)], d = T[3072 + ((j >> 30) & 1023)];
    const double2 ab = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    const double2 cd = make_double2(c.x * d.x - c.y * d.y, c.x * d.y + c.y * d.x);
    const double2 f = make_double2(ab.x * cd.x - ab.y * cd.y, ab.x * cd.y + ab.y * cd.x);
    const double2 v = s[j];
    re = fma(f.x, v.x, fma(-f.y, v.y, re));
    im = fma(f.x, v.y, fma(f.y, v.x, im));
  }
  __shared__ double rr[256], ri[256];
  rr[threadIdx.x] = re;
  ri[threadIdx.x] = im;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      rr[threadIdx.x] += rr[threadIdx.x + w];
      ri[threadIdx.x] += ri[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(rr[0], ri[0]);
}

__global__ void k_overlap_final(const double2* __restrict__ partial, int n, double2* __restrict__ out) {
  __shared__ double rr[256], ri[256];
  double re = 0.0, im = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    re += partial[i].x;
    im += partial[i].y;
  }
  rr[threadIdx.x] = re;
  ri[threadIdx.x] = im;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      rr[threadIdx.x] += rr[threadIdx.x + w];
      ri[threadIdx.x] += ri[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = make_double2(rr[0], ri[0]);
}

int overlap_scratch_bytes() { return (4096 + kOvBlocks + 1) * 16; }

int launch_overlap(const double* state, uint64_t n, const double* d_tabs, double* d_work, CUstream_st* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) cudaFuncSetAttribute(k_overlap, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 16);
  double2* part = reinterpret_cast<double2*>(d_work);
  k_overlap<<<kOvBlocks, 256, 4096 * 16, st>>>(reinterpret_cast<const double2*>(state), n,
                                               reinterpret_cast<const double2*>(d_tabs), part);
  k_overlap_final<<<1, 256, 0, st>>>(part, kOvBlocks, part + kOvBlocks);
  return (int)cudaGetLastError();
}

__global__ void k_set_one(double2* s) { s[0] = make_double2(1.0, 0.0); }

int launch_fill_zero_one(double* state, uint64_t n, int set_first, CUstream_st* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(state, 0, n * 16, s);
  if (e != cudaSuccess) return (int)e;
  if (set_first) k_set_one<<<1, 1, 0, s>>>(reinterpret_cast<double2*>(state));
  return (int)cudaGetLastError();
}

}  // namespace qk
