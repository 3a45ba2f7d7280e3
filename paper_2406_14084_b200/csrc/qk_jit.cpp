// qk_jit.cpp — load-time specialisation of gate-block passes for sm_100a.
//
// The persistent TMA pass of qk_tma.cu interprets a phase program. Its
// register array crosses data-dependent branches, and the register moves at
// those merges dominate heavy passes (SASS: ~2300 MOVs, ~950 instructions per
// thread per phase against ~210 useful). Here every distinct pass *structure*
// (chunk width, phases, register sets, op kinds and slots) is emitted as
// straight-line CUDA with all indices as immediates and compiled once with
// NVRTC. Angles and table offsets stay kernel parameters, so structurally
// identical passes share one kernel.
//
// Cubins are cached in process and on disk ($QK_JIT_CACHE, default
// ~/.cache/qkb200/jit). NVRTC is dlopen'ed; without it the interpreter runs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <set>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "qk_internal.h"

namespace qk {
namespace {

// ---- NVRTC through dlopen -------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  bool ok = false;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char*) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    n.create = (decltype(n.create))dlsym(h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(h, "nvrtcCompileProgram");
    n.cubin_size = (decltype(n.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(h, "nvrtcGetCUBIN");
    n.log_size = (decltype(n.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(h, "nvrtcGetProgramLog");
    n.destroy = (decltype(n.destroy))dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.destroy;
  });
  return n;
}

// ---- kernel skeleton (same protocol as qk_tma.cu) ----------------------------
const char* kPreamble = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
struct alignas(64) QkMap { unsigned char b[128]; };
struct QkJitParams {
  QkMap map;
  const double2* tabs;
  double2* state;
  double2* out;
  u64 nchunks;
  double* nrm;
  u64 split;  // sub-launch over part of the chunks (qk_insert); 0 = every chunk
  long long toff[QK_NTAB + 1];
  double coef[QK_NCOEF + 1];
  QkMap smap;  // unbounded view of the state (TMA-store epilogue; map may be a bounded load view)
};
__device__ __forceinline__ u32 su32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(u64* b, u32 parity) {
  asm volatile("{\n\t.reg .pred P;\nQKW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra QKW_%=;\n}"
               ::"r"(su32(b)), "r"(parity) : "memory"); }
__device__ __forceinline__ void tma_load(void* dst, const QkMap* map, int c0, int c1, u64* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory"); }
__device__ __forceinline__ void tma_prefetch(const QkMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1) : "memory"); }
__device__ __forceinline__ u32 mapa(u32 a, u32 r) {
  u32 d; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r)); return d; }
__device__ __forceinline__ void mbar_arrive_remote(u32 rbar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory"); }
__device__ __forceinline__ void mbar_wait_cl(u64* b, u32 parity) {
  asm volatile("{\n\t.reg .pred P;\nQKC_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra QKC_%=;\n}"
               ::"r"(su32(b)), "r"(parity) : "memory"); }
__device__ __forceinline__ double2 ld_cl(u32 a) {
  double2 v; asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ u32 cl_rank() { u32 r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ u32 cl_id() { u32 r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
__device__ __forceinline__ u32 cl_num() { u32 r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void gbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory"); }
__device__ __forceinline__ u32 swz(u32 i) { return i ^ ((i >> 3) & 7u); }
// split word: bits 0..1 n, bits 2+6k.. position k (chunk-index bit, ascending),
// bit 20+k its value, bit 23 accumulate the fused norm. The compact counter c
// enumerates the chunks whose n fixed bits hold those values.
__device__ __forceinline__ u64 qk_insert(u64 c, u64 w) {
  const int n = (int)(w & 3ull);
  for (int k = 0; k < n; ++k) {
    const int pos = (int)((w >> (2 + 6 * k)) & 63ull);
    const u64 v = (w >> (20 + k)) & 1ull;
    c = ((c >> pos) << (pos + 1)) | (v << pos) | (c & ((1ull << pos) - 1ull));
  }
  return c;
}
__device__ __forceinline__ void hb(double2& a, double2& b) {
  a.x += b.x; a.y += b.y; b.x = fma(-2.0, b.x, a.x); b.y = fma(-2.0, b.y, a.y); }
__device__ __forceinline__ void xb(double2& a, double2& b) { double2 t = a; a = b; b = t; }
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }
)CUDA";

struct Gen {
  std::ostringstream o;
  int ntab = 0, ncoef = 0;
};

// One real output of a 2x2 complex map as a minimal FMA chain: terms with
// coefficient 0 vanish, +-1 are free adds, the rest read a parameter slot
// (pushed to `coef`). Structure (which terms are 0 / +-1 / general) is part of
// the kernel source; general values stay parameters.
typedef std::map<double, int> SlotCache;  // value -> parameter slot (one gate's coefficients)

std::string lin(const std::vector<std::pair<double, std::string>>& terms, std::vector<double>* coef,
                SlotCache* cache) {
  std::string e;
  std::vector<std::pair<double, std::string>> gen;
  for (auto& t : terms) {
    if (t.first == 0.0) continue;
    if (t.first == 1.0 || t.first == -1.0) {
      const bool neg = t.first < 0;
      if (e.empty()) e = neg ? "(-" + t.second + ")" : t.second;
      else e = "(" + e + (neg ? " - " : " + ") + t.second + ")";
    } else {
      gen.push_back(t);
    }
  }
  for (auto& t : gen) {
    auto it = cache->find(t.first);
    if (it == cache->end()) {
      it = cache->emplace(t.first, (int)coef->size()).first;
      coef->push_back(t.first);
    }
    const std::string c = "p.coef[" + std::to_string(it->second) + "]";
    if (e.empty()) e = "(" + c + " * " + t.second + ")";
    else e = "fma(" + c + ", " + t.second + ", " + e + ")";
  }
  return e.empty() ? "0.0" : e;
}

// n0 = m00 a + m01 b, n1 = m10 a + m11 b (m = 8 doubles: re, im row-major)
void emit_mat(std::ostringstream& b, int j, int jj, const double* m, std::vector<double>* coef,
              SlotCache* cache) {
  const std::string A = "v[" + std::to_string(j) + "]", B = "v[" + std::to_string(jj) + "]";
  auto out = [&](const double* r) {
    // re: r0 a.x - r1 a.y + r2 b.x - r3 b.y ; im: r0 a.y + r1 a.x + r2 b.y + r3 b.x
    std::string x = lin({{r[0], A + ".x"}, {-r[1], A + ".y"}, {r[2], B + ".x"}, {-r[3], B + ".y"}}, coef, cache);
    std::string y = lin({{r[0], A + ".y"}, {r[1], A + ".x"}, {r[2], B + ".y"}, {r[3], B + ".x"}}, coef, cache);
    return "make_double2(" + x + ", " + y + ")";
  };
  const std::string n0 = out(m), n1 = out(m + 4);
  b << "    { const double2 n0 = " << n0 << ", n1 = " << n1 << "; " << A << " = n0; " << B << " = n1; }\n";
}

// ---- shared-memory layouts ---------------------------------------------------
// A layout maps chunk index i to the 16-B slot i ^ sum_{p >= 3, bit p of i} m[p]
// (m[p] < 8 only touches the bank bits 0..2, so it is a bijection). LDS.128 /
// STS.128 are served 8 lanes at a time; lanes 0..2 of a phase sit on chunk
// positions a0..a2, and the access is conflict-free iff their bank
// contributions are linearly independent over GF(2). Phase 0 reads the TMA
// SWIZZLE_128B image (m[3..5] = 1, 2, 4, nothing above); every later layout
// is chosen per phase transition so that both the writing phase's lanes and
// the reading phase's lanes are conflict-free.
typedef std::vector<uint8_t> Layout;

Layout sw128_layout(int C) {
  Layout m(C, 0);
  for (int p = 0; p < C; ++p) m[p] = p < 3 ? (uint8_t)(1u << p) : (p < 6 ? (uint8_t)(1u << (p - 3)) : 0);
  return m;
}

// TMA SWIZZLE_64B image (64-B rows): byte bits [4:5] ^= [7:8], i.e. i[0:1] ^= i[3:4]
Layout sw64_layout(int C) {
  Layout m(C, 0);
  for (int p = 0; p < C; ++p) m[p] = p < 3 ? (uint8_t)(1u << p) : (p < 5 ? (uint8_t)(1u << (p - 3)) : 0);
  return m;
}

bool indep3(uint8_t a, uint8_t b, uint8_t c) {
  return a && b && c && a != b && (a ^ b) != c && a != c && b != c;
}

Layout choose_layout(int C, const uint8_t* wl, const uint8_t* rl) {
  Layout m(C, 0);
  for (int p = 0; p < 3 && p < C; ++p) m[p] = (uint8_t)(1u << p);
  std::vector<int> freep;
  for (int k = 0; k < 3; ++k) {
    if (wl[k] >= 3 && std::find(freep.begin(), freep.end(), wl[k]) == freep.end()) freep.push_back(wl[k]);
    if (rl[k] >= 3 && std::find(freep.begin(), freep.end(), rl[k]) == freep.end()) freep.push_back(rl[k]);
  }
  const int nf = (int)freep.size();
  long long total = 1;
  for (int k = 0; k < nf; ++k) total *= 7;
  for (long long code = 0; code < total; ++code) {
    long long c = code;
    for (int k = 0; k < nf; ++k) {
      m[freep[k]] = (uint8_t)(1 + c % 7);
      c /= 7;
    }
    if (indep3(m[wl[0]], m[wl[1]], m[wl[2]]) && indep3(m[rl[0]], m[rl[1]], m[rl[2]])) return m;
  }
  return sw128_layout(C);  // no conflict-free choice (cannot happen for distinct lanes)
}

uint32_t lay(const Layout& m, uint32_t i) {
  uint32_t s = i;
  for (int p = 3; p < (int)m.size(); ++p)
    if (i >> p & 1) s ^= m[p];
  return s;
}

// base slot of a thread in layout m: XOR of its thread bits' slot contributions
void emit_lay_base(std::ostringstream& o, const char* var, const Layout& m, const uint8_t* tpos, int n) {
  o << "    const u32 " << var << " = 0u";
  for (int k = 0; k < n; ++k) o << " ^ (((tid >> " << k << ") & 1u) * " << lay(m, 1u << tpos[k]) << "u)";
  o << ";\n";
}

void emit_bits(std::ostringstream& o, const char* var, const char* src, const uint8_t* pos, int n) {
  o << "    const u32 " << var << " = 0u";
  for (int k = 0; k < n; ++k) o << " | (((" << src << " >> " << k << ") & 1u) << " << (int)pos[k] << ")";
  o << ";\n";
}

// TMA loads (or L2 prefetches) of one strided tile, coordinates computed from
// the chunk index `cv` (its bit k = the k-th non-tile physical bit).
std::string lazy_loads(const TmaParams& tp, const char* cv, const char* dst, bool prefetch, const char* ind) {
  TileDims td;
  if (!tile_dims(tp.tbit, tp.C, tp.nbits, &td, tp.rowbits)) return "";
  std::vector<int> oidx(tp.nbits, -1), tidx(tp.nbits, -1);
  for (int k = 0; k < tp.C; ++k) tidx[tp.tbit[k]] = k;
  int no = 0;
  for (int p = 0; p < tp.nbits; ++p)
    if (tidx[p] < 0) oidx[p] = no++;
  std::ostringstream o;
  for (int it = 0; it < (1 << td.nit); ++it) {
    std::vector<std::string> cs;
    for (int jd = 0; jd < td.rank; ++jd) {
      if (jd == 0) {
        cs.push_back("0");
        continue;
      }
      std::ostringstream c;
      c << "(int)(0ull";
      uint64_t konst = 0;
      for (int p = td.lo[jd]; p < td.lo[jd] + td.len[jd]; ++p) {
        if (oidx[p] >= 0)
          c << " | (((" << cv << " >> " << oidx[p] << ") & 1ull) << " << p - td.lo[jd] << ")";
        else if (td.box[jd] == 1 && tidx[p] >= td.inbox && ((it >> (tidx[p] - td.inbox)) & 1))
          konst |= 1ull << (p - td.lo[jd]);
      }
      c << " | " << konst << "ull)";
      cs.push_back(c.str());
    }
    o << ind;
    if (prefetch) {
      o << "asm volatile(\"cp.async.bulk.prefetch.tensor." << td.rank << "d.L2.global.tile [%0, {";
    } else {
      o << "asm volatile(\"cp.async.bulk.tensor." << td.rank
        << "d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {";
    }
    const int base = prefetch ? 1 : 2;
    for (int jd = 0; jd < td.rank; ++jd) o << (jd ? ", " : "") << "%" << base + jd;
    if (prefetch) {
      o << "}];\" :: \"l\"(&p.map)";
    } else {
      o << "}], [%" << base + td.rank << "];\" :: \"r\"(su32(" << dst << " + " << ((size_t)it << td.inbox) * 16
        << ")), \"l\"(&p.map)";
    }
    for (auto& c : cs) o << ", \"r\"(" << c << ")";
    if (!prefetch) o << ", \"r\"(su32(full + s))";
    o << " : \"memory\");\n";
  }
  return o.str();
}

}  // namespace

// TMA stores of one strided tile from the stage image (same boxes and
// coordinates as lazy_loads, so an in-place pass writes back what it read).
std::string lazy_stores(const TmaParams& tp, const char* cv, const char* src, const char* ind) {
  TileDims td;
  if (!tile_dims(tp.tbit, tp.C, tp.nbits, &td, tp.rowbits)) return "";
  std::vector<int> oidx(tp.nbits, -1), tidx(tp.nbits, -1);
  for (int k = 0; k < tp.C; ++k) tidx[tp.tbit[k]] = k;
  int no = 0;
  for (int p = 0; p < tp.nbits; ++p)
    if (tidx[p] < 0) oidx[p] = no++;
  std::ostringstream o;
  for (int it = 0; it < (1 << td.nit); ++it) {
    o << ind << "asm volatile(\"cp.async.bulk.tensor." << td.rank << "d.global.shared::cta.bulk_group [%0, {";
    for (int jd = 0; jd < td.rank; ++jd) o << (jd ? ", " : "") << "%" << 1 + jd;
    o << "}], [%" << 1 + td.rank << "];\" :: \"l\"(&p.smap)";
    for (int jd = 0; jd < td.rank; ++jd) {
      if (jd == 0) {
        o << ", \"r\"(0)";
        continue;
      }
      o << ", \"r\"((int)(0ull";
      uint64_t konst = 0;
      for (int p = td.lo[jd]; p < td.lo[jd] + td.len[jd]; ++p) {
        if (oidx[p] >= 0)
          o << " | (((" << cv << " >> " << oidx[p] << ") & 1ull) << " << p - td.lo[jd] << ")";
        else if (td.box[jd] == 1 && tidx[p] >= td.inbox && ((it >> (tidx[p] - td.inbox)) & 1))
          konst |= 1ull << (p - td.lo[jd]);
      }
      o << " | " << konst << "ull))";
    }
    o << ", \"r\"(su32(" << src << " + " << ((size_t)it << td.inbox) * 16 << ")) : \"memory\");\n";
  }
  o << ind << "asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n";
  return o.str();
}

// Shared-memory slices of per-chunk diagonal tables (12-bit passes with the
// table-aware chunk order). A table's chunk bits (co_v) are its top index
// bits, so the entries one chunk reads are one contiguous slice of
// 2^(inner bits). With the chunk order a CTA keeps the same slices over long
// stretches; staged in shared memory they stop being L2 gathers.
// Returns the slice size (entries) per table slot (0 = not staged).
std::vector<int> slice_plan(const TmaParams& tp, int st) {
  std::vector<int> out;
  // Measured: in-place QAOA33 (21 chunk bits, ~14k chunks per CTA) 1.69 ->
  // 1.63 s; QAOA30 (18 chunk bits) loses 0.165 -> 0.174 s, so only large states
  const bool on = tp.C >= 12 && !tp.xbits && tp.nbits - tp.C >= 20 && !getenv("QK_NO_SLICES") &&
                  !getenv("QK_NO_CORDER");
  long budget = (long)(218 << 10) - (long)st * (16L << tp.C);
  // a reload happens whenever the staged tables' chunk bits change: keep at
  // least 2^6 consecutive chunks per slice set (the low counter bits)
  const int nouter = tp.nbits - tp.C;
  const char* mr = getenv("QK_SLICE_RUN");
  const int min_run = mr ? atoi(mr) : 6;
  uint64_t cmask = 0;
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) {
      const TOp& op = tp.ops[o];
      if (op.code != OP_DIAG) continue;
      uint32_t inner = 0;
      for (int k = 0; k < 12; ++k) inner |= op.tcontrib[k];
      for (int j = 0; j < (1 << tp.M); ++j) inner |= op.pr[j];
      int ents = 1;
      while ((uint32_t)ents <= inner) ents <<= 1;
      bool outer_top = true;
      for (int k = 0; k < op.nco; ++k) outer_top = outer_top && op.co_v[k] >= (uint32_t)ents;
      uint64_t m2 = cmask;
      for (int k = 0; k < op.nco; ++k) m2 |= 1ull << op.co_k[k];
      if (on && op.nco > 0 && outer_top && (long)ents * 16 <= budget &&
          nouter - __builtin_popcountll(m2) >= min_run) {
        out.push_back(ents);
        budget -= (long)ents * 16;
        cmask = m2;
      } else {
        out.push_back(0);
      }
    }
  return out;
}

int jit_slice_bytes(const TmaParams& tp) {
  int ng = 0, st = 0;
  if (tma_smem_bytes(tp.C, tp.M, &ng, &st, tp.smax) < 0) return 0;
  int b = 0;
  for (int e : slice_plan(tp, st)) b += e * 16;
  if (tp.norm) b += 16 * 32 * 8;  // per-warp partial sums of the fused norm
  int nq = 0;                     // OP_QUAD factors: C + 1 per op per stage
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) nq += tp.ops[o].code == OP_QUAD;
  b += nq * (tp.C + 1 + 32 + (1 << std::max(0, tp.C - tp.M - 5))) * 16 * (st + 1);  // + the pending slot
  if (jit_pairs(tp)) b += 8 * st;                                                     // pair barriers
  return b;
}

static uint64_t table_chunk_mask(const TmaParams& tp);
// the specialised kernel walks the table-aware chunk order (cmap)
bool jit_corder(const TmaParams& tp) {
  return table_chunk_mask(tp) && tp.C >= 12 && !getenv("QK_NO_CORDER");
}

// Chunk bits the pass's diagonal tables read (per-chunk table terms).
static uint64_t table_chunk_mask(const TmaParams& tp) {
  uint64_t tmask = 0;
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o2 = tp.ph[ph].op_begin; o2 < tp.ph[ph].op_end; ++o2)
      if (tp.ops[o2].code == OP_DIAG)
        for (int k = 0; k < tp.ops[o2].nco; ++k) tmask |= 1ull << tp.ops[o2].co_k[k];
  return tmask;
}

// Cluster pairs for strided tiles with 128-B rows. Such a tile reads and
// writes 128-B pieces, and HBM serves isolated 128-B accesses at ~5 TB/s
// against ~6.1 TB/s for 256-B ones (tools/strided_bench.cu). When the
// lowest non-tile bit is address bit 3, chunks 2u and 2u + 1 hold the two
// halves of every 256-B segment: a 2-CTA cluster takes both, and its two
// producers meet at a per-stage mbarrier before every TMA load, so the halves
// reach the memory controller together.
bool jit_pairs(const TmaParams& tp) {
  if (!getenv("QK_PAIR") || !tp.lazy || tp.xbits || tp.rowbits != 3 || tp.nchunks < 2 || (tp.nchunks & 1)) return false;
  int ng = 0, st = 0;
  if (tma_smem_bytes(tp.C, tp.M, &ng, &st, tp.smax) < 0 || st < 2) return false;
  if (table_chunk_mask(tp) && tp.C >= 12 && !getenv("QK_NO_CORDER")) return false;  // chunk order walk
  uint32_t tb = 0;
  for (int x = 0; x < tp.C; ++x) tb |= 1u << tp.tbit[x];
  return (tb & 0xFu) == 0x7u;  // bits 0..2 in the tile, bit 3 the lowest chunk bit
}

// Emit the source of one pass. Returns false when the structure is outside
// what the generator covers (the caller keeps the interpreter).
bool jit_source(const TmaParams& tp, std::string* src, std::vector<long long>* toff,
                std::vector<double>* coef, int variant, const std::vector<QuadOp>* quad) {
  const int C = tp.C, M = tp.M, T = C - M, NA = 1 << M;
  if (M != 4 && M != 3 && M != 5) return false;
  if (M == 5 && (variant & 2)) return false;  // (the table-group pair factors index 4 slots)
  std::ostringstream b, pro;  // pro: consumer prologue (loop-invariant table values)
  toff->clear();
  coef->clear();
  // tables and coefficients become parameter slots in program order
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) {
      const TOp& op = tp.ops[o];
      if (op.code == OP_DIAG) toff->push_back(op.table);
    }
  // OP_QUAD / OP_QLITE ops: their data offsets follow the tables in toff;
  // only OP_QUAD has per-chunk factors (fac slots, numbered by qfac)
  std::vector<int> qops, qfac;
  int NQ = 0;
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o)
      if (tp.ops[o].code == OP_QUAD || tp.ops[o].code == OP_QLITE) {
        qops.push_back(o);
        qfac.push_back(tp.ops[o].code == OP_QUAD ? NQ++ : -1);
      }
  const int QT = (int)toff->size();
  for (int o : qops) toff->push_back(tp.ops[o].table);
  const int NO = tp.nbits - C;
  const QuadLayout QL = quad_layout(C, M, NO), QL0 = quad_layout(C, M, 0);
  // per OP_QUAD and stage: b_l (C), b0, then the products of b over the lane
  // thread bits (32 entries) and over the warp thread bits times b0
  const int FS = C + 1 + 32 + (1 << std::max(0, C - M - 5));
  if ((NQ || !qops.empty()) && (NO > 32 || C + 1 > 32 || tp.xbits)) return false;
  int ng = 0, st = 0;
  if (tma_smem_bytes(C, M, &ng, &st, tp.smax) < 0) return false;
  // registers: 4 per complex entry, 2^M entries per table; one table for
  // 16-amplitude threads, two for 8-amplitude threads
  const char* hz = getenv("QK_JIT_HOIST");
  // (none for 512-thread groups: 120 registers per thread leave no room)
  const int hoist = (variant & 1) ? 0
                                  : std::min<int>((int)toff->size(),
                                                  hz ? atoi(hz) : ((1 << (C - M)) * ng > 256 || M == 5 ? 0 : (M == 4 ? 1 : 2)));
  // hoist the first `hoist` tables that have no per-chunk (outer-bit) term
  // and load the first `early` per-chunk tables at the top of the chunk
  // iteration, so their L2 latency overlaps the stage wait and earlier phases
  std::vector<char> hoisted, early;
  {
    const char* ez = getenv("QK_JIT_EARLY");
    int left = hoist, eleft = ez ? atoi(ez) : 0;
    for (int ph = 0; ph < tp.nphases; ++ph)
      for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o)
        if (tp.ops[o].code == OP_DIAG) {
          const bool h = left > 0 && tp.ops[o].nco == 0;
          const bool e = !h && eleft > 0 && tp.ops[o].nco > 0;
          hoisted.push_back(h);
          early.push_back(e);
          if (h) --left;
          if (e) --eleft;
        }
  }
  // shared-memory slices (one consumer group only: the reload is a group barrier)
  std::vector<int> slices = ng == 1 ? slice_plan(tp, st) : std::vector<int>();
  slices.resize(hoisted.size(), 0);
  std::vector<int> slice_off(slices.size(), 0);
  uint64_t smask = 0;
  {
    int off = 0, t = 0;
    for (int ph = 0; ph < tp.nphases; ++ph)
      for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) {
        const TOp& op = tp.ops[o];
        if (op.code != OP_DIAG) continue;
        if (hoisted[t] || early[t]) slices[t] = 0;
        slice_off[t] = off;
        off += slices[t];
        if (slices[t])
          for (int k = 0; k < op.nco; ++k) smask |= 1ull << op.co_k[k];
        ++t;
      }
  }
  std::ostringstream ear;  // per-iteration early table loads
  for (size_t t = 0; t < hoisted.size(); ++t)
    if (hoisted[t]) pro << "  double2 tv" << t << "[" << NA << "];\n";
  // OP_QUAD / OP_QLITE: a thread's chunk-invariant factors (w or E, and the
  // active slots' v_s / e_s) stay in registers while they fit (~24 registers)
  std::vector<char> qhoisted(qops.size(), 0);
  {
    // (measured spill-free: one OP_QUAD hoisted; with many OP_QLITE only ~8)
    // (variant bit 4 orders OP_QUAD factors, so a pass without OP_QUAD reuses
    // it for a larger budget: QFT's OP_QLITE-heavy passes, 48 registers)
    const char* qb = getenv("QK_QHOIST");
    int budget = qb ? atoi(qb) : ((int)qops.size() > NQ ? 8 : 20);
    if (!qb && !NQ && !qops.empty() && (variant & 4)) budget = 48;
    for (size_t q = 0; q < qops.size(); ++q) {
      const TOp& op = tp.ops[qops[q]];
      const int act = op.code == OP_QUAD ? M : __builtin_popcount(op.pr[0] & ((1u << M) - 1));
      const int regs = 4 * (1 + act);
      if (regs > budget) continue;
      budget -= regs;
      qhoisted[q] = 1;
      pro << "  double2 qw" << q << ", qv" << q << "[" << M << "];\n";
      // per-thread columns (qk_internal.h QuadLayout): entry k of thread tid at k * 2^T + tid
      pro << "  { const double2* qt = p.tabs + p.toff[" << QT + q << "] + " << QL.thr / 2 << " + tid;\n";
      pro << "    qw" << q << " = __ldg(qt);\n";
      for (int sl = 0; sl < M; ++sl)
        if (op.code == OP_QUAD || (op.pr[0] >> sl & 1))
          pro << "    qv" << q << "[" << sl << "] = __ldg(qt + " << (1 + sl) * (1 << (C - M)) << ");\n";
      pro << "  }\n";
    }
  }
  const int GT = 1 << T;
  const int consumers = GT * ng;
  const int rows_chunk = 1 << (C - 3);
  b << "    double2 v[" << NA << "];\n";
  // layouts[k]: the smem image phase k reads (0: TMA SWIZZLE_128B)
  std::vector<Layout> layouts(tp.nphases);
  layouts[0] = (tp.lazy && tp.rowbits == 2) ? sw64_layout(C) : sw128_layout(C);
  // keep the previous layout when the next phase's lanes are conflict-free
  // under it too: an unchanged layout needs no barrier between a phase's
  // reads and its writes
  for (int ph = 1; ph < tp.nphases; ++ph) {
    const Layout& prev = layouts[ph - 1];
    const uint8_t* rl = tp.ph[ph].tpos;
    if (getenv("QK_JIT_SW128") || indep3(prev[rl[0]], prev[rl[1]], prev[rl[2]])) layouts[ph] = prev;
    else layouts[ph] = choose_layout(C, tp.ph[ph - 1].tpos, rl);
  }
  // Cluster-exchange store (xbits = X > 0): 2^X CTAs of a cluster hold the
  // 2^X chunks of one supertile (cluster rank = the X spectator qubits). The
  // last phase writes its chunk back to shared memory; after a cluster-wide
  // `ready`, CTA b gathers the amplitudes whose X highest-destination chunk
  // bits equal b from all 2^X CTAs (ld.shared::cluster) and stores them with
  // the spectators on destination bits 0..X-1, i.e. whole 2^X-amplitude runs.
  const int X = tp.xbits, NR = 1 << X;
  std::vector<int> gb, jl, tj, rj;  // gather / lane / thread / register chunk positions
  Layout lf;
  if (X) {
    if (T < 2 + X || X > 4) return false;
    std::vector<int> ord;
    for (int q = 0; q < C; ++q) ord.push_back(q);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) { return tp.dpos[a] < tp.dpos[c]; });
    gb.assign(ord.end() - X, ord.end());
    jl.assign(ord.begin(), ord.begin() + 2);
    tj.assign(ord.begin() + 2, ord.begin() + 2 + (T - 2 - X));
    rj.assign(ord.begin() + 2 + (T - 2 - X), ord.end() - X);
    const uint8_t rl[3] = {(uint8_t)jl[0], (uint8_t)jl[1], (uint8_t)(tj.empty() ? rj[0] : tj[0])};
    const Layout& ll = layouts[tp.nphases - 1];
    lf = indep3(ll[rl[0]], ll[rl[1]], ll[rl[2]]) ? ll : choose_layout(C, tp.ph[tp.nphases - 1].tpos, rl);
  }
  // Variant bit 8: TMA-store epilogue (lazy in-place passes). The last phase
  // writes its amplitudes into the stage at their destination tile positions
  // (the TMA image layout); the producer stores the image with the same boxes
  // it loaded and waits for the TMA unit to have read it before it refills the
  // stage. The consumers issue no global stores.
  std::vector<int> Dm(C, -1);  // tile position -> destination tile position
  bool tstore = (variant & 8) && tp.lazy && !tp.xbits && tp.permuted && !getenv("QK_NO_TSTORE");
  if (tstore)
    for (int x = 0; x < C && tstore; ++x) {
      for (int k = 0; k < C; ++k)
        if (tp.tbit[k] == tp.dpos[x]) Dm[x] = k;
      tstore = Dm[x] >= 0;
    }
  if ((variant & 8) && !tstore) return false;
  auto dmap = [&](uint32_t pos) {
    uint32_t d = 0;
    for (int x = 0; x < C; ++x)
      if (pos >> x & 1) d |= 1u << Dm[x];
    return d;
  };
  int tab_i = 0;
  const int exp_skip = getenv("QK_EXP_SKIP") ? atoi(getenv("QK_EXP_SKIP")) : 0;
  for (int ph = 0; ph < tp.nphases; ++ph) {
    const TPhase& D = tp.ph[ph];
    const bool last = ph + 1 == tp.nphases;
    b << "    {  // phase " << ph << "\n";
    emit_bits(b, "lt", "tid", D.tpos, T);
    const Layout& rdl = layouts[ph];
    emit_lay_base(b, "lr", rdl, D.tpos, T);
    for (int j = 0; j < NA; ++j) b << "    v[" << j << "] = sm[lr ^ " << lay(rdl, D.rloc[j]) << "u];\n";
    if (last) b << "    (void)0;\n";
    for (int o = D.op_begin; o < D.op_end; ++o) {
      const TOp& op = tp.ops[o];
      // dev attribution only (wrong results): QK_EXP_SKIP bit 1 drops
      // OP_QUAD/OP_QLITE, bit 2 one-qubit steps, bit 4 tables and scales
      if (exp_skip && (((exp_skip & 1) && (op.code == OP_QUAD || op.code == OP_QLITE)) ||
                       ((exp_skip & 2) && op.code == STEP_1Q) ||
                       ((exp_skip & 4) && (op.code == OP_DIAG || op.code == OP_SCALE)))) {
        if (op.code == OP_DIAG) ++tab_i;
        continue;
      }
      // quadratic table group: consecutive eligible tables of this phase
      // (not hoisted / early / sliced) applied as one factor per amplitude
      if ((variant & 2) && quad && op.code == OP_DIAG && o < (int)quad->size() && (*quad)[o].ok &&
          !hoisted[tab_i] && !early[tab_i] && !(slices[tab_i] > 0)) {
        int o2 = o, ti2 = tab_i;
        while (o2 < D.op_end && tp.ops[o2].code == OP_DIAG && (*quad)[o2].ok && !hoisted[ti2] && !early[ti2] &&
               !(slices[ti2] > 0)) {
          ++o2;
          ++ti2;
        }
        // slots of the group: register slot s is in table t's support when pr[1 << s] != 0
        uint32_t gslots = 0;
        for (int oo = o; oo < o2; ++oo)
          for (int sl = 0; sl < M; ++sl)
            if (tp.ops[oo].pr[1 << sl]) gslots |= 1u << sl;
        b << "    {  // quadratic table group (ops " << o << ".." << o2 - 1 << ")\n";
        b << "      double2 F0";
        for (int sl = 0; sl < M; ++sl)
          if (gslots >> sl & 1) b << ", G" << sl;
        b << ";\n";
        uint32_t gseen = 0;
        for (int oo = o; oo < o2; ++oo, ++tab_i) {
          const TOp& q = tp.ops[oo];
          b << "      { const double2* tb = p.tabs + p.toff[" << tab_i << "];\n";
          b << "        const u32 pt = 0u";
          for (int k = 0; k < T; ++k)
            if (q.tcontrib[k]) b << " | (((tid >> " << k << ") & 1u) * " << q.tcontrib[k] << "u)";
          for (int k = 0; k < q.nco; ++k)
            b << " | ((u32)((chunk >> " << (int)q.co_k[k] << ") & 1ull) * " << q.co_v[k] << "u)";
          b << ";\n        const double2 a0 = __ldg(tb + pt);\n";
          b << "        " << (oo == o ? "F0 = a0;" : "F0 = cm(F0, a0);") << "\n";
          const double inv2 = (*quad)[oo].inv2;
          int ci_inv = -1;
          if (inv2 != 1.0) {
            ci_inv = (int)coef->size();
            coef->push_back(inv2);
          }
          for (int sl = 0; sl < M; ++sl) {
            if (!q.pr[1 << sl]) continue;
            b << "        { const double2 as = __ldg(tb + (pt | " << q.pr[1 << sl] << "u));\n";
            // as * conj(a0)
            b << "          double2 r = make_double2(fma(as.x, a0.x, as.y * a0.y), fma(as.y, a0.x, -as.x * a0.y));\n";
            if (ci_inv >= 0) b << "          r.x *= p.coef[" << ci_inv << "]; r.y *= p.coef[" << ci_inv << "];\n";
            b << "          " << ((gseen >> sl & 1) ? "G" + std::to_string(sl) + " = cm(G" + std::to_string(sl) + ", r);"
                                                  : "G" + std::to_string(sl) + " = r;")
              << " }\n";
            gseen |= 1u << sl;
          }
          b << "      }\n";
        }
        // pair factors of the group: product over its tables
        double P[16][2];
        for (int a = 0; a < 16; ++a) P[a][0] = 1.0, P[a][1] = 0.0;
        for (int oo = o; oo < o2; ++oo)
          for (int a = 0; a < 16; ++a) {
            const double re = P[a][0] * (*quad)[oo].pf[a][0] - P[a][1] * (*quad)[oo].pf[a][1];
            const double im = P[a][0] * (*quad)[oo].pf[a][1] + P[a][1] * (*quad)[oo].pf[a][0];
            if ((*quad)[oo].pf[a][0] != 0.0 || (*quad)[oo].pf[a][1] != 0.0) P[a][0] = re, P[a][1] = im;
          }
        for (int j = 0; j < NA; ++j) {
          // f_j = F0 * prod_{s in j} G_s * prod_{s < s' in j} pf[s][s']
          std::string f = "F0";
          double pr = 1.0, pi = 0.0;
          for (int sa = 0; sa < M; ++sa) {
            if (!(j >> sa & 1)) continue;
            if (gslots >> sa & 1) f = "cm(" + f + ", G" + std::to_string(sa) + ")";
            for (int sb2 = sa + 1; sb2 < M; ++sb2)
              if (j >> sb2 & 1) {
                const double re = pr * P[sa * 4 + sb2][0] - pi * P[sa * 4 + sb2][1];
                const double im = pr * P[sa * 4 + sb2][1] + pi * P[sa * 4 + sb2][0];
                pr = re;
                pi = im;
              }
          }
          if (pr != 1.0 || pi != 0.0) {
            const int ci = (int)coef->size();
            coef->push_back(pr);
            coef->push_back(pi);
            f = "cm(" + f + ", make_double2(p.coef[" + std::to_string(ci) + "], p.coef[" + std::to_string(ci + 1) + "]))";
          }
          b << "      v[" << j << "] = cm(v[" << j << "], " << f << ");\n";
        }
        b << "    }\n";
        o = o2 - 1;
        continue;
      }
      switch (op.code) {
        case STEP_1Q:
          for (int s = 0; s < M; ++s) {
            const int k = op.st[s];
            if (!k) continue;
            SlotCache cache;
            for (int j = 0; j < NA; ++j) {
              if (j & (1 << s)) continue;
              const int jj = j | (1 << s);
              if (k == 1) b << "    hb(v[" << j << "], v[" << jj << "]);\n";
              else if (k == 2) b << "    xb(v[" << j << "], v[" << jj << "]);\n";
              else emit_mat(b, j, jj, tp.coef + op.cf[s], coef, &cache);
            }
          }
          break;
        case OP_DIAG: {
          // The table index is chunk-local: a thread reads the same 2^M
          // entries for every chunk, so the first `hoist` tables are loaded
          // once before the chunk loop and stay in registers.
          const int ti = tab_i++;
          const bool hz = hoisted[ti], ez = early[ti];
          if (slices[ti] > 0) {
            // this chunk's slice sits in shared memory (reloaded when the chunk's table bits change)
            b << "    { const double2* tb = sl + " << slice_off[ti] << ";\n";
            b << "      const u32 pt = 0u";
            for (int k = 0; k < T; ++k)
              if (op.tcontrib[k]) b << " | (((tid >> " << k << ") & 1u) * " << op.tcontrib[k] << "u)";
            b << ";\n";
            for (int j = 0; j < NA; ++j)
              if (!((op.unit >> j) & 1)) b << "      v[" << j << "] = cm(v[" << j << "], tb[pt | " << op.pr[j] << "u]);\n";
            b << "    }\n";
            break;
          }
          std::ostringstream& dst = hz ? pro : (ez ? ear : b);
          const std::string ind = hz ? "  " : "    ";
          if (ez) ear << "    double2 te" << ti << "[" << NA << "];\n";
          dst << ind << "{ const double2* tb = p.tabs + p.toff[" << ti << "];\n";
          dst << ind << "  const u32 pt = 0u";
          for (int k = 0; k < T; ++k)
            if (op.tcontrib[k]) dst << " | (((tid >> " << k << ") & 1u) * " << op.tcontrib[k] << "u)";
          for (int k = 0; k < op.nco; ++k)  // folded diagonal gates on bits outside the chunk
            dst << " | ((u32)((chunk >> " << (int)op.co_k[k] << ") & 1ull) * " << op.co_v[k] << "u)";
          dst << ";\n";
          // entries that are exactly 1 for every thread and chunk (op.unit) are skipped
          auto live = [&](int j) { return !((op.unit >> j) & 1); };
          if (hz) {
            for (int j = 0; j < NA; ++j)
              if (live(j)) pro << "    tv" << ti << "[" << j << "] = __ldg(tb + (pt | " << op.pr[j] << "u));\n";
            pro << "  }\n";
            for (int j = 0; j < NA; ++j)
              if (live(j)) b << "    v[" << j << "] = cm(v[" << j << "], tv" << ti << "[" << j << "]);\n";
          } else if (ez) {
            for (int j = 0; j < NA; ++j)
              if (live(j)) ear << "      te" << ti << "[" << j << "] = __ldg(tb + (pt | " << op.pr[j] << "u));\n";
            ear << "    }\n";
            for (int j = 0; j < NA; ++j)
              if (live(j)) b << "    v[" << j << "] = cm(v[" << j << "], te" << ti << "[" << j << "]);\n";
          } else {
            for (int j = 0; j < NA; ++j)
              if (live(j)) b << "      v[" << j << "] = cm(v[" << j << "], __ldg(tb + (pt | " << op.pr[j] << "u)));\n";
            b << "    }\n";
          }
          break;
        }
        case OP_CX: {
          const int r = op.r0;
          if (op.creg) {
            for (int j = 0; j < NA; ++j)
              if (!(j & (1 << r)) && ((j >> op.r1) & 1)) b << "    xb(v[" << j << "], v[" << (j | (1 << r)) << "]);\n";
          } else {
            b << "    if ((lt >> " << op.ctrl << ") & 1u) {\n";
            for (int j = 0; j < NA; ++j)
              if (!(j & (1 << r))) b << "      xb(v[" << j << "], v[" << (j | (1 << r)) << "]);\n";
            b << "    }\n";
          }
          break;
        }
        case OP_SWAP:
          for (int j = 0; j < NA; ++j)
            if (((j >> op.r0) & 1) && !((j >> op.r1) & 1))
              b << "    xb(v[" << j << "], v[" << (j ^ (1 << op.r0) ^ (1 << op.r1)) << "]);\n";
          break;
        case OP_QLITE: {
          // E(tid) prod_{active s in j} e_s(tid), times pj[j] where it is not 1
          int q = 0;
          while (qops[q] != o) ++q;
          const uint32_t act = op.pr[0] & ((1u << M) - 1), pjm = op.pr[1] | ((uint32_t)op.pr[3] << 16);
          b << "    { const double2* qd = p.tabs + p.toff[" << QT + q << "];\n";
          // the pj constants: kernel parameters when the planner passed them
          // (uniform over threads and chunks), else loads from the op's data
          const QuadOp* qk = (quad && o < (int)quad->size() && (*quad)[o].npj == NA) ? &(*quad)[o] : nullptr;
          auto pjv = [&](int jj) -> std::string {
            if (!qk) return "__ldg(qd + " + std::to_string(QL0.pj / 2 + jj) + ")";
            const int ci = (int)coef->size();
            coef->push_back(qk->pj[jj][0]);
            coef->push_back(qk->pj[jj][1]);
            return "make_double2(p.coef[" + std::to_string(ci) + "], p.coef[" + std::to_string(ci + 1) + "])";
          };
          if (op.pr[2] == 1) {  // constants per register amplitude
            for (int jj = 0; jj < NA; ++jj)
              if (pjm >> jj & 1) b << "      v[" << jj << "] = cm(v[" << jj << "], " << pjv(jj) << ");\n";
            b << "    }\n";
            break;
          }
          const bool e_one = op.pr[2] == 2;
          if (e_one) {
            for (int sl = 0; sl < M; ++sl)
              if (act >> sl & 1) {
                if (qhoisted[q]) b << "      const double2 e" << sl << " = qv" << q << "[" << sl << "];\n";
                else b << "      const double2 e" << sl << " = __ldg(qd + " << QL0.thr / 2 + (1 + sl) * (1 << (C - M)) << " + tid);\n";
              }
          } else if (qhoisted[q]) {
            b << "      const double2 E = qw" << q << ";\n";
            for (int sl = 0; sl < M; ++sl)
              if (act >> sl & 1) b << "      const double2 e" << sl << " = qv" << q << "[" << sl << "];\n";
          } else {
            b << "      const double2* qt = qd + " << QL0.thr / 2 << " + tid;\n";
            b << "      const double2 E = __ldg(qt);\n";
            for (int sl = 0; sl < M; ++sl)
              if (act >> sl & 1) b << "      const double2 e" << sl << " = __ldg(qt + " << (1 + sl) * (1 << (C - M)) << ");\n";
          }
          // partial products over the active slots, depth-first ("" = exactly 1)
          std::function<void(int, int, const std::string&)> visit = [&](int j, int bit, const std::string& f) {
            if (bit < 0) {
              // every amplitude whose active bits are j (the inactive slots vary freely)
              for (int jj = 0; jj < NA; ++jj) {
                if ((uint32_t)(jj & (int)act) != (uint32_t)j) continue;
                std::string m;
                if (pjm >> jj & 1) {
                  const std::string pv = pjv(jj);
                  m = f.empty() ? pv : "cm(" + f + ", " + pv + ")";
                }
                else m = f;
                if (!m.empty()) b << "      v[" << jj << "] = cm(v[" << jj << "], " << m << ");\n";
              }
              return;
            }
            if (!(act >> bit & 1)) {
              visit(j, bit - 1, f);
              return;
            }
            visit(j, bit - 1, f);
            const std::string g = "F" + std::to_string(bit);
            b << "      { const double2 " << g << " = "
              << (f.empty() ? "e" + std::to_string(bit) : "cm(" + f + ", e" + std::to_string(bit) + ")") << ";\n";
            visit(j | (1 << bit), bit - 1, g);
            b << "      }\n";
          };
          visit(0, M - 1, e_one ? "" : "E");
          b << "    }\n";
          break;
        }
        case OP_QUAD: {
          // b0 w prod_{thread bits set} b_l, then prod_{s in j} b_R(s) v_s and pj[j]
          int q = 0;
          while (qops[q] != o) ++q;
          const int qf = qfac[q];
          int R[kMaxTM];
          for (int sl = 0; sl < M; ++sl) R[sl] = __builtin_ctz(D.rloc[1 << sl]);
          b << "    { const double2* fq = fac + ((u32)s * " << NQ << "u + " << qf << "u) * " << FS << "u;\n";
          b << "      const double2* qd = p.tabs + p.toff[" << QT + q << "];\n";
          b << "      const double2 Bt = cm(fq[" << C + 1 << " + (tid & 31u)], fq[" << C + 33 << " + (tid >> 5)]);\n";
          if (qhoisted[q]) {
            b << "      double2 E = cm(Bt, qw" << q << ");\n";
          } else {
            b << "      const double2* qt = qd + " << QL.thr / 2 << " + tid;\n";
            b << "      double2 E = cm(Bt, __ldg(qt));\n";
          }
          for (int sl = 0; sl < M; ++sl) {
            if (qhoisted[q]) b << "      const double2 e" << sl << " = cm(fq[" << R[sl] << "], qv" << q << "[" << sl << "]);\n";
            else b << "      const double2 e" << sl << " = cm(fq[" << R[sl] << "], __ldg(qt + " << (1 + sl) * (1 << (C - M)) << "));\n";
          }
          // depth-first over the slots: a stack of M + 1 partial products
          const QuadOp* qk = (quad && o < (int)quad->size() && (*quad)[o].npj == NA) ? &(*quad)[o] : nullptr;
          std::function<void(int, int, const std::string&)> visit = [&](int j, int bit, const std::string& f) {
            if (bit < 0) {
              if (__builtin_popcount((unsigned)j) >= 2 && qk) {
                const int ci = (int)coef->size();
                coef->push_back(qk->pj[j][0]);
                coef->push_back(qk->pj[j][1]);
                if (qk->pj[j][0] == 1.0 && qk->pj[j][1] == 0.0)
                  b << "      v[" << j << "] = cm(v[" << j << "], " << f << ");\n";
                else
                  b << "      v[" << j << "] = cm(v[" << j << "], cm(" << f << ", make_double2(p.coef[" << ci << "], p.coef["
                    << ci + 1 << "])));\n";
              } else if (__builtin_popcount((unsigned)j) >= 2)
                b << "      v[" << j << "] = cm(v[" << j << "], cm(" << f << ", __ldg(qd + " << QL.pj / 2 + j << ")));\n";
              else
                b << "      v[" << j << "] = cm(v[" << j << "], " << f << ");\n";
              return;
            }
            visit(j, bit - 1, f);
            const std::string g = "F" + std::to_string(bit);
            b << "      { const double2 " << g << " = cm(" << f << ", e" << bit << ");\n";
            visit(j | (1 << bit), bit - 1, g);
            b << "      }\n";
          };
          visit(0, M - 1, "E");
          b << "    }\n";
          break;
        }
        case OP_SCALE: {
          const int ci = (int)coef->size();
          coef->push_back(tp.coef[op.coef]);
          coef->push_back(tp.coef[op.coef + 1]);
          if (tp.coef[op.coef + 1] == 0.0) {
            b << "    { const double sc = p.coef[" << ci << "];\n";
            for (int j = 0; j < NA; ++j) b << "      v[" << j << "].x *= sc; v[" << j << "].y *= sc;\n";
          } else {
            b << "    { const double2 sc = make_double2(p.coef[" << ci << "], p.coef[" << ci + 1 << "]);\n";
            for (int j = 0; j < NA; ++j) b << "      v[" << j << "] = cm(v[" << j << "], sc);\n";
          }
          b << "    }\n";
          break;
        }
        default:
          return false;
      }
    }
    if (last && X) {
      // a thread rewrites its own amplitudes, but at other slots when the
      // layout changes: every read of the phase must land first
      if (lf != rdl) b << "    gbar(bar_id, " << GT << ");\n";
      emit_lay_base(b, "lw", lf, D.tpos, T);
      for (int j = 0; j < NA; ++j) b << "    sm[lw ^ " << lay(lf, D.rloc[j]) << "u] = v[" << j << "];\n";
      // generic writes of the stage must be ordered before the TMA (async
      // proxy) refill that follows the `done` exchange
      b << "    fence_async_smem();\n";
      b << "    gbar(bar_id, " << GT << ");\n";
      b << "    if (tid == 0) {\n";
      if (getenv("QK_X_FENCE")) b << "      asm volatile(\"fence.acq_rel.cluster;\" ::: \"memory\");\n";
      b << "      for (u32 q = 0; q < " << NR << "u; ++q) mbar_arrive_remote(mapa(su32(ready + s), q));\n    }\n";
      b << "    mbar_wait_cl(ready + s, round & 1u);\n";
      b << "    {\n      const u32 rr = (tid >> 2) & " << NR - 1 << "u;\n";
      b << "      const u32 rb = mapa(su32(sm), rr);\n";
      // slot and destination of the thread's base amplitude
      b << "      const u32 gs = 0u";
      for (int k = 0; k < 2; ++k) b << " ^ (((tid >> " << k << ") & 1u) * " << lay(lf, 1u << jl[k]) << "u)";
      for (size_t k = 0; k < tj.size(); ++k) b << " ^ (((tid >> " << 2 + X + k << ") & 1u) * " << lay(lf, 1u << tj[k]) << "u)";
      for (int k = 0; k < X; ++k) b << " ^ (((rank >> " << k << ") & 1u) * " << lay(lf, 1u << gb[k]) << "u)";
      b << ";\n      const u64 dst = dsup";
      for (int k = 0; k < 2; ++k) b << " | ((u64)((tid >> " << k << ") & 1u) << " << (int)tp.dpos[jl[k]] << ")";
      for (size_t k = 0; k < tj.size(); ++k) b << " | ((u64)((tid >> " << 2 + X + k << ") & 1u) << " << (int)tp.dpos[tj[k]] << ")";
      for (int k = 0; k < X; ++k) b << " | ((u64)((rr >> " << k << ") & 1u) << " << (int)tp.dpos[tp.xpos[k]] << ")";
      for (int k = 0; k < X; ++k) b << " | ((u64)((rank >> " << k << ") & 1u) << " << (int)tp.dpos[gb[k]] << ")";
      b << ";\n";
      for (int jj = 0; jj < NA; ++jj) {
        uint32_t ci = 0;
        for (int m = 0; m < M; ++m)
          if (jj >> m & 1) ci |= 1u << rj[m];
        b << "      v[" << jj << "] = ld_cl(rb + ((gs ^ " << lay(lf, ci) << "u) << 4));\n";
      }
      for (int jj = 0; jj < NA; ++jj) {
        uint64_t d = 0;
        for (int m = 0; m < M; ++m)
          if (jj >> m & 1) d |= 1ull << tp.dpos[rj[m]];
        b << "      st_cs(p.out + (dst | " << d << "ull), v[" << jj << "]);\n";
      }
      b << "    }\n    gbar(bar_id, " << GT << ");\n";
      b << "    if (tid == 0)\n      for (u32 q = 0; q < " << NR << "u; ++q) mbar_arrive_remote(mapa(su32(done + s), q));\n";
    } else if (!last) {
      const Layout& wrl = layouts[ph + 1];
      if (wrl != rdl) b << "    gbar(bar_id, " << GT << ");\n";
      emit_lay_base(b, "lw", wrl, D.tpos, T);
      for (int j = 0; j < NA; ++j) b << "    sm[lw ^ " << lay(wrl, D.rloc[j]) << "u] = v[" << j << "];\n";
      b << "    gbar(bar_id, " << GT << ");\n";
    } else if (tstore) {
      // every thread's reads of the stage are done before any final write
      b << "    gbar(bar_id, " << GT << ");\n";
      b << "    { const u32 ls = 0u";
      for (int k = 0; k < T; ++k) b << " ^ (((tid >> " << k << ") & 1u) * " << lay(layouts[0], dmap(1u << D.tpos[k])) << "u)";
      b << ";\n";
      for (int j = 0; j < NA; ++j) b << "      sm[ls ^ " << lay(layouts[0], dmap(D.rloc[j])) << "u] = v[" << j << "];\n";
      b << "    }\n";
      b << "    fence_async_smem();\n    gbar(bar_id, " << GT << ");\n";
      b << "    if (tid == 0) mbar_arrive(empty + s);\n";
      if (tp.norm)
        for (int j = 0; j < NA; ++j) b << "    nacc = fma(v[" << j << "].x, v[" << j << "].x, fma(v[" << j << "].y, v[" << j << "].y, nacc));\n";
    } else {
      b << "    fence_async_smem();\n    gbar(bar_id, " << GT << ");\n";
      b << "    if (tid == 0) mbar_arrive(empty + s);\n";
      if (tp.permuted && !(exp_skip & 8)) {  // (bit 8: contiguous store, timing only)
        b << "    u64 dst = 0ull";
        for (int k = 0; k < tp.nbits - C; ++k) b << " | (((chunk >> " << k << ") & 1ull) << " << (int)tp.dpos[C + k] << ")";
        b << ";\n";
        for (int k = 0; k < T; ++k) b << "    if ((tid >> " << k << ") & 1u) dst |= " << tp.ldst_t[k] << "ull;\n";
        b << "    double2* g = p.out + dst;\n";
        for (int j = 0; j < NA; ++j) b << "    st_cs(g + " << tp.ldst_r[j] << "ull, v[" << j << "]);\n";
      } else {
        b << "    double2* g = p.out + (chunk << " << C << ");\n";
        for (int j = 0; j < NA; ++j) b << "    st_cs(g + (lt | " << D.rloc[j] << "u), v[" << j << "]);\n";
      }
      if (tp.norm)
        for (int j = 0; j < NA; ++j) b << "    nacc = fma(v[" << j << "].x, v[" << j << "].x, fma(v[" << j << "].y, v[" << j << "].y, nacc));\n";
    }
    b << "    }\n";
  }
  std::ostringstream o;
  o << "#define QK_NTAB " << toff->size() << "\n#define QK_NCOEF " << coef->size() << "\n";
  o << kPreamble;
  if (X) {
    // supertile u: outer source bits O (ascending) <- bits of u, spectators <- rank
    std::vector<int> O;
    for (int q = C; q < tp.nbits; ++q) {
      bool sp = false;
      for (int k = 0; k < X; ++k) sp = sp || tp.xpos[k] == q;
      if (!sp) O.push_back(q);
    }
    o << "extern \"C\" __global__ void __launch_bounds__(" << 32 + consumers << ", 1) qk_jitx(const __grid_constant__ QkJitParams p) {\n"
      << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
      << "  unsigned char* base = smem_raw;\n"
      << "  const u32 stage_bytes = " << (16u << C) << "u;\n"
      << "  u64* full = (u64*)(base + " << (size_t)st * (16u << C) << "ull);\n"
      << "  u64* done = full + " << st << ";\n"
      << "  u64* ready = done + " << st << ";\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    for (int s = 0; s < " << st << "; ++s) { mbar_init(full + s, 1); mbar_init(done + s, " << NR << "); mbar_init(ready + s, " << NR << "); }\n"
      << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n"
      << "  __syncthreads();\n"
      << "  cluster_sync();\n"
      << "  const u32 rank = cl_rank();\n"
      << "  const u64 CID = cl_id(), NCL = cl_num();\n"
      << "  if (threadIdx.x < 32) {\n"
      << "    if (threadIdx.x == 0) {\n"
      << "      asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&p.map) : \"memory\");\n"
      << "      for (u64 i = 0;; ++i) {\n"
      << "        const u64 u = CID + i * NCL;\n"
      << "        if (u >= p.nchunks) break;\n"
      << "        const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
      << "        if (round > 0) { mbar_wait_cl(done + s, (round - 1) & 1u); fence_async_smem(); }\n"
      << "        mbar_expect_tx(full + s, stage_bytes);\n"
      << "        unsigned char* dst = base + (size_t)s * stage_bytes;\n"
      << "        const u64 caddr = 0ull";
    for (size_t k = 0; k < O.size(); ++k) o << " | (((u >> " << k << ") & 1ull) << " << O[k] << ")";
    for (int k = 0; k < X; ++k) o << " | ((u64)((rank >> " << k << ") & 1u) << " << (int)tp.xpos[k] << ")";
    o << ";\n        const int row0 = (int)(caddr >> 3);\n";
    for (int t = 0; t < tp.ntma; ++t)
      o << "        tma_load(dst + " << t * tp.box_rows * 128 << ", &p.map, 0, row0 + " << t * tp.box_rows << ", full + s);\n";
    o << "      }\n    }\n    __syncwarp();\n  } else {\n"
      << "  const int ct = threadIdx.x - 32;\n"
      << "  const int g = ct >> " << T << ";\n"
      << "  const u32 tid = ct & " << (GT - 1) << "u;\n"
      << pro.str()
      << "  const int bar_id = 1 + g;\n"
      << "  for (u64 i = g;; i += " << ng << ") {\n"
      << "    const u64 u = CID + i * NCL;\n"
      << "    if (u >= p.nchunks) break;\n"
      << "    const u64 dsup = 0ull";
    for (size_t k = 0; k < O.size(); ++k) o << " | (((u >> " << k << ") & 1ull) << " << (int)tp.dpos[O[k]] << ")";
    o << ";\n"
      << "    const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
      << "    double2* sm = (double2*)(base + (size_t)s * stage_bytes);\n"
      << "    mbar_wait(full + s, round & 1u);\n"
      << b.str()
      << "  }\n  }\n  cluster_sync();\n}\n";
    *src = o.str();
    return true;
  }
  // Chunk order for passes with per-chunk table terms: every CTA walks one
  // contiguous range of a counter whose high bits are the chunk bits the
  // tables read, so a CTA keeps the same table slices (and their L1 lines)
  // over long stretches instead of switching slices every chunk.
  const uint64_t tmask = table_chunk_mask(tp);
  const int nouter = tp.nbits - C;
  // (12-bit chunks only: QAOA30 0.166 -> 0.162 s, QAOA33r3 1.73 -> 1.64 s;
  // QFT30's 10-bit passes lose 4%, their CTAs then spread over more pages)
  const bool corder = tmask && C >= 12 && !getenv("QK_NO_CORDER");
  const bool pair = jit_pairs(tp);
  if (corder) {
    std::vector<int> ord;
    for (int k = 0; k < nouter; ++k)
      if (!(tmask >> k & 1)) ord.push_back(k);
    for (int k = 0; k < nouter; ++k)
      if (tmask >> k & 1) ord.push_back(k);
    o << "__device__ __forceinline__ u64 cmap(u64 c) {\n  return 0ull";
    for (size_t j = 0; j < ord.size(); ++j) o << " | (((c >> " << j << ") & 1ull) << " << ord[j] << ")";
    o << ";\n}\n";
  }
  // counter -> chunk for iteration i of this CTA; `nxt` = the chunk st iterations later
  // (split sub-launches, the passes next to an overlapped exchange, walk the
  // grid-stride order over their part of the chunks)
  auto chunk_of = [&](const char* iv) {
    std::ostringstream c;
    if (pair) {  // pair u = cluster + i * clusters; the cluster rank is chunk bit 0
      c << "(p.split ? qk_insert(2ull * (CID + " << iv << " * NCL) + RK, p.split) : (2ull * (CID + " << iv
        << " * NCL) + RK))";
      return c.str();
    }
    c << "(p.split ? qk_insert(blockIdx.x + " << iv << " * G, p.split) : ";
    if (corder) c << "cmap(blockIdx.x * PER + " << iv << "))";
    else c << "(blockIdx.x + " << iv << " * G))";
    return c.str();
  };
  auto chunk_ok = [&](const char* iv) {
    std::ostringstream c;
    if (pair) {
      c << "(2ull * (CID + " << iv << " * NCL) < p.nchunks)";
      return c.str();
    }
    if (corder)
      c << "(p.split ? (blockIdx.x + " << iv << " * G < p.nchunks) : (" << iv << " < PER && blockIdx.x * PER + " << iv
        << " < p.nchunks))";
    else c << "(blockIdx.x + " << iv << " * G < p.nchunks)";
    return c.str();
  };
  size_t fac_off = 0;
  {
    size_t planned = 0;
    for (int e : slice_plan(tp, st)) planned += (size_t)e * 16;
    fac_off = (size_t)st * (16u << C) + 16 * st + planned + (tp.norm ? 16 * 32 * 8 : 0);
  }
  const size_t pair_off = fac_off + (size_t)NQ * FS * 16 * (st + 1);
  // (dev: QK_JIT_MAXNREG caps registers instead of the launch bounds; note
  // that 17 warps allocate like 20, so 544 threads fit only up to 96)
  const int maxreg = getenv("QK_JIT_MAXNREG") ? atoi(getenv("QK_JIT_MAXNREG")) : 0;
  if (maxreg > 0)
    o << "extern \"C\" __global__ void __maxnreg__(" << maxreg << ") qk_jit(const __grid_constant__ QkJitParams p) {\n";
  else
    o << "extern \"C\" __global__ void __launch_bounds__(" << 32 + consumers << ", 1) qk_jit(const __grid_constant__ QkJitParams p) {\n";
  o
    << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
    << "  unsigned char* base = smem_raw;\n"
    << "  const u32 stage_bytes = " << (16u << C) << "u;\n"
    << "  u64* full = (u64*)(base + " << (size_t)st * (16u << C) << "ull);\n"
    << "  u64* empty = full + " << st << ";\n";
  if (pair) o << "  u64* pairb = (u64*)(base + " << pair_off << "ull);\n";
  o << "  if (threadIdx.x == 0) {\n"
    << "    for (int s = 0; s < " << st << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n";
  if (pair) o << "    for (int s = 0; s < " << st << "; ++s) mbar_init(pairb + s, 1);\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n"
    << (pair ? "  cluster_sync();\n" : "  __syncthreads();\n")
    << "  const u64 G = gridDim.x;\n"
    << "  const u64 PER = (p.nchunks + G - 1) / G;\n"
    << "  (void)PER;\n"
    << "  double2* fac = (double2*)(base + " << fac_off << "ull);\n"
    << "  (void)fac;\n";
  if (pair) o << "  const u64 CID = cl_id(), NCL = cl_num();\n  const u32 RK = cl_rank();\n";
  if (!NQ) {
    o << "  if (threadIdx.x < 32) {\n"
      << "    if (threadIdx.x == 0) {\n"
      << "      asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&p.map) : \"memory\");\n"
      << "      for (u64 i = 0;; ++i) {\n"
      << "        if (!" << chunk_ok("i") << ") break;\n"
      << "        const u64 chunk = " << chunk_of("i") << ";\n"
      << "        const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
      << "        if (round > 0) mbar_wait(empty + s, (round - 1) & 1u);\n";
    if (tstore)
      o << "        if (round > 0) {\n          const u64 pchunk = " << chunk_of(("(i - " + std::to_string(st) + "ull)").c_str())
        << ";\n          unsigned char* srcb = base + (size_t)s * stage_bytes;\n"
        << lazy_stores(tp, "pchunk", "srcb", "          ")
        << "          asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n        }\n";
  } else {
    // OP_QUAD: the whole producer warp turns the chunk bits into the
    // per-position factors of every quadratic op in a pending slot while the
    // stage is still in use (sincos and L2 reads off the refill path), copies
    // them into the stage's slot once it is free, and lane 0 arms the stage:
    // the consumers' full-barrier wait acquires both the tile and the factors
    o << "  if (threadIdx.x < 32) {\n"
      << "    const u32 lane = threadIdx.x;\n"
      << "    if (lane == 0) asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&p.map) : \"memory\");\n"
      << "    for (u64 i = 0;; ++i) {\n"
      << "      if (!" << chunk_ok("i") << ") break;\n"
      << "      const u64 chunk = " << chunk_of("i") << ";\n"
      << "      const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
      << (variant & 4 ? "      double2* const pend = fac + (u32)s * " + std::to_string(NQ * FS) + "u;\n"
                      : "      double2* const pend = fac + " + std::to_string(st * NQ * FS) + "u;\n");
  }
  std::ostringstream fsrc;  // producer-side factors of the OP_QUAD ops
  if (NQ) {
    std::ostringstream& o = fsrc;
    for (size_t qi = 0; qi < qops.size(); ++qi) {
      if (qfac[qi] < 0) continue;
      const int q = qfac[qi];
      o << "      { const double* qd = (const double*)(p.tabs + p.toff[" << QT + (int)qi << "]);\n"
        // boo[k][k'] is 0 for k' >= k: every lane sums a full unrolled row
        << "        double t = 0.0;\n"
        << "        if (lane < " << NO << "u) {\n"
        << "          const double* row = qd + " << QL.boo << " + lane * " << NO << "u;\n"
        << "          double t0 = __ldg(qd + " << QL.ao << " + lane), t1 = 0.0;\n"
        << "#pragma unroll\n"
        << "          for (int k = 0; k < " << NO << "; k += 2) {\n"
        << "            t0 += ((chunk >> k) & 1ull) ? __ldg(row + k) : 0.0;\n"
        << "            if (k + 1 < " << NO << ") t1 += ((chunk >> (k + 1)) & 1ull) ? __ldg(row + k + 1) : 0.0;\n"
        << "          }\n"
        << "          t = ((chunk >> lane) & 1ull) ? t0 + t1 : 0.0;\n"
        << "        }\n"
        << "        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);\n"
        << "        double a = 0.0;\n"
        << "        if (lane < " << C << "u) {\n"
        << "          const double* row = qd + " << QL.bto << " + lane * " << NO << "u;\n"
        << "          double a0 = __ldg(qd + " << QL.at << " + lane), a1 = 0.0;\n"
        << "#pragma unroll\n"
        << "          for (int k = 0; k < " << NO << "; k += 2) {\n"
        << "            a0 += ((chunk >> k) & 1ull) ? __ldg(row + k) : 0.0;\n"
        << "            if (k + 1 < " << NO << ") a1 += ((chunk >> (k + 1)) & 1ull) ? __ldg(row + k + 1) : 0.0;\n"
        << "          }\n"
        << "          a = a0 + a1;\n"
        << "        } else if (lane == " << C << "u) {\n"
        << "          a = __ldg(qd + " << QL.phi0 << ") + t;\n"
        << "        }\n"
        << "        double2* fs = pend + " << q * FS << "u;\n"
        << "        if (lane <= " << C << "u) { double sn, cs; sincos(a, &sn, &cs); fs[lane] = make_double2(cs, sn); }\n"
        << "        __syncwarp();\n";
      // products over the thread bits of the phase that applies the op
      int oph = 0;
      while (!(qops[qi] >= tp.ph[oph].op_begin && qops[qi] < tp.ph[oph].op_end)) ++oph;
      const uint8_t* tpos = tp.ph[oph].tpos;
      const int TB = C - M;
      o << "        { double2 x = make_double2(1.0, 0.0);\n";
      for (int k = 0; k < 5 && k < TB; ++k)
        o << "          { const double2 f = fs[" << (int)tpos[k] << "]; const bool on = (lane >> " << k
          << ") & 1u; x = cm(x, make_double2(on ? f.x : 1.0, on ? f.y : 0.0)); }\n";
      o << "          fs[" << C + 1 << " + lane] = x; }\n";
      o << "        if (lane < " << (1 << std::max(0, TB - 5)) << "u) { double2 y = fs[" << C << "];\n";
      for (int k = 5; k < TB; ++k)
        o << "          { const double2 f = fs[" << (int)tpos[k] << "]; const bool on = (lane >> " << k - 5
          << ") & 1u; y = cm(y, make_double2(on ? f.x : 1.0, on ? f.y : 0.0)); }\n";
      o << "          fs[" << C + 33 << " + lane] = y; }\n"
        << "      }\n";
    }
  }
  std::string tstore_src;
  if (tstore && NQ)
    tstore_src = "      if (lane == 0 && round > 0) {\n        const u64 pchunk = " +
                 chunk_of(("(i - " + std::to_string(st) + "ull)").c_str()) +
                 ";\n        unsigned char* srcb = base + (size_t)s * stage_bytes;\n" +
                 lazy_stores(tp, "pchunk", "srcb", "        ") +
                 "        asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n      }\n";
  if (NQ && (variant & 4))  // variant bit 4: factors straight into the stage's slot after the wait
    o << "      if (lane == 0 && round > 0) mbar_wait(empty + s, (round - 1) & 1u);\n"
      << tstore_src
      << "      __syncwarp();\n" << fsrc.str() << "      __syncwarp();\n"
      << "      if (lane == 0) {\n";
  else if (NQ)
    o << fsrc.str() << "      if (lane == 0 && round > 0) mbar_wait(empty + s, (round - 1) & 1u);\n"
      << tstore_src
      << "      __syncwarp();\n"
      << "      for (u32 e = lane; e < " << NQ * FS << "u; e += 32u) fac[(u32)s * " << NQ * FS << "u + e] = pend[e];\n"
      << "      __syncwarp();\n"
      << "      if (lane == 0) {\n";
  if (pair)
    o << "        mbar_arrive_remote(mapa(su32(pairb + s), RK ^ 1u));\n"
      << "        mbar_wait(pairb + s, round & 1u);\n";
  o << "        mbar_expect_tx(full + s, stage_bytes);\n"
    << "        unsigned char* dst = base + (size_t)s * stage_bytes;\n";
  const char* pfe = getenv("QK_JIT_PREFETCH");
  if (tp.lazy) {
    // strided tile (qk_internal.h tile_dims): one N-D box per value of the
    // iterated top tile bits; coordinates from the chunk's outer bits
    o << lazy_loads(tp, "chunk", "dst", false, "        ");
    // L2 prefetch of the refill only while the tile spans few 2-MiB pages:
    // with rows on up to 1024 pages the extra translations cost more than the
    // prefetch hides (H33's 1024-page pass: 88 -> 65 ms without it; U33's
    // 8-page 13-bit pass: 64 ms with it, 68 ms without). 64-B-row tiles
    // never gain (H33's 8-page one: 50 ms without, 62 ms with).
    int pagebits = 0;
    for (int x = 0; x < C; ++x) pagebits += tp.tbit[x] >= 17;
    if (pfe ? atoi(pfe) != 0 : (st <= 2 && pagebits <= 4 && tp.rowbits == 3)) {
      const std::string ni = "(i + " + std::to_string(st) + "ull)";
      o << "        if (" << chunk_ok(ni.c_str()) << ") {\n"
        << "          const u64 nchunk = " << chunk_of(ni.c_str()) << ";\n"
        << lazy_loads(tp, "nchunk", nullptr, true, "          ") << "        }\n";
    }
  } else {
  o << "        const int row0 = (int)(chunk * " << rows_chunk << "ull);\n";
  for (int t = 0; t < tp.ntma; ++t)
    o << "        tma_load(dst + " << t * tp.box_rows * 128 << ", &p.map, 0, row0 + " << t * tp.box_rows << ", full + s);\n";
  }
  // with a shallow ring, pull the chunk that will refill this stage into L2
  // now, so its load hits L2 when the stage is released
  if (!tp.lazy && (pfe ? atoi(pfe) != 0 : st <= 2)) {
    const std::string ni = "(i + " + std::to_string(st) + "ull)";
    o << "        if (" << chunk_ok(ni.c_str()) << ") {\n"
      << "          const int prow = (int)((" << chunk_of(ni.c_str()) << ") * " << rows_chunk << "ull);\n";
    for (int t = 0; t < tp.ntma; ++t)
      o << "          tma_prefetch(&p.map, 0, prow + " << t * tp.box_rows << ");\n";
    o << "        }\n";
  }
  // TMA-store epilogue: after the last refill the final uses of the stages
  // still hold results; store them and wait for the writes
  std::string drain;
  if (tstore)
    drain = std::string("    { u64 I = 0;\n      while (") + chunk_ok("I") + ") ++I;\n" +
            "      for (u64 j = I > " + std::to_string(st) + "ull ? I - " + std::to_string(st) + "ull : 0ull; j < I; ++j) {\n" +
            "        const int s = (int)(j % " + std::to_string(st) + "); const u32 round = (u32)(j / " + std::to_string(st) + ");\n" +
            "        mbar_wait(empty + s, round & 1u);\n" +
            "        const u64 pchunk = " + chunk_of("j") + ";\n" +
            "        unsigned char* srcb = base + (size_t)s * stage_bytes;\n" + lazy_stores(tp, "pchunk", "srcb", "        ") +
            "      }\n      asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n    }\n";
  if (NQ)
    o << "      }\n    }\n" << (drain.empty() ? "" : "    if (lane == 0)\n" + drain) << "    return;\n  }\n";
  else
    o << "      }\n" << drain << "    }\n    return;\n  }\n";
  o << "  const int ct = threadIdx.x - 32;\n"
    << "  const int g = ct >> " << T << ";\n"
    << "  const u32 tid = ct & " << (GT - 1) << "u;\n"
    << pro.str()
    << "  const int bar_id = 1 + g;\n";
  if (smask) {
    o << "  double2* sl = (double2*)(base + " << (size_t)st * (16u << C) + 16 * st << "ull);\n"
      << "  u64 skey = ~0ull;\n";
  }
  if (tp.norm) o << "  double nacc = 0.0;\n";
  o << "  for (u64 i = g;; i += " << ng << ") {\n"
    << "    if (!" << chunk_ok("i") << ") break;\n"
    << "    const u64 chunk = " << chunk_of("i") << ";\n"
    << "    const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
    << "    double2* sm = (double2*)(base + (size_t)s * stage_bytes);\n";
  if (smask) {
    // every thread passed the previous chunk's last barrier after its table reads
    o << "    if ((chunk & " << smask << "ull) != skey) {\n";
    int t = 0;
    for (int ph = 0; ph < tp.nphases; ++ph)
      for (int o2 = tp.ph[ph].op_begin; o2 < tp.ph[ph].op_end; ++o2) {
        const TOp& op = tp.ops[o2];
        if (op.code != OP_DIAG) continue;
        if (slices[t] > 0) {
          o << "      { const double2* src = p.tabs + p.toff[" << t << "] + (0ull";
          for (int k = 0; k < op.nco; ++k)
            o << " | ((u64)((chunk >> " << (int)op.co_k[k] << ") & 1ull) * " << op.co_v[k] << "ull)";
          o << ");\n        for (u32 e = tid; e < " << slices[t] << "u; e += " << GT << "u) sl[" << slice_off[t]
            << " + e] = __ldg(src + e); }\n";
        }
        ++t;
      }
    o << "      skey = chunk & " << smask << "ull;\n      gbar(bar_id, " << GT << ");\n    }\n";
  }
  o << ear.str()
    << "    mbar_wait(full + s, round & 1u);\n"
    << b.str()
    << "  }\n";
  if (tp.norm) {
    // fused norm: per group, warp sums then the group's warps in order (deterministic)
    size_t planned = 0;
    for (int e : slice_plan(tp, st)) planned += (size_t)e * 16;
    const size_t noff = (size_t)st * (16u << C) + 16 * st + planned;
    o << "  {\n    double* red = (double*)(base + " << noff << "ull) + g * 32;\n"
      << "    double t = nacc;\n"
      << "    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);\n"
      << "    if ((tid & 31u) == 0) red[tid >> 5] = t;\n"
      << "    gbar(bar_id, " << GT << ");\n"
      << "    if (tid == 0) {\n      double sum = 0.0;\n"
      << "      for (int w = 0; w < " << std::max(1, GT / 32) << "; ++w) sum += red[w];\n"
      << "      if ((p.split >> 23) & 1ull) p.nrm[blockIdx.x * " << ng << " + g] += sum;\n"
      << "      else p.nrm[blockIdx.x * " << ng << " + g] = sum;\n    }\n  }\n";
  }
  o << "}\n";
  *src = o.str();
  return true;
}

namespace {

struct Entry {
  std::string cubin;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  bool failed = false;
};

std::mutex g_mu;
std::map<std::string, Entry*> g_cache;  // source -> compiled kernel (process-wide)

std::string cache_dir() {
  const char* e = getenv("QK_JIT_CACHE");
  if (e && *e) return e;
  const char* home = getenv("HOME");
  return std::string(home && *home ? home : "/tmp") + "/.cache/qkb200/jit";
}

void mkdirs(const std::string& p) {
  std::string cur;
  for (size_t i = 0; i < p.size(); ++i) {
    cur.push_back(p[i]);
    if (p[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
  }
  mkdir(p.c_str(), 0755);
}

std::string hash_hex(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  char buf[32];
  snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return buf;
}

bool compile_one(const std::string& src, std::string* cubin, std::string* log) {
  const std::string path = cache_dir() + "/" + hash_hex(src) + "_" + std::to_string(src.size()) + ".cubin";
  if (FILE* f = fopen(path.c_str(), "rb")) {
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    cubin->resize(n > 0 ? n : 0);
    const bool ok = n > 0 && fread(&(*cubin)[0], 1, n, f) == (size_t)n;
    fclose(f);
    if (ok) return true;
  }
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    *log = "nvrtc unavailable";
    return false;
  }
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, src.c_str(), "qk_jit.cu", 0, nullptr, nullptr)) return false;
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "-lineinfo",
                        "--extra-device-vectorization"};
  const int rc = nv.compile(prog, 5, opts);
  if (rc) {
    size_t ls = 0;
    if (nv.log_size && nv.log) {
      nv.log_size(prog, &ls);
      log->resize(ls);
      nv.log(prog, &(*log)[0]);
    }
    nv.destroy(&prog);
    return false;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  cubin->resize(n);
  nv.cubin(prog, &(*cubin)[0]);
  nv.destroy(&prog);
  mkdirs(cache_dir());
  const std::string tmp = path + ".tmp" + std::to_string((long long)getpid());
  if (FILE* f = fopen(tmp.c_str(), "wb")) {
    fwrite(cubin->data(), 1, cubin->size(), f);
    fclose(f);
    rename(tmp.c_str(), path.c_str());
  }
  return true;
}

}  // namespace

bool jit_available() { return !getenv("QK_NO_JIT") && nvrtc().ok; }

// Compile (in parallel) and load every source not yet in the cache.
// handles[i] receives an opaque kernel handle or nullptr on failure.
void jit_build(const std::vector<std::string>& srcs, std::vector<void*>* handles) {
  handles->assign(srcs.size(), nullptr);
  std::vector<size_t> todo;
  std::vector<Entry*> ents(srcs.size(), nullptr);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < srcs.size(); ++i) {
      auto it = g_cache.find(srcs[i]);
      if (it == g_cache.end()) {
        Entry* e = new Entry();
        g_cache[srcs[i]] = e;
        ents[i] = e;
        todo.push_back(i);
      } else {
        ents[i] = it->second;
      }
    }
  }
  if (!todo.empty()) {
    std::atomic<size_t> next{0};
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < std::min<size_t>(nt, todo.size()); ++t)
      pool.emplace_back([&] {
        for (size_t k; (k = next++) < todo.size();) {
          Entry* e = ents[todo[k]];
          std::string log;
          if (!compile_one(srcs[todo[k]], &e->cubin, &log)) {
            e->failed = true;
            if (getenv("QK_JIT_VERBOSE")) fprintf(stderr, "qk_jit: compile failed: %s\n", log.c_str());
          }
        }
      });
    for (auto& th : pool) th.join();
    if (getenv("QK_JIT_VERBOSE")) fprintf(stderr, "qk_jit: built %zu kernels (%zu requested)\n", todo.size(), srcs.size());
    for (size_t k : todo) {
      Entry* e = ents[k];
      if (e->failed) continue;
      if (cudaLibraryLoadData(&e->lib, e->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
          (cudaLibraryGetKernel(&e->kern, e->lib, "qk_jit") != cudaSuccess &&
           cudaLibraryGetKernel(&e->kern, e->lib, "qk_jitx") != cudaSuccess)) {
        cudaGetLastError();
        e->failed = true;
        continue;
      }
      cudaFuncSetAttribute((const void*)e->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaGetLastError();
    }
  }
  for (size_t i = 0; i < srcs.size(); ++i)
    (*handles)[i] = (ents[i] && !ents[i]->failed) ? (void*)ents[i]->kern : nullptr;
}

// Launch a JIT kernel: params blob = QkJitParams laid out by jit_params().
int jit_launch(void* kern, const void* params, int C, int M, uint64_t nchunks, int num_sms, CUstream_st* stream,
               int smax, int extra_smem, int cluster) {
  int ng = 0, st = 0;
  const int smem0 = tma_smem_bytes(C, M, &ng, &st, smax);
  if (smem0 < 0) return -1;
  const int smem = smem0 + extra_smem;
  if (smem < 0) return -1;
  const int threads = 32 + (1 << (C - M)) * ng;
  const uint64_t grid = nchunks < (uint64_t)num_sms ? nchunks : (uint64_t)num_sms;
  {  // library kernels take their function attributes per device
    static std::mutex mu;
    static std::set<std::pair<void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({kern, dev}).second) {
      cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaGetLastError();
    }
  }
  void* args[] = {const_cast<void*>(params)};
  if (cluster > 1) {
    // as many co-resident clusters as the device holds (one CTA per SM)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = reinterpret_cast<cudaStream_t>(stream);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static std::mutex mu;
    static std::map<std::tuple<void*, int, int>, int> fit;
    int dev = 0, ncl = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = fit.find({kern, dev, smem});
      if (it == fit.end()) {
        cfg.gridDim = dim3((unsigned)(num_sms / cluster * cluster));
        if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)kern, &cfg) != cudaSuccess || ncl < 1) {
          cudaGetLastError();
          ncl = num_sms / cluster / 2;
        }
        fit[{kern, dev, smem}] = ncl;
      } else {
        ncl = it->second;
      }
    }
    const uint64_t want = (nchunks + cluster - 1) / cluster;
    cfg.gridDim = dim3((unsigned)(cluster * (want < (uint64_t)ncl ? want : (uint64_t)ncl)));
    return (int)cudaLaunchKernelExC(&cfg, (const void*)kern, args);
  }
  cudaError_t e = cudaLaunchKernel((const void*)kern, dim3((unsigned)grid), dim3(threads), args, smem,
                                   reinterpret_cast<cudaStream_t>(stream));
  return (int)e;
}

// Launch a cluster-exchange pass: 2^xbits CTAs per cluster, as many
// resident clusters as fit (persistent over the nsuper supertiles).
int jit_launch_x(void* kern, const void* params, int C, int M, int xbits, uint64_t nsuper, CUstream_st* stream) {
  int ng = 0, st = 0;
  const int smem0 = tma_smem_bytes(C, M, &ng, &st);
  if (smem0 < 0) return -1;
  const int smem = smem0 + 8 * st;  // + the `ready` barriers
  const int threads = 32 + (1 << (C - M)) * ng;
  const int csize = 1 << xbits;
  static std::mutex mu;
  static std::map<std::pair<void*, int>, int> max_clusters;
  int ncl = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(kern, smem);
    auto it = max_clusters.find(key);
    if (it == max_clusters.end()) {
      if (csize > 8) cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csize;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(csize * 64);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      if (getenv("QK_JIT_VERBOSE")) fprintf(stderr, "qk_jit: cluster %d: %d resident clusters\n", csize, n);
      it = max_clusters.emplace(key, n).first;
    }
    ncl = it->second;
  }
  if (ncl <= 0) return (int)cudaErrorLaunchOutOfResources;
  const uint64_t grid_cl = nsuper < (uint64_t)ncl ? nsuper : (uint64_t)ncl;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(grid_cl * csize));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<void*>(params)};
  return (int)cudaLaunchKernelExC(&cfg, (const void*)kern, args);
}

}  // namespace qk
