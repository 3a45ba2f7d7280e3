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

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
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
  long long toff[QK_NTAB + 1];
  double coef[QK_NCOEF + 1];
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
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void gbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory"); }
__device__ __forceinline__ u32 swz(u32 i) { return i ^ ((i >> 3) & 7u); }
__device__ __forceinline__ void hb(double2& a, double2& b) {
  a.x += b.x; a.y += b.y; b.x = fma(-2.0, b.x, a.x); b.y = fma(-2.0, b.y, a.y); }
__device__ __forceinline__ void xb(double2& a, double2& b) { double2 t = a; a = b; b = t; }
__device__ __forceinline__ void mb(double2& a, double2& b, const double* m) {
  double2 n0, n1;
  n0.x = fma(m[0], a.x, fma(-m[1], a.y, fma(m[2], b.x, -m[3] * b.y)));
  n0.y = fma(m[0], a.y, fma(m[1], a.x, fma(m[2], b.y, m[3] * b.x)));
  n1.x = fma(m[4], a.x, fma(-m[5], a.y, fma(m[6], b.x, -m[7] * b.y)));
  n1.y = fma(m[4], a.y, fma(m[5], a.x, fma(m[6], b.y, m[7] * b.x)));
  a = n0; b = n1; }
// real 2x2 (RY, Hadamard-like): 8 FP64 ops per pair
__device__ __forceinline__ void mr(double2& a, double2& b, const double* m) {
  double2 n0, n1;
  n0.x = fma(m[0], a.x, m[2] * b.x); n0.y = fma(m[0], a.y, m[2] * b.y);
  n1.x = fma(m[4], a.x, m[6] * b.x); n1.y = fma(m[4], a.y, m[6] * b.y);
  a = n0; b = n1; }
// real diagonal, imaginary off-diagonal (RX): 8 FP64 ops per pair
__device__ __forceinline__ void mx(double2& a, double2& b, const double* m) {
  double2 n0, n1;
  n0.x = fma(m[0], a.x, -m[3] * b.y); n0.y = fma(m[0], a.y, m[3] * b.x);
  n1.x = fma(m[6], b.x, -m[5] * a.y); n1.y = fma(m[6], b.y, m[5] * a.x);
  a = n0; b = n1; }
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }
)CUDA";

struct Gen {
  std::ostringstream o;
  int ntab = 0, ncoef = 0;
};

void emit_bits(std::ostringstream& o, const char* var, const char* src, const uint8_t* pos, int n) {
  o << "    const u32 " << var << " = 0u";
  for (int k = 0; k < n; ++k) o << " | (((" << src << " >> " << k << ") & 1u) << " << (int)pos[k] << ")";
  o << ";\n";
}

}  // namespace

// Emit the source of one pass. Returns false when the structure is outside
// what the generator covers (the caller keeps the interpreter).
bool jit_source(const TmaParams& tp, std::string* src, std::vector<long long>* toff,
                std::vector<double>* coef) {
  const int C = tp.C, M = tp.M, T = C - M, NA = 1 << M;
  if (M != 4 && M != 3) return false;
  std::ostringstream b;
  toff->clear();
  coef->clear();
  // tables and coefficients become parameter slots in program order
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) {
      const TOp& op = tp.ops[o];
      if (op.code == OP_DIAG) toff->push_back(op.table);
    }
  int ng = 0, st = 0;
  if (tma_smem_bytes(C, M, &ng, &st) < 0) return false;
  const int GT = 1 << T;
  const int consumers = GT * ng;
  const int rows_chunk = 1 << (C - 3);
  b << "    double2 v[" << NA << "];\n";
  int tab_i = 0;
  for (int ph = 0; ph < tp.nphases; ++ph) {
    const TPhase& D = tp.ph[ph];
    const bool last = ph + 1 == tp.nphases;
    b << "    {  // phase " << ph << "\n";
    emit_bits(b, "lt", "tid", D.tpos, T);
    for (int j = 0; j < NA; ++j) b << "    v[" << j << "] = sm[swz(lt | " << D.rloc[j] << "u)];\n";
    if (last) b << "    (void)0;\n";
    for (int o = D.op_begin; o < D.op_end; ++o) {
      const TOp& op = tp.ops[o];
      switch (op.code) {
        case STEP_1Q:
          for (int s = 0; s < M; ++s) {
            const int k = op.st[s];
            if (!k) continue;
            int ci = -1;
            const char* fn = "mb";
            if (k == 3) {
              ci = (int)coef->size();
              const double* m = tp.coef + op.cf[s];
              for (int q = 0; q < 8; ++q) coef->push_back(m[q]);
              // m = m00r m00i m01r m01i m10r m10i m11r m11i
              if (m[1] == 0.0 && m[3] == 0.0 && m[5] == 0.0 && m[7] == 0.0) fn = "mr";
              else if (m[1] == 0.0 && m[7] == 0.0 && m[2] == 0.0 && m[4] == 0.0) fn = "mx";
            }
            for (int j = 0; j < NA; ++j) {
              if (j & (1 << s)) continue;
              const int jj = j | (1 << s);
              if (k == 1) b << "    hb(v[" << j << "], v[" << jj << "]);\n";
              else if (k == 2) b << "    xb(v[" << j << "], v[" << jj << "]);\n";
              else b << "    " << fn << "(v[" << j << "], v[" << jj << "], p.coef + " << ci << ");\n";
            }
          }
          break;
        case OP_DIAG: {
          b << "    { const double2* tb = p.tabs + p.toff[" << tab_i++ << "];\n";
          b << "      const u32 pt = 0u";
          for (int k = 0; k < T; ++k)
            if (op.tcontrib[k]) b << " | (((tid >> " << k << ") & 1u) * " << op.tcontrib[k] << "u)";
          b << ";\n";
          for (int j = 0; j < NA; ++j) b << "      v[" << j << "] = cm(v[" << j << "], __ldg(tb + (pt | " << op.pr[j] << "u)));\n";
          b << "    }\n";
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
        case OP_SCALE: {
          const int ci = (int)coef->size();
          coef->push_back(tp.coef[op.coef]);
          b << "    { const double sc = p.coef[" << ci << "];\n";
          for (int j = 0; j < NA; ++j) b << "      v[" << j << "].x *= sc; v[" << j << "].y *= sc;\n";
          b << "    }\n";
          break;
        }
        default:
          return false;
      }
    }
    if (!last) {
      for (int j = 0; j < NA; ++j) b << "    sm[swz(lt | " << D.rloc[j] << "u)] = v[" << j << "];\n";
      b << "    gbar(bar_id, " << GT << ");\n";
    } else {
      b << "    fence_async_smem();\n    gbar(bar_id, " << GT << ");\n";
      b << "    if (tid == 0) mbar_arrive(empty + s);\n";
      if (tp.permuted) {
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
    }
    b << "    }\n";
  }
  std::ostringstream o;
  o << "#define QK_NTAB " << toff->size() << "\n#define QK_NCOEF " << coef->size() << "\n";
  o << kPreamble;
  o << "extern \"C\" __global__ void __launch_bounds__(" << 32 + consumers << ", 1) qk_jit(const __grid_constant__ QkJitParams p) {\n"
    << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
    << "  unsigned char* base = smem_raw;\n"
    << "  const u32 stage_bytes = " << (16u << C) << "u;\n"
    << "  u64* full = (u64*)(base + " << (size_t)st * (16u << C) << "ull);\n"
    << "  u64* empty = full + " << st << ";\n"
    << "  if (threadIdx.x == 0) {\n"
    << "    for (int s = 0; s < " << st << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n"
    << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n"
    << "  __syncthreads();\n"
    << "  const u64 G = gridDim.x;\n"
    << "  if (threadIdx.x < 32) {\n"
    << "    if (threadIdx.x == 0) {\n"
    << "      asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&p.map) : \"memory\");\n"
    << "      for (u64 i = 0;; ++i) {\n"
    << "        const u64 chunk = blockIdx.x + i * G;\n"
    << "        if (chunk >= p.nchunks) break;\n"
    << "        const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
    << "        if (round > 0) mbar_wait(empty + s, (round - 1) & 1u);\n"
    << "        mbar_expect_tx(full + s, stage_bytes);\n"
    << "        unsigned char* dst = base + (size_t)s * stage_bytes;\n"
    << "        const int row0 = (int)(chunk * " << rows_chunk << "ull);\n";
  for (int t = 0; t < tp.ntma; ++t)
    o << "        tma_load(dst + " << t * tp.box_rows * 128 << ", &p.map, 0, row0 + " << t * tp.box_rows << ", full + s);\n";
  o << "      }\n    }\n    return;\n  }\n"
    << "  const int ct = threadIdx.x - 32;\n"
    << "  const int g = ct >> " << T << ";\n"
    << "  const u32 tid = ct & " << (GT - 1) << "u;\n"
    << "  const int bar_id = 1 + g;\n"
    << "  for (u64 i = g;; i += " << ng << ") {\n"
    << "    const u64 chunk = blockIdx.x + i * G;\n"
    << "    if (chunk >= p.nchunks) break;\n"
    << "    const int s = (int)(i % " << st << "); const u32 round = (u32)(i / " << st << ");\n"
    << "    double2* sm = (double2*)(base + (size_t)s * stage_bytes);\n"
    << "    mbar_wait(full + s, round & 1u);\n"
    << b.str()
    << "  }\n}\n";
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
          cudaLibraryGetKernel(&e->kern, e->lib, "qk_jit") != cudaSuccess) {
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
int jit_launch(void* kern, const void* params, int C, int M, uint64_t nchunks, int num_sms, CUstream_st* stream) {
  int ng = 0, st = 0;
  const int smem = tma_smem_bytes(C, M, &ng, &st);
  if (smem < 0) return -1;
  const int threads = 32 + (1 << (C - M)) * ng;
  const uint64_t grid = nchunks < (uint64_t)num_sms ? nchunks : (uint64_t)num_sms;
  void* args[] = {const_cast<void*>(params)};
  cudaError_t e = cudaLaunchKernel((const void*)kern, dim3((unsigned)grid), dim3(threads), args, smem,
                                   reinterpret_cast<cudaStream_t>(stream));
  return (int)e;
}

}  // namespace qk
