// qk_runtime.cpp — host runtime behind the C ABI in include/qkb200.h.
//
// Owns the HBM-resident complex128 state, parses the optimized circuit format
// (circuit.py:245-397), compiles every instruction into device plans once per
// load (gate blocks -> passes/phases/ops + diagonal tables; SQS/CSQS -> tile
// permutation descriptors), and replays them with asynchronous launches on one
// stream per handle (Simulator.run, simulator.py:529-555).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <deque>
#include <map>
#include <memory>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>  // environ
#include <string>
#include <string_view>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/qkb200.h"
#include "qk_internal.h"

using namespace qk;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                          \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess)                                                      \
      return fail(QK_ECUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), \
                  __FILE__, __LINE__, cudaGetErrorString(_e));                  \
  } while (0)

const double kSqrt1_2 = 1.0 / std::sqrt(2.0);   // simulator.py:34
const double kDefaultAngle = 3.14159265358979323846 / 4.0;  // circuit.py:21

const char* kKindName[] = {"H", "X", "U", "CX", "CP", "SWAP", "RX", "RY", "RZ", "RZZ", "D"};
const int kArity[] = {1, 1, 1, 2, 2, 2, 1, 1, 1, 2, -1};
const int kNParams[] = {0, 0, 3, 0, 1, 0, 1, 1, 1, 1, -1};

bool is_diag(int kind) { return kind == QK_RZ || kind == QK_RZZ || kind == QK_CP || kind == QK_D; }

struct GateH {
  int kind = 0;
  std::vector<int> t;
  std::vector<double> p;  // angles; D: re,im pairs
  long gid = 0;
};

struct InstrH {
  int type = 0;  // QK_INS_*
  std::vector<GateH> gates;
  std::vector<int> a, b;
  // cross-block pass of the scheduler (reblock): targets are wires (start
  // positions); the tile holds tile_w, and the store puts rows_next on the
  // row bits 0.. and the next pass's wires on the lowest tile bits after them
  int rb = 0;
  std::vector<int> tile_w, rows_next;
  // reblocked cross-shard CSQS: the wire at every position just before it
  std::vector<int> xw;
};

// ---------------------------------------------------------------------------
// parser: restates circuit.py:245-287, 332-397 (messages included)

struct Tok {
  std::string s;
};

bool parse_int(const std::string& s, long* out) {
  // Python int(): optional sign, digits, surrounding whitespace already stripped
  if (s.empty()) return false;
  size_t i = 0;
  if (s[0] == '+' || s[0] == '-') i = 1;
  if (i >= s.size()) return false;
  for (size_t j = i; j < s.size(); ++j)
    if (!isdigit((unsigned char)s[j]) && s[j] != '_') return false;
  errno = 0;
  std::string t;
  for (char ch : s)
    if (ch != '_') t.push_back(ch);
  *out = strtol(t.c_str(), nullptr, 10);
  return errno == 0;
}

bool parse_float(const std::string& s, double* out) {
  if (s.empty()) return false;
  char* end = nullptr;
  *out = strtod(s.c_str(), &end);
  return end && *end == '\0';
}

std::string pyrepr(const std::string& s) { return "'" + s + "'"; }

struct Parser {
  int n, c, local;
  std::string msg;
  int line_no = 0;
  int code = QK_OK;

  int err(int ln, const std::string& m) {
    line_no = ln;
    msg = "line " + std::to_string(ln) + ": " + m;
    code = QK_EPARSE;
    return code;
  }
  int verr(const std::string& m) {
    msg = m;
    code = QK_EINVAL;
    return code;
  }

  int gate_line(const std::vector<std::string>& tk, int ln, GateH* g) {
    const std::string& k0 = tk[0];
    int kind = -1, darity = -1;
    if (k0.size() > 1 && k0[0] == 'D' &&
        std::all_of(k0.begin() + 1, k0.end(), [](char ch) { return isdigit((unsigned char)ch); })) {
      kind = QK_D;
      darity = atoi(k0.c_str() + 1);
    } else {
      for (int i = 0; i < 10; ++i)
        if (k0 == kKindName[i]) kind = i;
      if (kind < 0) return err(ln, "unknown gate symbol " + pyrepr(k0));
    }
    g->kind = kind;
    if (kind == QK_D) {
      const long want = 1 + darity + 2 * (1L << std::min(darity, 30));
      if ((long)tk.size() != want)
        return err(ln, "D" + std::to_string(darity) + " line needs " + std::to_string(want) +
                           " tokens, got " + std::to_string(tk.size()));
      for (int j = 0; j < darity; ++j) {
        long v;
        if (!parse_int(tk[1 + j], &v))
          return err(ln, "invalid literal for int() with base 10: " + pyrepr(tk[1 + j]));
        g->t.push_back((int)v);
      }
      for (size_t j = 1 + darity; j < tk.size(); ++j) {
        double v;
        if (!parse_float(tk[j], &v)) return err(ln, "could not convert string to float: " + pyrepr(tk[j]));
        g->p.push_back(v);
      }
      g->gid = -1;
    } else {
      const int ar = kArity[kind], np = kNParams[kind];
      std::vector<std::string> ptok;
      if ((int)tk.size() == 1 + ar + 1) {
      } else if ((int)tk.size() == 1 + ar + 1 + np) {
        ptok.assign(tk.begin() + 1 + ar + 1, tk.end());
      } else {
        return err(ln, std::string("wrong token count for ") + kKindName[kind] + ": got " +
                           std::to_string(tk.size()));
      }
      for (int j = 0; j < ar; ++j) {
        long v;
        if (!parse_int(tk[1 + j], &v))
          return err(ln, "invalid literal for int() with base 10: " + pyrepr(tk[1 + j]));
        g->t.push_back((int)v);
      }
      long gid;
      if (!parse_int(tk[1 + ar], &gid))
        return err(ln, "invalid literal for int() with base 10: " + pyrepr(tk[1 + ar]));
      g->gid = gid;
      if (ptok.empty()) {
        g->p.assign(np, kDefaultAngle);
      } else {
        for (auto& s : ptok) {
          double v;
          if (!parse_float(s, &v)) return err(ln, "could not convert string to float: " + pyrepr(s));
          g->p.push_back(v);
        }
      }
    }
    for (int q : g->t)
      if (q < 0 || q >= n)
        return err(ln, "qubit index out of range: " + std::to_string(q) + " (N=" + std::to_string(n) + ")");
    for (size_t i = 0; i < g->t.size(); ++i)
      for (size_t j = i + 1; j < g->t.size(); ++j)
        if (g->t[i] == g->t[j])
          return err(ln, std::string("duplicate target qubits in ") + kKindName[kind]);
    if (g->gid < 0 && kind != QK_D) return err(ln, "negative gate id " + std::to_string(g->gid));
    if (kind == QK_D && darity < 2) return verr("fused diagonal needs at least 2 qubits");
    return QK_OK;
  }

  int run(const char* text, size_t len, std::vector<InstrH>* out) {
    std::vector<std::pair<int, std::vector<std::string>>> lines;
    size_t pos = 0;
    int ln = 0;
    while (pos <= len) {
      size_t e = pos;
      while (e < len && text[e] != '\n') ++e;
      ++ln;
      std::string line(text + pos, e - pos);
      if (!line.empty() && line.back() == '\r') line.pop_back();
      const size_t hash = line.find('#');
      if (hash != std::string::npos) line.resize(hash);
      std::vector<std::string> tk;
      size_t i = 0;
      while (i < line.size()) {
        while (i < line.size() && isspace((unsigned char)line[i])) ++i;
        size_t j = i;
        while (j < line.size() && !isspace((unsigned char)line[j])) ++j;
        if (j > i) tk.emplace_back(line.substr(i, j - i));
        i = j;
      }
      if (!tk.empty()) lines.emplace_back(ln, std::move(tk));
      if (e >= len) break;
      pos = e + 1;
    }
    size_t i = 0;
    while (i < lines.size()) {
      const int lno = lines[i].first;
      const auto& tk = lines[i].second;
      if (tk.size() != 1) {
        std::string j;
        for (size_t q = 0; q < tk.size(); ++q) j += (q ? " " : "") + tk[q];
        return err(lno, "expected a record count, got " + pyrepr(j));
      }
      long count;
      if (!parse_int(tk[0], &count)) return err(lno, "expected a record count, got " + pyrepr(tk[0]));
      if (count < 1) return err(lno, "record count must be positive");
      if (i + 1 + (size_t)count > lines.size())
        return err(lno, "record claims " + std::to_string(count) + " lines but file ends early");
      const std::string& first = lines[i + 1].second[0];
      if (first == "SQS" || first == "CSQS") {
        if (count != 1) return err(lno, "swap records hold exactly one line");
        const int l2 = lines[i + 1].first;
        const auto& st = lines[i + 1].second;
        if (st.size() < 2) return err(l2, first + " needs a pair count");
        long m;
        if (!parse_int(st[1], &m)) return err(l2, "invalid literal for int() with base 10: " + pyrepr(st[1]));
        std::vector<int> ops;
        for (size_t q = 2; q < st.size(); ++q) {
          long v;
          if (!parse_int(st[q], &v)) return err(l2, "invalid literal for int() with base 10: " + pyrepr(st[q]));
          ops.push_back((int)v);
        }
        if ((long)st.size() != 2 + 2 * m)
          return err(l2, first + " " + std::to_string(m) + " needs exactly " + std::to_string(2 + 2 * m) +
                             " tokens, got " + std::to_string(st.size()));
        InstrH ins;
        ins.type = first == "SQS" ? QK_INS_SQS : QK_INS_CSQS;
        ins.a.assign(ops.begin(), ops.begin() + m);
        ins.b.assign(ops.begin() + m, ops.end());
        if (ins.type == QK_INS_SQS) {
          for (int x : ins.a)
            for (int y : ins.b)
              if (x == y) return verr("swap sets must be disjoint");
          for (int q : ins.a)
            if (q < 0 || q >= local) return err(l2, "SQS index " + std::to_string(q) + " outside local range");
          for (int q : ins.b)
            if (q < 0 || q >= local) return err(l2, "SQS index " + std::to_string(q) + " outside local range");
        } else {
          for (int q : ins.a)
            if (q < 0 || q >= local)
              return err(l2, "CSQS local index " + std::to_string(q) + " outside local range");
          for (int q : ins.b)
            if (q < local || q >= n)
              return err(l2, "CSQS rank index " + std::to_string(q) + " outside rank range");
        }
        out->push_back(std::move(ins));
      } else {
        InstrH ins;
        ins.type = QK_INS_BLOCK;
        for (long q = 0; q < count; ++q) {
          const int l2 = lines[i + 1 + q].first;
          GateH g;
          if (gate_line(lines[i + 1 + q].second, l2, &g)) return code;
          if (c > 0)
            for (int t : g.t)
              if (t >= c)
                return err(l2, "gate target " + std::to_string(t) + " >= chunk qubits C=" + std::to_string(c));
          ins.gates.push_back(std::move(g));
        }
        out->push_back(std::move(ins));
      }
      i += 1 + count;
    }
    return QK_OK;
  }
};

// ---------------------------------------------------------------------------
// gate constants (circuit.py:420-463; simulator.py:242-310)

typedef std::complex<double> cplx;

cplx cexpi(double x) { return cplx(std::cos(x), std::sin(x)); }

// diagonal entries; targets[0] = MSB of the entry index
std::vector<cplx> diag_entries(const GateH& g) {
  const double th = g.p.empty() ? 0.0 : g.p[0];
  switch (g.kind) {
    case QK_RZ: return {cexpi(-0.5 * th), cexpi(0.5 * th)};
    case QK_RZZ: {
      const cplx em = cexpi(-0.5 * th), ep = cexpi(0.5 * th);
      return {em, ep, ep, em};
    }
    case QK_CP: return {1.0, 1.0, 1.0, cexpi(th)};
    default: {
      std::vector<cplx> e;
      for (size_t i = 0; i + 1 < g.p.size(); i += 2) e.emplace_back(g.p[i], g.p[i + 1]);
      return e;
    }
  }
}

// 2x2 matrix (row-major m00 m01 m10 m11) of U, RX, RY
void mat2(const GateH& g, cplx m[4]) {
  if (g.kind == QK_U) {
    const double th = g.p[0], ph = g.p[1], lam = g.p[2];
    const double ct = std::cos(th / 2), st = std::sin(th / 2);
    m[0] = ct;
    m[1] = -cexpi(lam) * st;
    m[2] = cexpi(ph) * st;
    m[3] = cexpi(ph + lam) * ct;
  } else if (g.kind == QK_RX) {
    const double c = std::cos(g.p[0] / 2), s = std::sin(g.p[0] / 2);
    m[0] = c;
    m[1] = cplx(0, -s);
    m[2] = cplx(0, -s);
    m[3] = c;
  } else {  // RY
    const double c = std::cos(g.p[0] / 2), s = std::sin(g.p[0] / 2);
    m[0] = c;
    m[1] = -s;
    m[2] = s;
    m[3] = c;
  }
}

// m = lam * f with the larger of |m00|, |m01| factored out (exactly 1 in f).
// A unitary 2x2 has |m00| = |m11| >= 1/sqrt2 or |m01| = |m10| >= 1/sqrt2, so
// f stays well conditioned. The scalar lam is global to the pass (every
// amplitude is touched by the gate) and joins the pass scale; the kernels then
// apply f, whose exact ones and zeros (RX: 1 and -i tan, RY: 1 and +-tan)
// make the butterfly 4 FMAs per pair instead of 8-16.
void factor_mat(const cplx m[4], cplx f[4], cplx* lam) {
  const int piv = std::abs(m[0]) >= std::abs(m[1]) ? 0 : 1;
  const cplx l = m[piv];
  auto div = [&](cplx x) {
    if (l.imag() == 0.0) return cplx(x.real() / l.real(), x.imag() / l.real());
    if (l.real() == 0.0) return cplx(x.imag() / l.imag(), -x.real() / l.imag());
    return x / l;
  };
  for (int k = 0; k < 4; ++k) f[k] = k == piv ? cplx(1.0, 0.0) : div(m[k]);
  *lam = l;
}

// ---------------------------------------------------------------------------
// plans

struct HostPlan {
  std::vector<PassDesc> passes;
  std::vector<PhaseDesc> phases;
  std::vector<OpDesc> ops;
  std::vector<double> coef;
  std::vector<TableDesc> tables;
  std::vector<TableGate> tgates;
  std::vector<double> entries;  // complex pairs
  int64_t pool = 0;             // table pool size (complex entries)
  std::vector<SqsDesc> sqs;
  // OP_QUAD data (qk_internal.h QuadLayout), copied into the pool at upload
  std::vector<std::pair<int64_t, std::vector<double>>> qcopy;
  void clear() { *this = HostPlan(); }
};

struct InstrPlan {
  int type;
  int pass0 = 0, npass = 0;  // block
  std::vector<int> dest;     // block: destination bit of each source bit (fused SQS), empty if none
  int permuted = 0;          // block: last pass scatters out-of-place (set at upload)
  int fused_by = -1;         // SQS/CSQS: index of the block whose last pass absorbs it
  int synthetic = 0;         // block: layout-restore pass appended by the planner
  std::vector<int> xspec;    // block: spectator source bits of a cluster-exchange store (qk_jit.cpp)
  int lazy = 0;              // SQS / local CSQS absorbed into the lazy layout: no kernel
  std::vector<int> tile;     // block: strided tile (physical bits) of a lazy in-place pass
  std::vector<int> xlay;     // cross-process CSQS: layout (reference bit -> physical) at the exchange
  int sqs = -1;              // SQS / single-device CSQS
  int csqs_s = 0;            // multi-process CSQS
  std::vector<int> a, b;
  double bytes = 0;          // algorithmic HBM bytes
  // cross-process CSQS pipelined with its neighbour passes (set at upload):
  // the pass before (ovl_p), the exchange and the pass after (ovl_q) all run
  // in 2^ovl_k parts split on the same physical bits ovl_f (outside both
  // tiles and outside the exchanged bits), so part f of the exchange (comm
  // stream) overlaps part f+1 of the pass before and part f-1 of the pass after
  int ovl_p = -1, ovl_q = -1, ovl_k = 0;
  int ovl_f[2] = {0, 0};          // split bits (physical)
  int ovl_cp[2] = {0, 0};         // their chunk-index bits in ovl_p / ovl_q
  int ovl_cq[2] = {0, 0};
};

int popc(uint64_t x) { return __builtin_popcountll(x); }

// thread-bit order: lane bits 0..2 (the 8 lanes of one 128-bit shared-memory
// wavefront) on the lowest positions whose SWIZZLE_128B bank contributions
// (p < 3: bit p, 3 <= p < 6: bit p-3, none above) are independent, so the TMA
// image is read conflict-free; the remaining thread bits follow ascending, so
// a phase without register qubits among 0..4 stores whole 512-B runs.
std::vector<int> order_tpos(const std::vector<int>& T) {
  if (T.size() < 3) return T;
  std::vector<int> first;
  uint32_t span = 1;  // bit x set: x is in the span of the chosen masks
  for (int p : T) {
    if (p >= 6) break;
    const uint32_t m = 1u << (p % 3);
    if (span >> m & 1) continue;
    first.push_back(p);
    uint32_t ns = span;
    for (uint32_t x = 0; x < 8; ++x)
      if (span >> x & 1) ns |= 1u << (x ^ m);
    span = ns;
    if (first.size() == 3) break;
  }
  std::vector<int> out = first;
  for (int p : T)
    if (std::find(first.begin(), first.end(), p) == first.end()) out.push_back(p);
  return out;
}

// Phase of a diagonal gate as a quadratic form in its target bits:
// e(x) = exp(i phi(x)), phi(x) = c + sum_j lin[j] x_j + sum_{j<j'} pair[j][j'] x_j x_j'
// (x_j = the bit of target j; targets[0] is the MSB of the entry index,
// circuit.py:426-463). RZ, RZZ and CP use their angle directly; D<k> entries
// must be unit (|e| = 1 to 1e-13) and, for k >= 3, have no Moebius terms of
// degree >= 3 (mod 2 pi). False otherwise: the gate then stays in a table.
double wrap_angle(double x) {
  const double tp = 6.283185307179586476925286766559;
  return x - tp * std::nearbyint(x / tp);
}

bool quad_terms(const GateH& g, double* c, double lin[13], double pair[13][13]) {
  const int nt = (int)g.t.size();
  if (nt < 1 || nt > 13 || !is_diag(g.kind)) return false;
  std::vector<double> ph((size_t)1 << nt, 0.0);
  const double th = g.p.empty() ? 0.0 : g.p[0];
  if (g.kind == QK_RZ && nt == 1) {
    ph[0] = -0.5 * th;
    ph[1] = 0.5 * th;
  } else if (g.kind == QK_RZZ && nt == 2) {
    ph[0] = ph[3] = -0.5 * th;
    ph[1] = ph[2] = 0.5 * th;
  } else if (g.kind == QK_CP && nt == 2) {
    ph[3] = th;
  } else {
    const std::vector<cplx> e = diag_entries(g);
    if (e.size() != ph.size()) return false;
    for (size_t x = 0; x < e.size(); ++x) {
      if (std::fabs(std::abs(e[x]) - 1.0) > 1e-13) return false;
      ph[x] = std::arg(e[x]);
    }
  }
  // Moebius transform: ph[m] becomes the coefficient of prod_{b in m} x_b
  for (int b = 0; b < nt; ++b)
    for (size_t x = 0; x < ph.size(); ++x)
      if (x >> b & 1) ph[x] -= ph[x ^ ((size_t)1 << b)];
  for (size_t m = 0; m < ph.size(); ++m)
    if (popc(m) >= 3 && std::fabs(wrap_angle(ph[m])) > 1e-12) return false;
  *c = ph[0];
  for (int j = 0; j < nt; ++j) {
    lin[j] = ph[(size_t)1 << (nt - 1 - j)];
    for (int j2 = j + 1; j2 < nt; ++j2) pair[j][j2] = ph[((size_t)1 << (nt - 1 - j)) | ((size_t)1 << (nt - 1 - j2))];
  }
  return true;
}

bool quad_gate(const GateH& g) {
  double c, lin[13], pair[13][13];
  return quad_terms(g, &c, lin, pair);
}

struct Item {
  int type;  // 0 gate, 1 diag run
  const GateH* g;
  int run;
};

bool m5_enabled() { return getenv("QK_M5") && jit_available(); }

// Compile the gates of one pass over chunk address bits Q (ascending) of a
// vector of `nbits` address bits.
int compile_pass(HostPlan& hp, const std::vector<const GateH*>& gates_in, const std::vector<int>& Q,
                 int nbits, uint64_t ncta_override, std::string& emsg, const std::vector<int>* dest = nullptr,
                 int lanes_req = 5, bool allow_quad = false) {
  // 0. U(th, ph, la) = P(ph) RY(th) P(la) with P(a) = diag(1, e^{ia}) exactly
  //    (circuit.py:420-423 Qiskit form). A run of U gates on distinct qubits
  //    becomes [all P(la)] [all RY] [all P(ph)]: the phase gates join two
  //    diagonal tables and each RY costs 4 FMAs per pair instead of 12.
  std::deque<GateH> expanded;
  std::vector<const GateH*> gates;
  for (size_t i = 0; i < gates_in.size();) {
    const GateH* g = gates_in[i];
    if (g->kind != QK_U || getenv("QK_NO_UDECOMP") || g->p.size() < 3) {
      gates.push_back(g);
      ++i;
      continue;
    }
    size_t e = i;
    uint64_t seen = 0;
    while (e < gates_in.size() && gates_in[e]->kind == QK_U && gates_in[e]->p.size() >= 3 &&
           !(seen >> gates_in[e]->t[0] & 1))
      seen |= 1ull << gates_in[e++]->t[0];
    auto phase = [&](int q, double a) {
      GateH d;
      d.kind = QK_D;
      d.t = {q};
      d.p = {1.0, 0.0, std::cos(a), std::sin(a)};
      expanded.push_back(d);
      gates.push_back(&expanded.back());
    };
    for (size_t k = i; k < e; ++k) phase(gates_in[k]->t[0], gates_in[k]->p[2]);
    for (size_t k = i; k < e; ++k) {
      GateH ry;
      ry.kind = QK_RY;
      ry.t = gates_in[k]->t;
      ry.p = {gates_in[k]->p[0]};
      expanded.push_back(ry);
      gates.push_back(&expanded.back());
    }
    for (size_t k = i; k < e; ++k) phase(gates_in[k]->t[0], gates_in[k]->p[1]);
    i = e;
  }
  const int C = (int)Q.size();
  int M = std::min(kMaxM, C);
  if (C >= 9 && C <= 12 && Q.back() == C - 1 && getenv("QK_M")) M = std::max(3, std::min(4, atoi(getenv("QK_M"))));
  // five register qubits (32 amplitudes per thread, two 128-thread groups per
  // CTA): fewer phases for wide passes; specialised kernels only
  if (allow_quad && C == 12 && m5_enabled()) M = 5;
  int loc[64];
  for (int& x : loc) x = -1;
  for (int l = 0; l < C; ++l) loc[Q[l]] = l;

  // 1. diagonal runs (diagonal gates commute with each other and with any gate
  //    on disjoint qubits: a diagonal gate joins the latest run unless a
  //    non-diagonal gate emitted after that run touches one of its qubits)
  std::vector<Item> items;
  std::vector<std::vector<const GateH*>> runs;
  std::vector<uint32_t> run_support;
  int last_run = -1;
  uint32_t blocked = 0;
  int nh = 0;
  // diagonal gates may also act on address bits outside the chunk (diagonal
  // blocks folded into this pass): their value is fixed per chunk, so they
  // only add a per-chunk term to the table index (specialised kernels only)
  std::vector<uint64_t> run_outer;
  // OP_QUAD runs (allow_quad, specialised kernels): every gate's phase is
  // quadratic, so the run is one op whatever its width and outer bits
  std::vector<char> run_quad;
  for (const GateH* g : gates) {
    uint32_t tm = 0;
    uint64_t om = 0;
    for (int t : g->t) {
      if (t >= 0 && t < 64 && loc[t] < 0 && is_diag(g->kind) && t < nbits) {
        om |= 1ull << t;
        continue;
      }
      if (t >= 64 || loc[t] < 0) {
        emsg = "gate target outside pass chunk";
        return QK_ESIM;
      }
      tm |= 1u << loc[t];
    }
    if (is_diag(g->kind)) {
      const bool gq = allow_quad && quad_gate(*g);
      const int width = last_run >= 0 ? popc(run_support[last_run] | tm) + popc(run_outer[last_run] | om) : 99;
      const bool fits_table = width <= 14 && last_run >= 0 && popc(run_outer[last_run] | om) <= 8;
      if (last_run >= 0 && !(tm & blocked) && ((gq && run_quad[last_run]) || fits_table)) {
        runs[last_run].push_back(g);
        run_support[last_run] |= tm;
        run_outer[last_run] |= om;
        run_quad[last_run] = run_quad[last_run] && gq;
      } else {
        if (popc(om) > 8 && !gq) {
          emsg = "diagonal gate over too many bits outside the chunk";
          return QK_ESIM;
        }
        runs.push_back({g});
        run_support.push_back(tm);
        run_outer.push_back(om);
        run_quad.push_back(gq);
        last_run = (int)runs.size() - 1;
        blocked = 0;
        items.push_back({1, nullptr, last_run});
      }
    } else {
      items.push_back({0, g, -1});
      blocked |= tm;
      if (g->kind == QK_H) ++nh;
    }
  }
  // 1b. One-qubit gates on distinct qubits with nothing between them commute.
  //     Order each such segment so the first phase takes high positions and
  //     the low positions 0..4 go to the second: the first phase then reads
  //     the TMA image (bank bits from positions < 6) conflict-free and the
  //     last phase keeps lanes on the low positions (whole-run stores).
  if (!getenv("QK_NO_REORDER")) {
    auto one_q = [&](const Item& it) {
      return it.type == 0 && it.g->t.size() == 1 &&
             (it.g->kind == QK_H || it.g->kind == QK_X || it.g->kind == QK_U || it.g->kind == QK_RX ||
              it.g->kind == QK_RY);
    };
    for (size_t a = 0; a < items.size();) {
      if (!one_q(items[a])) {
        ++a;
        continue;
      }
      size_t b = a;
      uint32_t seen = 0;
      while (b < items.size() && one_q(items[b]) && !(seen >> loc[items[b].g->t[0]] & 1))
        seen |= 1u << loc[items[b++].g->t[0]];
      if (b - a > (size_t)M) {
        std::vector<Item> hi, lo;
        for (size_t k = a; k < b; ++k) (loc[items[k].g->t[0]] < 5 ? lo : hi).push_back(items[k]);
        auto pos = [&](const Item& it) { return loc[it.g->t[0]]; };
        std::stable_sort(hi.begin(), hi.end(), [&](const Item& x, const Item& y) { return pos(x) > pos(y); });
        std::stable_sort(lo.begin(), lo.end(), [&](const Item& x, const Item& y) { return pos(x) < pos(y); });
        // second group: the M lowest positions; low positions beyond M join
        // the first group (the last phase keeps lanes 0..4 on positions 0..4)
        const size_t nmid = std::min(lo.size(), (size_t)M);
        const size_t nextra = lo.size() - nmid;
        const size_t nhi0 = nextra < (size_t)M ? std::min(hi.size(), (size_t)M - nextra) : 0;
        std::vector<Item> ord;
        for (size_t k = 0; k < nhi0; ++k) ord.push_back(hi[k]);
        for (size_t k = nmid; k < lo.size(); ++k) ord.push_back(lo[k]);
        for (size_t k = 0; k < nmid; ++k) ord.push_back(lo[k]);
        for (size_t k = nhi0; k < hi.size(); ++k) ord.push_back(hi[k]);
        for (size_t k = 0; k < ord.size(); ++k) items[a + k] = ord[k];
      }
      a = b;
    }
  }
  // 2. register needs per item
  auto needs = [&](const Item& it) -> std::vector<int> {
    if (it.type == 1) return {};
    const GateH* g = it.g;
    if (g->kind == QK_CX) return {loc[g->t[1]]};
    std::vector<int> r;
    for (int t : g->t) r.push_back(loc[t]);
    return r;
  };
  // 3. phases
  struct PhaseB {
    std::vector<int> R;
    std::vector<int> items;
  };
  std::vector<PhaseB> phs;
  // Positions that fill a phase's free register slots: the highest chunk
  // positions, or for a fused (permuted) store the positions with the highest
  // destinations, so the last phase keeps the store lanes (the lowest
  // destinations) off its registers and needs no extra layout-only phase.
  std::vector<int> fill_order;
  for (int q = C - 1; q >= 0; --q) fill_order.push_back(q);
  if (dest && !getenv("QK_FILL_HIGH"))
    std::stable_sort(fill_order.begin(), fill_order.end(), [&](int x, int y) { return (*dest)[Q[x]] > (*dest)[Q[y]]; });
  // the store lanes of a fused pass: positions landing on destination bits 0..lanes_req-1
  std::vector<char> lane_pos(C, 0);
  if (dest)
    for (int i = 0; i < lanes_req && i < C; ++i) lane_pos[fill_order[C - 1 - i]] = 1;
  // Dependency-aware list scheduling: gates that commute (disjoint qubits,
  // diagonal runs, a diagonal on a CX control, CX sharing only a target or
  // only a control) may run in any order. Each phase picks the register set
  // that lets the most ready items run (program-order lookahead vs the most
  // frequent qubits among upcoming items), simulated greedily.
  if (!getenv("QK_OLD_PHASES")) {
    const size_t n = items.size();
    auto support = [&](const Item& it) -> uint32_t {
      if (it.type == 1) return run_support[it.run];
      uint32_t m = 0;
      for (int t : it.g->t) m |= 1u << loc[t];
      return m;
    };
    auto commute = [&](const Item& a, const Item& b) {
      const uint32_t sa = support(a), sb = support(b), both = sa & sb;
      if (!both) return true;
      if (a.type == 1 && b.type == 1) return true;
      const Item* d = a.type == 1 ? &a : (b.type == 1 ? &b : nullptr);
      const Item* o = d == &a ? &b : &a;
      if (d && o->type == 0 && o->g->kind == QK_CX) return both == (1u << loc[o->g->t[0]]);  // diag on control
      if (!d && a.g->kind == QK_CX && b.g->kind == QK_CX) {
        const int ac = loc[a.g->t[0]], at = loc[a.g->t[1]], bc = loc[b.g->t[0]], bt = loc[b.g->t[1]];
        if (at == bt && ac != bc && ac != bt && bc != at) return true;   // same target
        if (ac == bc && at != bt && at != bc && bt != ac) return true;   // same control
      }
      return false;
    };
    std::vector<std::vector<int>> preds(n);
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < i; ++j)
        if (!commute(items[j], items[i])) preds[i].push_back((int)j);
    std::vector<char> done(n, 0);
    size_t left = n;
    auto in_r = [](const std::vector<int>& R, int q) { return std::find(R.begin(), R.end(), q) != R.end(); };
    auto runs_with = [&](const std::vector<int>& R, std::vector<char>& dn, std::vector<int>* order) {
      int cnt = 0;
      for (bool progress = true; progress;) {
        progress = false;
        for (size_t i = 0; i < n; ++i) {
          if (dn[i]) continue;
          bool ok = true;
          for (int p : preds[i]) ok = ok && dn[p];
          if (!ok) continue;
          for (int q : needs(items[i])) ok = ok && in_r(R, q);
          if (!ok) continue;
          dn[i] = 1;
          ++cnt;
          progress = true;
          if (order) order->push_back((int)i);
        }
      }
      return cnt;
    };
    while (left) {
      // first ready item that needs registers (diagonal-only readiness runs anywhere)
      int first = -1;
      for (size_t i = 0; i < n && first < 0; ++i) {
        if (done[i]) continue;
        bool ok = true;
        for (int p : preds[i]) ok = ok && done[p];
        if (ok && !needs(items[i]).empty()) first = (int)i;
      }
      std::vector<std::vector<int>> cands;
      if (first >= 0) {
        std::vector<int> base = needs(items[first]);
        // (a) program-order lookahead over the items not yet done
        std::vector<int> a = base;
        for (size_t j = first + 1; j < n && (int)a.size() < M; ++j)
          if (!done[j])
            for (int q : needs(items[j]))
              if ((int)a.size() < M && !in_r(a, q)) a.push_back(q);
        cands.push_back(a);
        // (b) most frequent qubits among the next 48 items' needs
        std::vector<int> freq(C, 0);
        int seen = 0;
        for (size_t j = first; j < n && seen < 48; ++j)
          if (!done[j]) {
            ++seen;
            for (int q : needs(items[j])) freq[q]++;
          }
        std::vector<int> b = base;
        while ((int)b.size() < M) {
          int best = -1;
          for (int q = 0; q < C; ++q)
            if (!in_r(b, q) && freq[q] > 0 && (best < 0 || freq[q] > freq[best])) best = q;
          if (best < 0) break;
          b.push_back(best);
        }
        cands.push_back(b);
        // (c) the store-lane positions with pending work first, so the last
        // phase can keep them as lanes (no layout-only phase at the end)
        std::vector<int> c3 = base;
        for (int q = 0; q < C && (int)c3.size() < M; ++q)
          if (lane_pos[q] && freq[q] > 0 && !in_r(c3, q)) c3.push_back(q);
        while ((int)c3.size() < M) {
          int best = -1;
          for (int q = 0; q < C; ++q)
            if (!in_r(c3, q) && freq[q] > 0 && (best < 0 || freq[q] > freq[best])) best = q;
          if (best < 0) break;
          c3.push_back(best);
        }
        cands.push_back(c3);
      } else {
        cands.push_back({});
      }
      // ties go to the set with more store-lane positions: their gates run
      // early and the last phase can keep them as lanes
      int best_c = -1, best_n = -1, best_l = -1;
      for (size_t c = 0; c < cands.size(); ++c) {
        auto& R = cands[c];
        for (int q : fill_order)
          if ((int)R.size() < M && !in_r(R, q)) R.push_back(q);
        std::vector<char> dn = done;
        const int k = runs_with(R, dn, nullptr);
        int nl = 0;
        for (int q : R) nl += lane_pos[q];
        if (k > best_n || (k == best_n && nl > best_l)) {
          best_n = k;
          best_c = (int)c;
          best_l = nl;
        }
      }
      PhaseB pb;
      pb.R = cands[best_c];
      runs_with(pb.R, done, &pb.items);
      if (pb.items.empty()) {
        emsg = "internal: phase scheduling made no progress";
        return QK_ESIM;
      }
      left -= pb.items.size();
      phs.push_back(pb);
    }
  }
  // the program-order builder; the scheduled phases replace it only when
  // they need fewer phases (QAOA's layers keep the program-order phases)
  std::vector<PhaseB> sched;
  sched.swap(phs);
  for (size_t i = 0; i < items.size(); ++i) {
    std::vector<int> need = needs(items[i]);
    bool fits = !phs.empty();
    if (fits)
      for (int q : need)
        if (std::find(phs.back().R.begin(), phs.back().R.end(), q) == phs.back().R.end()) fits = false;
    if (!fits) {
      PhaseB pb;
      pb.R = need;
      for (size_t j = i + 1; j < items.size() && (int)pb.R.size() < M; ++j)
        for (int q : needs(items[j]))
          if ((int)pb.R.size() < M && std::find(pb.R.begin(), pb.R.end(), q) == pb.R.end())
            pb.R.push_back(q);
      for (int q : fill_order)
        if ((int)pb.R.size() < M && std::find(pb.R.begin(), pb.R.end(), q) == pb.R.end()) pb.R.push_back(q);
      phs.push_back(pb);
    }
    phs.back().items.push_back((int)i);
  }
  auto extra = [&](const std::vector<PhaseB>& v) {
    if (!dest || v.empty()) return 0;
    for (int q : v.back().R)
      if (lane_pos[q]) return 1;
    return 0;
  };
  if (getenv("QK_DUMP_SCHED"))
    fprintf(stderr, "phase builders: program order %zu+%d, list scheduler %zu+%d\n", phs.size(), extra(phs),
            sched.size(), extra(sched));
  if (!sched.empty() && sched.size() + extra(sched) < phs.size() + extra(phs)) phs.swap(sched);
  // (dev, timing only: drops the phases beyond QK_EXP_MAXPH and their gates)
  if (const char* mx = getenv("QK_EXP_MAXPH"))
    if ((int)phs.size() > atoi(mx) && atoi(mx) > 0) phs.resize(atoi(mx));
  // Quadratic runs of one phase (allow_quad): the parts of each run that no
  // later gate of the phase needs first — gates whose tile targets are thread
  // bits or slots no later gate of the phase acts on — commute with the rest
  // of the phase and gather in one run at its end. QFT's controlled-phase
  // ladders then cost one op per phase plus the slot pairs that must stay
  // between their H gates, instead of one op per H.
  if (allow_quad && !getenv("QK_NO_PHASE_MERGE")) {
    auto recompute = [&](int r) {
      uint32_t tm = 0;
      uint64_t om = 0;
      bool q = true;
      for (const GateH* g : runs[r]) {
        q = q && quad_gate(*g);
        for (int t : g->t) {
          if (loc[t] >= 0) tm |= 1u << loc[t];
          else om |= 1ull << t;
        }
      }
      run_support[r] = tm;
      run_outer[r] = om;
      run_quad[r] = q;
    };
    for (auto& pb : phs) {
      std::vector<size_t> qi;
      for (size_t k = 0; k < pb.items.size(); ++k) {
        const Item& it = items[pb.items[k]];
        if (it.type == 1 && run_quad[it.run]) qi.push_back(k);
      }
      if (qi.size() < 2) continue;
      // slots a later item of the phase acts on, per item position
      std::vector<uint32_t> later(pb.items.size() + 1, 0);
      for (size_t k = pb.items.size(); k-- > 0;) {
        later[k] = later[k + 1];
        for (int q : needs(items[pb.items[k]])) later[k] |= 1u << q;
      }
      std::vector<const GateH*> moved;
      std::vector<std::vector<const GateH*>> stay(qi.size());
      for (size_t a = 0; a < qi.size(); ++a) {
        const int r = items[pb.items[qi[a]]].run;
        for (const GateH* g : runs[r]) {
          bool mov = true;
          for (int t : g->t)
            if (loc[t] >= 0 && (later[qi[a] + 1] >> loc[t] & 1)) mov = false;
          (mov ? moved : stay[a]).push_back(g);
        }
      }
      // cost of a run: per-thread factors (thread bits or chunk bits in it) or
      // constants only (every target a slot of the phase)
      uint32_t slots = 0;
      for (int q : pb.R) slots |= 1u << q;
      auto cost = [&](const std::vector<const GateH*>& v) {
        if (v.empty()) return 0;
        int c = 1;
        for (const GateH* g : v)
          for (int t : g->t) {
            if (loc[t] < 0) return 6;
            if (!(slots >> loc[t] & 1)) c = 3;
          }
        return c;
      };
      int before = 0, after = cost(moved);
      for (size_t a = 0; a < qi.size(); ++a) {
        before += cost(runs[items[pb.items[qi[a]]].run]);
        after += cost(stay[a]);
      }
      if (moved.empty() || after >= before) continue;
      std::vector<int> keep;
      std::vector<char> drop(pb.items.size(), 0);
      for (size_t a = 0; a < qi.size(); ++a) {
        const int r = items[pb.items[qi[a]]].run;
        runs[r] = stay[a];
        if (stay[a].empty()) drop[qi[a]] = 1;
        else recompute(r);
      }
      for (size_t k = 0; k < pb.items.size(); ++k)
        if (!drop[k]) keep.push_back(pb.items[k]);
      runs.push_back(moved);
      run_support.push_back(0);
      run_outer.push_back(0);
      run_quad.push_back(true);
      recompute((int)runs.size() - 1);
      items.push_back({1, nullptr, (int)runs.size() - 1});
      keep.push_back((int)items.size() - 1);
      pb.items = keep;
    }
  }
  if (getenv("QK_DUMP_PHASES")) {
    fprintf(stderr, "pass C=%d dest=%d lanes:", C, dest ? 1 : 0);
    for (int q = 0; q < C; ++q)
      if (lane_pos[q]) fprintf(stderr, " %d", q);
    fprintf(stderr, "\n");
    for (auto& pb : phs) {
      fprintf(stderr, "  R={");
      for (int q : pb.R) fprintf(stderr, "%d%s ", q, lane_pos[q] ? "*" : "");
      fprintf(stderr, "} items:");
      for (int ii : pb.items) {
        const Item& it = items[ii];
        if (it.type == 1) {
          fprintf(stderr, " D[");
          for (int q = 0; q < C; ++q)
            if (run_support[it.run] >> q & 1) fprintf(stderr, "%d,", q);
          fprintf(stderr, "]");
        } else {
          fprintf(stderr, " g%d(", (int)it.g->kind);
          for (int t : it.g->t) fprintf(stderr, "%d,", loc[t]);
          fprintf(stderr, ")");
        }
      }
      fprintf(stderr, "\n");
    }
  }
  if (phs.empty() && !dest) return QK_OK;  // no gates at all: nothing to do
  if (dest) {
    // fused (permuted) store: the 5 positions landing on destination bits
    // 0..4 must be lanes of the last phase (512-B runs per warp store). If
    // the last phase holds one of them in a register slot, append a
    // layout-only phase whose register slots take the highest destinations.
    std::vector<int> by_dest;
    for (int q = 0; q < C; ++q) by_dest.push_back(q);
    std::sort(by_dest.begin(), by_dest.end(), [&](int x, int y) { return (*dest)[Q[x]] < (*dest)[Q[y]]; });
    bool ok = !phs.empty();
    for (int i = 0; i < lanes_req && i < C && ok; ++i)
      if (std::find(phs.back().R.begin(), phs.back().R.end(), by_dest[i]) != phs.back().R.end()) ok = false;
    if (!ok) {
      PhaseB pb;
      for (int i = C - 1; i >= 0 && (int)pb.R.size() < M; --i) pb.R.push_back(by_dest[i]);
      phs.push_back(pb);
    }
  }
  // 4. tables for runs (built on device at load), H scale folded into the first
  //    table. A run's table index bits are ordered for the phase that applies
  //    it: the lanes' positions first, then the register slots, so the 32
  //    lanes of a warp read one contiguous 512-B span of the table.
  cplx scale = (nh % 2 == 0) ? std::ldexp(1.0, -nh / 2) : std::ldexp(kSqrt1_2, -(nh - 1) / 2);
  std::vector<std::array<cplx, 4>> mat_f(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    const GateH* g = items[i].g;
    if (items[i].type != 0 || (g->kind != QK_U && g->kind != QK_RX && g->kind != QK_RY)) continue;
    cplx m[4], lam;
    mat2(*g, m);
    if (getenv("QK_NO_FACTOR")) {
      for (int k = 0; k < 4; ++k) mat_f[i][k] = m[k];
      continue;
    }
    factor_mat(m, mat_f[i].data(), &lam);
    scale *= lam;
  }
  bool scale_folded = (scale == cplx(1.0, 0.0));
  std::vector<int64_t> run_table(runs.size(), -1);
  std::vector<std::vector<int>> run_bidx(runs.size());
  std::vector<std::vector<int>> run_obidx(runs.size());  // physical outer bit -> table bit
  std::vector<char> run_scaled(runs.size(), 0);           // the pass scale is folded into it
  auto build_table = [&](int r, const std::vector<int>& order) -> int {
    const uint32_t S = run_support[r];
    std::vector<int> bidx(C, -1);
    int nb = 0;
    for (int p : order)
      if (p >= 0 && p < C && (S >> p & 1) && bidx[p] < 0) bidx[p] = nb++;
    for (int p = 0; p < C; ++p)
      if ((S >> p & 1) && bidx[p] < 0) bidx[p] = nb++;
    run_obidx[r].assign(64, -1);
    for (int p = 0; p < 64; ++p)
      if (run_outer[r] >> p & 1) run_obidx[r][p] = nb++;
    TableDesc td{};
    td.out = hp.pool;
    td.bits = nb;
    td.g0 = (int)hp.tgates.size();
    td.ng = (int)runs[r].size();
    td.scale = 1.0;
    td.scale_im = 0.0;
    if (!scale_folded) {
      td.scale = scale.real();
      td.scale_im = scale.imag();
      scale_folded = true;
      run_scaled[r] = 1;
    }
    for (const GateH* g : runs[r]) {
      TableGate tg{};
      tg.nt = (int)g->t.size();
      for (int j = 0; j < tg.nt; ++j) {
        const int t = g->t[j];
        tg.slot[j] = loc[t] >= 0 ? bidx[loc[t]] : run_obidx[r][t];
      }
      tg.entries = (int64_t)hp.entries.size() / 2;
      std::vector<cplx> e = diag_entries(*g);
      if (g->kind == QK_D) {
        for (auto& x : e)
          if (std::fabs(std::abs(x) - 1.0) > 1e-9) {
            emsg = "non-unitary fused gate";
            return QK_EINVAL;
          }
      }
      for (auto& x : e) {
        hp.entries.push_back(x.real());
        hp.entries.push_back(x.imag());
      }
      hp.tgates.push_back(tg);
    }
    run_table[r] = hp.pool;
    run_bidx[r] = bidx;
    hp.pool += (int64_t)1 << nb;
    hp.tables.push_back(td);
    return QK_OK;
  };
  // 5. emit phases and ops
  std::vector<int> O;
  for (int p = 0; p < nbits; ++p)
    if (std::find(Q.begin(), Q.end(), p) == Q.end()) O.push_back(p);
  // OP_QUAD data (qk_internal.h QuadLayout) of run r, applied in a phase whose
  // thread bits sit at chunk positions Tth and register slots at R
  auto build_quad = [&](int r, const std::vector<int>& Tth, const std::vector<int>& R, int64_t* out) -> int {
    const int nO = (int)O.size(), NB = C + nO, TT = (int)Tth.size();
    int idx[64];
    for (int& x : idx) x = -1;
    for (int l = 0; l < C; ++l) idx[Q[l]] = l;
    for (int k = 0; k < nO; ++k) idx[O[k]] = C + k;
    std::vector<double> lin(NB, 0.0), pr((size_t)NB * NB, 0.0);
    double ph0 = 0.0;
    for (const GateH* g : runs[r]) {
      double c, li[13], pa[13][13];
      if (!quad_terms(*g, &c, li, pa)) {
        emsg = "internal: non-quadratic gate in a quadratic run";
        return QK_ESIM;
      }
      ph0 += c;
      const int nt = (int)g->t.size();
      for (int j = 0; j < nt; ++j) {
        const int a = idx[g->t[j]];
        if (a < 0) {
          emsg = "internal: quadratic run target outside the address bits";
          return QK_ESIM;
        }
        lin[a] += li[j];
        for (int j2 = j + 1; j2 < nt; ++j2) {
          const int b2 = idx[g->t[j2]];
          if (b2 == a) lin[a] += pa[j][j2];  // x_a^2 = x_a
          else pr[(size_t)std::min(a, b2) * NB + std::max(a, b2)] += pa[j][j2];
        }
      }
    }
    auto P2 = [&](int a, int b2) { return pr[(size_t)std::min(a, b2) * NB + std::max(a, b2)]; };
    const QuadLayout L = quad_layout(C, M, nO);
    std::vector<double> d(L.total, 0.0);
    cplx sc(1.0, 0.0);
    if (!scale_folded) {
      sc = scale;
      scale_folded = true;
      run_scaled[r] = 1;
    }
    for (int tid = 0; tid < (1 << TT); ++tid) {
      double aw = 0.0;
      for (int k = 0; k < TT; ++k)
        if (tid >> k & 1)
          for (int k2 = k + 1; k2 < TT; ++k2)
            if (tid >> k2 & 1) aw += P2(Tth[k], Tth[k2]);
      const cplx w = sc * cexpi(wrap_angle(aw));
      // per-thread columns: entry k of thread tid at k * 2^(C-M) + tid (coalesced loads)
      auto cell = [&](int k) { return &d[L.thr + 2 * ((size_t)k * ((size_t)1 << (C - M)) + tid)]; };
      cell(0)[0] = w.real();
      cell(0)[1] = w.imag();
      for (int sl = 0; sl < M; ++sl) {
        double av = 0.0;
        for (int k = 0; k < TT; ++k)
          if (tid >> k & 1) av += P2(Tth[k], R[sl]);
        const cplx v = cexpi(wrap_angle(av));
        cell(1 + sl)[0] = v.real();
        cell(1 + sl)[1] = v.imag();
      }
    }
    for (int j = 0; j < (1 << M); ++j) {
      double ap = 0.0;
      for (int sa = 0; sa < M; ++sa)
        if (j >> sa & 1)
          for (int sb = sa + 1; sb < M; ++sb)
            if (j >> sb & 1) ap += P2(R[sa], R[sb]);
      const cplx v = cexpi(wrap_angle(ap));
      d[L.pj + 2 * j] = v.real();
      d[L.pj + 2 * j + 1] = v.imag();
    }
    d[L.phi0] = wrap_angle(ph0);
    for (int l = 0; l < C; ++l) d[L.at + l] = wrap_angle(lin[l]);
    for (int k = 0; k < nO; ++k) d[L.ao + k] = wrap_angle(lin[C + k]);
    for (int l = 0; l < C; ++l)
      for (int k = 0; k < nO; ++k) d[L.bto + l * nO + k] = wrap_angle(P2(l, C + k));
    for (int k = 0; k < nO; ++k)
      for (int k2 = 0; k2 < k; ++k2) d[L.boo + k * nO + k2] = wrap_angle(P2(C + k2, C + k));
    *out = hp.pool;
    hp.qcopy.emplace_back(hp.pool, std::move(d));
    hp.pool += L.total / 2;
    return QK_OK;
  };
  // OP_QLITE data of a run inside the tile: per thread E = scale * exp(i (phi0 +
  // linear terms of its set thread bits + their pairs)) and e_s = exp(i (linear
  // term of slot s + pairs with its set thread bits)); pj as for OP_QUAD.
  // masks: slots whose e_s differs from 1 for some thread, j whose pj != 1.
  auto build_qlite = [&](int r, const std::vector<int>& Tth, const std::vector<int>& R, int64_t* out,
                         uint16_t* slot_mask, uint32_t* pj_mask, uint16_t* flags) -> int {
    const int TT = (int)Tth.size();
    std::vector<double> lin(C, 0.0), pr((size_t)C * C, 0.0);
    double ph0 = 0.0;
    for (const GateH* g : runs[r]) {
      double c, li[13], pa[13][13];
      if (!quad_terms(*g, &c, li, pa)) {
        emsg = "internal: non-quadratic gate in a quadratic run";
        return QK_ESIM;
      }
      ph0 += c;
      const int nt = (int)g->t.size();
      for (int j = 0; j < nt; ++j) {
        const int a = loc[g->t[j]];
        if (a < 0) {
          emsg = "internal: tile quadratic run target outside the tile";
          return QK_ESIM;
        }
        lin[a] += li[j];
        for (int j2 = j + 1; j2 < nt; ++j2) {
          const int b2 = loc[g->t[j2]];
          if (b2 == a) lin[a] += pa[j][j2];
          else pr[(size_t)std::min(a, b2) * C + std::max(a, b2)] += pa[j][j2];
        }
      }
    }
    auto P2 = [&](int a, int b2) { return pr[(size_t)std::min(a, b2) * C + std::max(a, b2)]; };
    const QuadLayout L = quad_layout(C, M, 0);
    std::vector<double> d(L.total, 0.0);
    cplx sc(1.0, 0.0);
    if (!scale_folded) {
      sc = scale;
      scale_folded = true;
      run_scaled[r] = 1;
    }
    *slot_mask = 0;
    *pj_mask = 0;
    for (int tid = 0; tid < (1 << TT); ++tid) {
      double ae = ph0;
      for (int k = 0; k < TT; ++k)
        if (tid >> k & 1) {
          ae += lin[Tth[k]];
          for (int k2 = k + 1; k2 < TT; ++k2)
            if (tid >> k2 & 1) ae += P2(Tth[k], Tth[k2]);
        }
      const cplx e = sc * cexpi(wrap_angle(ae));
      auto cell = [&](int k) { return &d[L.thr + 2 * ((size_t)k * ((size_t)1 << (C - M)) + tid)]; };
      cell(0)[0] = e.real();
      cell(0)[1] = e.imag();
      for (int sl = 0; sl < M; ++sl) {
        double av = lin[R[sl]];
        for (int k = 0; k < TT; ++k)
          if (tid >> k & 1) av += P2(Tth[k], R[sl]);
        av = wrap_angle(av);
        if (av != 0.0) *slot_mask |= (uint16_t)(1u << sl);
        const cplx v = cexpi(av);
        cell(1 + sl)[0] = v.real();
        cell(1 + sl)[1] = v.imag();
      }
    }
    for (int j = 0; j < (1 << M); ++j) {
      double ap = 0.0;
      for (int sa = 0; sa < M; ++sa)
        if (j >> sa & 1)
          for (int sb = sa + 1; sb < M; ++sb)
            if (j >> sb & 1) ap += P2(R[sa], R[sb]);
      ap = wrap_angle(ap);
      if (ap != 0.0) *pj_mask |= 1u << j;
      const cplx v = cexpi(ap);
      d[L.pj + 2 * j] = v.real();
      d[L.pj + 2 * j + 1] = v.imag();
    }
    // every thread's row the same (the run reads only slots): the 2^M
    // products become constants in pj (flag 1); otherwise flag 2 when E is
    // exactly 1 for every thread (no thread-only or global phase)
    bool same = true, e_one = true;
    const size_t NT = (size_t)1 << (C - M);
    auto at = [&](int tid, int k) { return &d[L.thr + 2 * ((size_t)k * NT + tid)]; };
    for (int tid = 0; tid < (1 << TT); ++tid) {
      for (int k = 0; k <= M; ++k)
        same = same && at(tid, k)[0] == at(0, k)[0] && at(tid, k)[1] == at(0, k)[1];
      e_one = e_one && at(tid, 0)[0] == 1.0 && at(tid, 0)[1] == 0.0;
    }
    *flags = 0;
    if (same) {
      *flags = 1;
      *pj_mask = 0;
      *slot_mask = 0;
      for (int j = 0; j < (1 << M); ++j) {
        cplx f(at(0, 0)[0], at(0, 0)[1]);
        for (int sl = 0; sl < M; ++sl)
          if (j >> sl & 1) f *= cplx(at(0, 1 + sl)[0], at(0, 1 + sl)[1]);
        f *= cplx(d[L.pj + 2 * j], d[L.pj + 2 * j + 1]);
        d[L.pj + 2 * j] = f.real();
        d[L.pj + 2 * j + 1] = f.imag();
        if (f != cplx(1.0, 0.0)) *pj_mask |= 1u << j;
      }
    } else if (e_one) {
      *flags = 2;
    }
    *out = hp.pool;
    hp.qcopy.emplace_back(hp.pool, std::move(d));
    hp.pool += L.total / 2;
    return QK_OK;
  };
  // tile-only quadratic runs of a quad-enabled pass become OP_QLITE (a few
  // per-thread loads instead of 16 table gathers per run; QK_QLITE_TABLE1:
  // the first keeps its table, which the specialised kernel may hoist)
  bool tile_table_used = false;
  PassDesc pd{};
  pd.C = C;
  pd.M = M;
  pd.phase0 = (int)hp.phases.size();
  pd.nphases = (int)phs.size();
  if ((int)O.size() > kMaxOuter) {
    emsg = "too many outer bits";
    return QK_ESIM;
  }
  pd.nouter = (int)O.size();
  for (size_t k = 0; k < O.size(); ++k) pd.opos[k] = (uint8_t)O[k];
  pd.ncta = ncta_override ? ncta_override : (1ull << O.size());
  for (size_t ph = 0; ph < phs.size(); ++ph) {
    const PhaseB& pb = phs[ph];
    std::vector<int> T;
    for (int p = 0; p < C; ++p)
      if (std::find(pb.R.begin(), pb.R.end(), p) == pb.R.end()) T.push_back(p);
    if (dest && ph + 1 == phs.size()) {
      // last phase of a fused pass: lanes on the source bits that land lowest
      std::stable_sort(T.begin(), T.end(), [&](int x, int y) { return (*dest)[Q[x]] < (*dest)[Q[y]]; });
    } else {
      T = order_tpos(T);
    }
    PhaseDesc D{};
    D.tbits = C - M;
    for (int k = 0; k < D.tbits; ++k) {
      D.tpos[k] = (uint8_t)T[k];
      D.taddr[k] = 1ull << Q[T[k]];
    }
    for (int j = 0; j < (1 << M); ++j) {
      uint32_t rl = 0;
      uint64_t ra = 0;
      for (int s = 0; s < M; ++s)
        if (j >> s & 1) {
          rl |= 1u << pb.R[s];
          ra |= 1ull << Q[pb.R[s]];
        }
      D.rloc[j] = (uint16_t)rl;
      D.raddr[j] = ra;
    }
    D.op_begin = (int)hp.ops.size();
    auto slot = [&](int lpos) {
      for (int s = 0; s < M; ++s)
        if (pb.R[s] == lpos) return s;
      return -1;
    };
    for (int ii : pb.items) {
      const Item& it = items[ii];
      OpDesc op{};
      if (it.type == 1 && run_quad[it.run] && (run_outer[it.run] || popc(run_support[it.run]) > 14)) {
        // one OP_QUAD for the whole run (tile and chunk bits)
        std::vector<int> Tth(T.begin(), T.end());
        int64_t off = 0;
        int rc = build_quad(it.run, Tth, pb.R, &off);
        if (rc) return rc;
        op.code = OP_QUAD;
        op.table = off;
      } else if (it.type == 1 && allow_quad && run_quad[it.run] && (tile_table_used || !getenv("QK_QLITE_TABLE1")) &&
                 !getenv("QK_NO_QLITE")) {
        std::vector<int> Tth(T.begin(), T.end());
        int64_t off = 0;
        uint16_t sm = 0, fl = 0;
        uint32_t pm = 0;
        int rc = build_qlite(it.run, Tth, pb.R, &off, &sm, &pm, &fl);
        if (rc) return rc;
        op.code = OP_QLITE;
        op.table = off;
        op.pr[0] = sm;
        op.pr[1] = (uint16_t)(pm & 0xffffu);
        op.pr[3] = (uint16_t)(pm >> 16);  // (32 register amplitudes)
        op.pr[2] = fl;
      } else if (it.type == 1) {
        if (allow_quad && run_quad[it.run]) tile_table_used = true;
        const uint32_t S = run_support[it.run];
        if (run_table[it.run] < 0) {
          std::vector<int> order(T.begin(), T.end());
          for (int q : pb.R) order.push_back(q);
          int rc = build_table(it.run, order);
          if (rc) return rc;
        }
        const std::vector<int>& bidx = run_bidx[it.run];
        op.code = OP_DIAG;
        op.table = run_table[it.run];
        for (int k = 0; k < D.tbits; ++k) op.tcontrib[k] = (S >> T[k] & 1) ? (uint16_t)(1u << bidx[T[k]]) : 0;
        for (int j = 0; j < (1 << M); ++j) {
          uint32_t v = 0;
          for (int s2 = 0; s2 < M; ++s2)
            if ((j >> s2 & 1) && (S >> pb.R[s2] & 1)) v |= 1u << bidx[pb.R[s2]];
          op.pr[j] = (uint16_t)v;
        }
        for (size_t k = 0; k < O.size(); ++k)
          if (run_outer[it.run] >> O[k] & 1) {
            op.co_k[op.nco] = (uint8_t)k;
            op.co_v[op.nco] = (uint16_t)(1u << run_obidx[it.run][O[k]]);
            ++op.nco;
          }
        // register amplitudes whose table entry is exactly 1 whatever the
        // thread and chunk bits: every gate of the run has entry 1 for every
        // completion of its targets outside the register slots (a CP whose
        // register-slot target is 0). The specialised kernel skips them.
        if (!run_scaled[it.run] && !getenv("QK_NO_UNIT_SKIP")) {
          for (int j = 0; j < (1 << M); ++j) {
            bool one = true;
            for (const GateH* g : runs[it.run]) {
              const int nt = (int)g->t.size();
              if (nt > 8) {
                one = false;
                break;
              }
              uint32_t fixed_mask = 0, fixed_val = 0;
              for (int i = 0; i < nt; ++i) {
                const int lp = loc[g->t[i]];
                const int sl = lp >= 0 ? slot(lp) : -1;
                if (sl >= 0) {
                  fixed_mask |= 1u << (nt - 1 - i);
                  if (j >> sl & 1) fixed_val |= 1u << (nt - 1 - i);
                }
              }
              const std::vector<cplx> e = diag_entries(*g);
              for (uint32_t idx = 0; idx < (1u << nt) && one; ++idx)
                if ((idx & fixed_mask) == fixed_val && !(idx < e.size() && e[idx] == cplx(1.0, 0.0))) one = false;
              if (!one) break;
            }
            if (one) op.unit |= (uint16_t)(1u << j);
          }
        }
      } else {
        const GateH* g = it.g;
        switch (g->kind) {
          case QK_H: op.code = OP_H; op.r0 = slot(loc[g->t[0]]); break;
          case QK_X: op.code = OP_X; op.r0 = slot(loc[g->t[0]]); break;
          case QK_U:
          case QK_RX:
          case QK_RY: {
            op.code = OP_MAT;
            op.r0 = slot(loc[g->t[0]]);
            op.coef = (int)hp.coef.size();
            for (auto& x : mat_f[ii]) {
              hp.coef.push_back(x.real());
              hp.coef.push_back(x.imag());
            }
            break;
          }
          case QK_CX: {
            op.code = OP_CX;
            op.r0 = slot(loc[g->t[1]]);
            const int cs = slot(loc[g->t[0]]);
            if (cs >= 0) {
              op.ctrl_reg = 1;
              op.r1 = cs;
            } else {
              op.ctrl = loc[g->t[0]];
            }
            break;
          }
          case QK_SWAP: {
            op.code = OP_SWAP;
            const int s0 = slot(loc[g->t[0]]), s1 = slot(loc[g->t[1]]);
            op.r0 = std::min(s0, s1);
            op.r1 = std::max(s0, s1);
            break;
          }
          default:
            emsg = "no kernel for gate kind";
            return QK_ESIM;
        }
      }
      hp.ops.push_back(op);
    }
    if (ph + 1 == phs.size() && !scale_folded) {
      OpDesc op{};
      op.code = OP_SCALE;
      op.coef = (int)hp.coef.size();
      hp.coef.push_back(scale.real());
      hp.coef.push_back(scale.imag());
      hp.ops.push_back(op);
      scale_folded = true;
    }
    D.op_end = (int)hp.ops.size();
    hp.phases.push_back(D);
  }
  hp.passes.push_back(pd);
  return QK_OK;
}

// Chunk-address sets for a block: one pass with Q = [0, C) when every target
// fits kMaxC (chunk-local path, simulator.py:481-492); otherwise gates are
// grouped into memory-level passes whose Q = targets + lowest free bits
// (simulator.py:494-511, same per-amplitude gate order).
// chunk width of a block's single pass (0 if the block needs memory-level passes)
int block_chunk_width(const InstrH& ins, int L, int cmin = 10) {
  int maxt = -1;
  for (auto& g : ins.gates)
    for (int t : g.t) maxt = std::max(maxt, t);
  if (maxt < 0 || maxt >= kMaxC || maxt >= L) return 0;
  int C = std::max(maxt + 1, std::min(L, cmin));
  C = std::min(C, std::min(L, kMaxC));
  if (C > 12 && maxt < 12) C = 12;
  return C;
}

int compile_block(HostPlan& hp, const InstrH& ins, int L, int nbits, InstrPlan& ip,
                  std::string& emsg, int cmin = 10, int cfix = 0) {
  // a cluster-exchange store permutes through shared memory: no lane constraints
  const std::vector<int>* dest = (ip.dest.empty() || !ip.xspec.empty()) ? nullptr : &ip.dest;
  int maxt = -1;
  for (auto& g : ins.gates)
    for (int t : g.t) maxt = std::max(maxt, t);
  ip.pass0 = (int)hp.passes.size();
  if (maxt < 0 && !(dest && cfix)) return QK_OK;
  if (maxt >= L) {
    emsg = "gate target " + std::to_string(maxt) + " beyond local range";
    return QK_ESIM;
  }
  const int low_keep = std::min(3, L);
  if (maxt < kMaxC) {
    const int C = cfix ? std::max(cfix, block_chunk_width(ins, L, cmin)) : block_chunk_width(ins, L, cmin);
    std::vector<int> Q;
    for (int p = 0; p < C; ++p) Q.push_back(p);
    std::vector<const GateH*> gs;
    for (auto& g : ins.gates) gs.push_back(&g);
    int rc = compile_pass(hp, gs, Q, nbits, 0, emsg, dest);
    if (rc) return rc;
  } else {
    size_t i = 0;
    while (i < ins.gates.size()) {
      uint64_t U = 0;
      std::vector<const GateH*> gs;
      while (i < ins.gates.size()) {
        uint64_t tm = 0;
        for (int t : ins.gates[i].t) tm |= 1ull << t;
        if (!gs.empty() && popc(U | tm) > kMaxC - low_keep) break;
        U |= tm;
        gs.push_back(&ins.gates[i]);
        ++i;
      }
      const int C = std::min(L, std::max(popc(U) + low_keep, std::min(L, cmin)));
      std::vector<int> Q;
      for (int p = 0; p < L; ++p)
        if (U >> p & 1) Q.push_back(p);
      for (int p = 0; p < L && (int)Q.size() < std::min(C, kMaxC); ++p)
        if (!(U >> p & 1)) Q.push_back(p);
      std::sort(Q.begin(), Q.end());
      int rc = compile_pass(hp, gs, Q, nbits, 0, emsg);
      if (rc) return rc;
    }
  }
  ip.npass = (int)hp.passes.size() - ip.pass0;
  ip.bytes = 32.0 * std::ldexp(1.0, nbits) * ip.npass;
  return QK_OK;
}

// new[i] = old[bitswap(i, A, B)] over a vector of nbits address bits
int compile_sqs(HostPlan& hp, const std::vector<int>& A0, const std::vector<int>& B0, int nbits,
                bool paired = false) {
  // pairs sorted(A)[k] <-> sorted(B)[k] (simulator.py:85); `paired`: A[k] <-> B[k] as given
  std::vector<int> A = A0, B = B0;
  if (!paired) {
    std::sort(A.begin(), A.end());
    std::sort(B.begin(), B.end());
  }
  int partner[64];
  for (int& x : partner) x = -1;
  for (size_t k = 0; k < A.size(); ++k) {
    partner[A[k]] = B[k];
    partner[B[k]] = A[k];
  }
  const int w = std::min(kSqsW, nbits);
  std::vector<int> V;
  auto inV = [&](int p) { return std::find(V.begin(), V.end(), p) != V.end(); };
  for (int p = 0; p < w; ++p) V.push_back(p);
  for (int p = 0; p < w; ++p)
    if (partner[p] >= w) V.push_back(partner[p]);
  // fillers: grow the tile to 2^10 amplitudes, keeping pairs whole
  const int target = std::min(nbits, 10);
  for (int q = w; q < nbits && (int)V.size() < target; ++q) {
    if (inV(q)) continue;
    if (partner[q] < 0) {
      V.push_back(q);
    } else if (!inV(partner[q]) && V.size() + 2 <= 10) {
      V.push_back(q);
      V.push_back(partner[q]);
    }
  }
  std::sort(V.begin() + w, V.end());
  SqsDesc sd{};
  sd.w = w;
  sd.nv = (int)V.size();
  for (int b = 0; b < sd.nv; ++b) sd.vpos[b] = (uint8_t)V[b];
  std::vector<int> O;
  for (int p = 0; p < nbits; ++p)
    if (!inV(p)) O.push_back(p);
  sd.nouter = (int)O.size();
  for (size_t k = 0; k < O.size(); ++k) sd.opos[k] = (uint8_t)O[k];
  auto vidx = [&](int p) { return (int)(std::find(V.begin(), V.end(), p) - V.begin()); };
  auto oidx = [&](int p) { return (int)(std::find(O.begin(), O.end(), p) - O.begin()); };
  for (size_t k = 0; k < A.size(); ++k) {
    if (inV(A[k])) {
      sd.va[sd.nvp] = (uint8_t)vidx(A[k]);
      sd.vb[sd.nvp] = (uint8_t)vidx(B[k]);
      ++sd.nvp;
    } else {
      sd.oa[sd.nop] = (uint8_t)oidx(A[k]);
      sd.ob[sd.nop] = (uint8_t)oidx(B[k]);
      ++sd.nop;
    }
  }
  sd.ident = sd.nvp == 0;
  hp.sqs.push_back(sd);
  return (int)hp.sqs.size() - 1;
}

// reference shift_pairs (simulator.py:91-106): iteration-order remap for ranges
void shift_pairs(const std::vector<int>& a_bits, const std::vector<int>& b_bits, int cl, int n_local,
                 std::vector<int>& P, std::vector<int>& Qo) {
  std::vector<int> a = a_bits, b = b_bits;
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  int na = 0, nb = 0;
  for (int x : a) na += x < cl;
  for (int x : b) nb += x < cl;
  const int d = std::abs(na - nb);
  P.clear();
  Qo.clear();
  if (d == 0) return;
  const std::vector<int>& donors = na > nb ? b_bits : a_bits;
  std::vector<int> dout;
  for (int x : donors)
    if (x >= cl) dout.push_back(x);
  std::sort(dout.begin(), dout.end());
  std::vector<int> p0;
  for (int x = cl; x < cl + d; ++x)
    if (x < n_local) p0.push_back(x);
  std::vector<int> q0(dout.begin(), dout.begin() + std::min(dout.size(), p0.size()));
  p0.resize(q0.size());
  for (size_t i = 0; i < p0.size(); ++i)
    if (std::find(q0.begin(), q0.end(), p0[i]) == q0.end()) P.push_back(p0[i]);
  for (size_t i = 0; i < q0.size(); ++i)
    if (std::find(p0.begin(), p0.end(), q0[i]) == p0.end()) Qo.push_back(q0[i]);
}

}  // namespace

// ---------------------------------------------------------------------------
// handle

constexpr int kFreshBits = 13;  // widest TMA chunk: qk_reset writes this prefix

struct qk_sim {
  int n = 0, r = 0, b = 0, device = 0;
  int rank_lo = 0, count = 1;
  int L = 0, nbits = 0;  // local qubits, address bits held by this handle
  bool gbg = false;      // loaded by qk_load_gate_by_gate: one full sweep per gate
  // |0...0> after qk_reset with only the first kFreshAmps amplitudes written:
  // the first TMA pass of a run reads every other chunk as out-of-bounds zeros
  // (no HBM reads), anything else writes the whole state first (ensure_full)
  bool oop_sqs = false;  // relabeled program: unfused SQS permute into the second buffer
  // fused norm: the program's last data-writing pass sums |amp|^2 per consumer
  // group into d_nrm; valid until anything writes the state
  double* d_nrm = nullptr;
  int norm_pass = -1, nrm_parts = 0;
  bool norm_valid = false;
  bool fresh = false;
  // Zero support: during a run from a reset state every amplitude at a
  // physical address >= 2^zbits is exactly zero (64: unknown). A TMA pass then
  // loads through a view bounded at 2^zbits, so the TMA unit zero-fills the
  // rest without HBM reads, and the bound grows to the pass's highest tile bit
  // (its gates and in-tile permutation touch no other bit).
  int zbits = 64;
  // memory of the current buffer at amplitudes >= 2^zmem was never written in
  // this run (logically zero; 64: all written). A pass that reads through a
  // bounded view skips the chunks above its next bound (they are zero and no
  // later pass reads them); any reader outside the passes fills them first.
  int zmem = 64, zmem_next = 64;
  double fresh_saved = 0;  // read bytes skipped this way (kept out of the stats)
  std::vector<double> saved_i;  // per instruction of the last run: read bytes skipped
  double* state = nullptr;      // == bufs[cur]
  double* bufs[2] = {nullptr, nullptr};  // bufs[1]: out-of-place target of fused passes
  int cur = 0;
  size_t amps = 0;
  cudaStream_t stream = nullptr;
  // program
  std::vector<InstrH> prog;
  std::vector<InstrPlan> iplan;
  HostPlan hp;
  std::vector<int> final_perm;
  // lazy in-place layout: reference address bit q of the handle's state lives
  // at physical bit lay[q]; qk_run leaves lay_final (the plan's end layout)
  std::vector<int> lay, lay_final;
  // the plan's layout at its start (identity unless the first-use placement
  // applies): reference bit q at physical bit plan_lay0[q]; free on |0...0>
  std::vector<int> plan_lay0;
  std::vector<CUtensorMap> lazy_map1;  // per TMA pass: the strided view of bufs[1] (lazy passes)
  // device plan
  void* blob = nullptr;
  size_t blob_bytes = 0;
  PassDesc* d_pass = nullptr;
  PhaseDesc* d_phase = nullptr;
  OpDesc* d_ops = nullptr;
  double* d_coef = nullptr;
  SqsDesc* d_sqs = nullptr;
  double* d_pool = nullptr;
  size_t pool_bytes = 0;
  // scratch
  double* d_partial = nullptr;
  double* d_scalar = nullptr;
  void* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  // timing
  std::vector<cudaEvent_t> events;
  cudaEvent_t marks[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int per_launch = 0;
  // per kernel class: block passes, SQS, CSQS, cluster-exchange block passes
  double stat_ms[4] = {0, 0, 0, 0};
  double stat_launch[4] = {0, 0, 0, 0};
  double stat_bytes[4] = {0, 0, 0, 0};
  double stat_overlapped = 0;  // exchanges that ran overlapped with their neighbour passes
  // persistent TMA passes
  int num_sms = 148;
  bool allow_tma = true;
  CUtensorMap maps[2][6];
  bool map_ok[2][6] = {{false, false, false, false, false, false}, {false, false, false, false, false, false}};
  std::vector<TmaParams> tma;
  std::vector<int> pass_tma;
  std::vector<void*> pass_jit;                 // specialised kernel per pass (or nullptr)
  std::vector<std::vector<uint64_t>> jit_blob;  // its parameter block (map/state/out patched at launch)
  // specialised variants per pass (qk_jit.cpp variant bits) and the tuning key
  struct JitVar {
    int variant;
    void* kern;
    std::vector<uint64_t> blob;
  };
  std::vector<std::vector<JitVar>> pass_var;
  std::vector<std::string> pass_key;
  std::vector<int> tuning;           // per pass: index into pass_var being timed this run, -1 none
  std::vector<cudaEvent_t> tune_ev;  // per pass: start / end of the timed variant
  // multi-process
  qk_barrier_fn barrier = nullptr;
  void* barrier_ctx = nullptr;
  std::vector<double*> peers;   // by shard index: the peer's bufs[0]
  std::vector<double*> peers1;  // the peer's bufs[1] (double-buffered shards)
  int nshards = 1, shard = 0;
  // device-side exchange barrier: flag array behind bufs[0] (one slot per
  // shard), the peers' arrays through their mappings, and a per-handle epoch
  // (every shard runs the same exchanges, so the epochs agree)
  unsigned long long* flags = nullptr;
  std::vector<unsigned long long*> peer_flags;
  int* d_err = nullptr;
  bool ipc_mapped = false;     // peers[] came from cudaIpcOpenMemHandle (closed at destroy)
  // group handle (qk_create_multi): one member shard per device, this
  // handle owns them and holds no state of its own
  std::vector<qk_sim*> members;
  std::vector<char> skipped;   // per instruction of the last run: a swap of the fresh |0...0> (identity)
  // exchange overlap (QK_NO_OVERLAP disables): second stream for the peer
  // swaps, pass -> CSQS maps, per-part events, the CSQS whose pre-pass ran split
  cudaStream_t comm = nullptr;
  std::vector<int> ovl_by_p, ovl_by_q;
  cudaEvent_t ev_part[8] = {}, ev_x[8] = {};
  int ovl_live = -1;
  int overlap = 0;  // pipeline exchanges with their neighbour passes (peers on other GPUs; qk_set_overlap)
  std::vector<unsigned long long> pair_epoch;  // device barrier meetings per peer shard
  // host-only planning (qk_plan_dry): no device memory, tensor maps or kernel
  // builds; upload_plan stops after writing the generated pass sources
  bool dry = false;
  std::string dry_dir;
  // CUDA-graph replay of small runs (qk_run, graph_run): the launches of the
  // steps of a run from one host-side start state, captured once and replayed;
  // the host state the steps leave is kept with the graph and re-applied
  struct HostRunState {
    bool fresh = false;
    int zbits = 64, zmem = 64, zmem_next = 64, cur = 0, ovl_live = -1;
    double fresh_saved = 0;
    std::vector<double> saved_i;
    std::vector<char> skipped;
    std::vector<int> lay;
    size_t first_exec = 0;
  };
  struct GraphEnt {
    std::vector<int64_t> key;  // start state (graph_key) the graph was captured from
    cudaGraphExec_t exec = nullptr;
    HostRunState post;         // host state after its steps
  };
  std::deque<GraphEnt> graphs;                 // most recent last, at most kGraphs
  std::deque<std::vector<int64_t>> gseen;      // start states of recent eager runs
  uint64_t prog_gen = 0;      // identity of the uploaded plan (a graph holds its pointers)
  bool capturing = false;     // steps record no per-instruction events
  bool graph_timed = false;   // the run to finish was a replay: events[0..1] bracket it
  int graph_fails = 0;
  std::vector<double> last_ms;  // per instruction, the last eager run (replay time attribution)
  double stat_graph = 0;        // runs replayed from a graph
};

constexpr size_t kFlagBytes = 4096;  // 64 shards x 8 B, padded

namespace {

int ensure_scratch(qk_sim* s, size_t bytes) {
  if (s->scratch_bytes >= bytes) return QK_OK;
  if (s->d_scratch) cudaFree(s->d_scratch);
  s->d_scratch = nullptr;
  s->scratch_bytes = 0;
  CUDA_TRY(cudaMalloc(&s->d_scratch, bytes));
  s->scratch_bytes = bytes;
  return QK_OK;
}

template <class T>
size_t push_section(std::vector<char>& buf, const std::vector<T>& v) {
  size_t off = (buf.size() + 255) & ~(size_t)255;
  buf.resize(off + v.size() * sizeof(T));
  if (!v.empty()) memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D view of the state: rows of 8 amplitudes (16 doubles = 128 B), SWIZZLE_128B
const CUtensorMap* state_map(qk_sim* s, int buf, int box_rows) {
  const int slot = __builtin_ctz((unsigned)box_rows) - 3;  // 8..256 -> 0..5
  if (slot < 0 || slot > 5 || !s->bufs[buf]) return nullptr;
  if (s->dry) return &s->maps[buf][slot];
  if (!s->map_ok[buf][slot]) {
    auto fn = encode_fn();
    if (!fn || s->nbits < 3) return nullptr;
    cuuint64_t dims[2] = {16, (cuuint64_t)1 << (s->nbits - 3)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&s->maps[buf][slot], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, s->bufs[buf], dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return nullptr;
    s->map_ok[buf][slot] = true;
  }
  return &s->maps[buf][slot];
}

// A pass's load view of `buf` with only addresses < 2^zb in bounds (every
// other box is zero-filled by the TMA unit without touching HBM): on a fresh
// |0...0> (zb = kFreshBits) those are the only amplitudes qk_reset wrote, and
// later in a run from reset they are the only ones that can be nonzero.
bool fresh_map(qk_sim* s, const TmaParams& tp, int zb, double* buf, CUtensorMap* out) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  int rank;
  if (tp.lazy) {
    TileDims td{};
    if (!tile_dims(tp.tbit, tp.C, tp.nbits, &td, tp.rowbits)) return false;
    rank = td.rank;
    for (int j = 0; j < rank; ++j) {
      const int keep = std::max(0, std::min(td.len[j], zb - td.lo[j]));
      dims[j] = j == 0 ? (cuuint64_t)(2 << td.len[0]) : (cuuint64_t)1 << keep;
      if (j) strides[j - 1] = (cuuint64_t)16 << td.lo[j];
      box[j] = (cuuint32_t)td.box[j];
    }
  } else {
    rank = 2;
    dims[0] = 16;
    dims[1] = (cuuint64_t)1 << (zb - 3);
    strides[0] = 128;
    box[0] = 16;
    box[1] = (cuuint32_t)tp.box_rows;
  }
  return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, buf, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            (tp.lazy && tp.rowbits == 2) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Write the whole |0...0> state of a fresh handle (before anything but the
// first TMA pass reads or writes it).
int ensure_full(qk_sim* s) {
  s->zbits = 64;  // the caller reads or writes the state outside a pass
  if (!s->fresh) {
    if (s->zmem < s->nbits) {  // the part the skipping passes never wrote
      const size_t lo = (size_t)1 << s->zmem;
      s->zmem = 64;
      CUDA_TRY(cudaMemsetAsync(s->bufs[s->cur] + 2 * lo, 0, (s->amps - lo) * 16, s->stream));
    }
    return QK_OK;
  }
  s->fresh = false;
  s->zmem = 64;
  int rc = launch_fill_zero_one(s->bufs[0], s->amps, s->rank_lo == 0, (CUstream_st*)s->stream);
  return rc ? fail(QK_ECUDA, "state fill failed") : QK_OK;
}

// N-D strided view of `buf` for the tile of a lazy pass (qk_internal.h tile_dims)
bool g_dry_maps = false;  // qk_plan_dry: tensor maps are not encoded (no driver needed)

bool encode_lazy_map(const TmaParams& tp, double* buf, CUtensorMap* out) {
  TileDims td{};
  if (!tile_dims(tp.tbit, tp.C, tp.nbits, &td, tp.rowbits)) return false;
  if (g_dry_maps) return true;
  auto fn = encode_fn();
  if (!fn || !buf) return false;
  cuuint64_t dims[5];
  cuuint64_t strides[4];
  cuuint32_t box[5], es[5];
  for (int j = 0; j < td.rank; ++j) {
    dims[j] = j == 0 ? (cuuint64_t)(2 << td.len[0]) : (cuuint64_t)1 << td.len[j];
    if (j) strides[j - 1] = (cuuint64_t)16 << td.lo[j];
    box[j] = (cuuint32_t)td.box[j];
    es[j] = 1;
  }
  return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, td.rank, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            tp.rowbits == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tma(qk_sim* s, const PassDesc& pd, TmaParams& tp, const std::vector<int>* dest,
              const std::vector<int>* xspec = nullptr, const std::vector<int>* tile = nullptr) {
  if (getenv("QK_NO_TMA")) return false;
  const bool lz = tile && !tile->empty();
  if (pd.M < 3 || pd.M > kMaxTM || pd.C < 9 || pd.C > ((lz || getenv("QK_TMA13")) ? 13 : 12) || pd.nphases > kTMaxPh ||
      s->nbits > 34)
    return false;
  if (pd.nouter != s->nbits - pd.C) return false;
  std::vector<int> vdest;
  TileDims td{};
  if (lz) {
    // strided tile: chunk-local bit x <-> physical tile[x]; outer (chunk index)
    // bit k <-> the k-th non-tile bit; stored in place through the permuted path
    uint8_t tb[16];
    for (int x = 0; x < pd.C; ++x) tb[x] = (uint8_t)(*tile)[x];
    const int w = (pd.C > 2 && (*tile)[2] == 2) ? 3 : 2;
    if ((int)tile->size() != pd.C || !tile_dims(tb, pd.C, s->nbits, &td, w)) return false;
    std::vector<char> in(s->nbits, 0);
    for (int p : *tile) in[p] = 1;
    for (int p : *tile) vdest.push_back(dest ? (*dest)[p] : p);  // in-tile store permutation
    for (int p = 0; p < s->nbits; ++p)
      if (!in[p]) vdest.push_back(p);
    dest = &vdest;
  } else {
    for (int k = 0; k < pd.nouter; ++k)
      if (pd.opos[k] != pd.C + k) return false;
  }
  const HostPlan& hp = s->hp;
  const int box_rows = std::min(256, 1 << (pd.C - 3));
  memset(&tp, 0, sizeof tp);
  if (lz) {
    tp.lazy = 1;
    tp.rowbits = ((*tile)[2] == 2) ? 3 : 2;
    tp.C = pd.C;
    tp.nbits = s->nbits;
    for (int x = 0; x < pd.C; ++x) tp.tbit[x] = (uint8_t)(*tile)[x];
    if (!encode_lazy_map(tp, s->bufs[0], &tp.map)) return false;
  } else if (!state_map(s, 0, std::min(256, 1 << (pd.C - 3)))) {
    return false;
  }
  tp.tabs = s->d_pool;
  tp.direct_store = (getenv("QK_TMA_STORE") && !dest) ? 0 : 1;
  tp.nbits = s->nbits;
  if (dest) {
    tp.permuted = 1;
    for (int q = 0; q < s->nbits; ++q) tp.dpos[q] = (uint8_t)(*dest)[q];
    const PhaseDesc& D = s->hp.phases[pd.phase0 + pd.nphases - 1];
    for (int k = 0; k < D.tbits; ++k) tp.ldst_t[k] = 1ull << (*dest)[D.tpos[k]];
    for (int j = 0; j < (1 << pd.M); ++j) {
      uint64_t o = 0;
      for (int b = 0; b < pd.C; ++b)
        if (D.rloc[j] >> b & 1) o |= 1ull << (*dest)[b];
      tp.ldst_r[j] = o;
    }
  }
  tp.nchunks = 1ull << (s->nbits - pd.C);
  if (xspec && !xspec->empty()) {
    tp.xbits = (int)xspec->size();
    for (int k = 0; k < tp.xbits; ++k) tp.xpos[k] = (uint8_t)(*xspec)[k];
  }
  tp.C = pd.C;
  tp.M = pd.M;
  tp.nphases = pd.nphases;
  tp.box_rows = box_rows;
  tp.ntma = (1 << (pd.C - 3)) / box_rows;
  {
    // Two or more diagonal tables (64 KiB each at 12 bits) are gathered per
    // amplitude; with two 64-KiB stages instead of three the L1 keeps them
    // (QAOA30's 3-table passes: 6.7 -> 5.9 ms; light 1-table passes lose ~0.2 ms).
    // Three-phase passes with dense 2x2 gates gain too (~0.2 ms each).
    int ndiag = 0, nmat = 0;
    for (int ph = 0; ph < pd.nphases; ++ph) {
      const PhaseDesc& D = hp.phases[pd.phase0 + ph];
      for (int o = D.op_begin; o < D.op_end; ++o) {
        ndiag += hp.ops[o].code == OP_DIAG;
        nmat += hp.ops[o].code == OP_MAT;
      }
    }
    // (the dense-gate cap predates the quadratic phases: with tables replaced
    // by OP_QUAD / OP_QLITE, QAOA30's passes run 3% faster on three stages;
    // QK_SMAX_MAT=1 restores it)
    const bool l1_tables = ndiag >= 2 || (getenv("QK_SMAX_MAT") && pd.nphases >= 3 && nmat >= 5);
    // Narrower chunks with any table keep 128 KiB of stages (QFT30: 38.0 ->
    // 34.9 ms with 8 instead of 12 16-KiB stages; 4 stages starve the loads).
    if (!tp.xbits && !getenv("QK_NO_SMAX")) {
      if (pd.C == 12 && l1_tables) tp.smax = 2;
      else if (pd.C <= 11 && ndiag >= 1) tp.smax = (128 << 10) / (16 << pd.C);
    }
  }
  if (tma_smem_bytes(pd.C, pd.M, &tp.ng, &tp.stages, tp.smax) < 0) return false;
  int ncoef = 0, nsteps = 0;
  for (int ph = 0; ph < pd.nphases; ++ph) {
    const PhaseDesc& D = hp.phases[pd.phase0 + ph];
    TPhase& T = tp.ph[ph];
    for (int k = 0; k < 12; ++k) T.tpos[k] = D.tpos[k];
    for (int j = 0; j < kMaxNA; ++j) T.rloc[j] = D.rloc[j];
    T.op_begin = (int16_t)nsteps;
    TOp* cur1q = nullptr;  // open STEP_1Q (one-qubit gates on distinct slots commute)
    for (int o = D.op_begin; o < D.op_end; ++o) {
      const OpDesc& op = hp.ops[o];
      const bool one_q = op.code == OP_H || op.code == OP_X || op.code == OP_MAT;
      if (one_q && cur1q && cur1q->st[op.r0] == 0) {
        // joins the open step
      } else {
        if (nsteps >= kTMaxOps) return false;
        TOp& t = tp.ops[nsteps++];
        memset(&t, 0, sizeof t);
        cur1q = nullptr;
        if (one_q) {
          t.code = STEP_1Q;
          cur1q = &t;
        } else {
          t.code = (int8_t)op.code;
          t.r0 = (int8_t)op.r0;
          t.r1 = (int8_t)op.r1;
          t.creg = (int8_t)op.ctrl_reg;
          t.ctrl = (int16_t)op.ctrl;
          if (op.table > INT32_MAX) return false;
          t.table = (int32_t)op.table;
          for (int k = 0; k < 12; ++k) t.tcontrib[k] = op.tcontrib[k];
          for (int j = 0; j < kMaxNA; ++j) t.pr[j] = op.pr[j];
          t.nco = (int8_t)op.nco;
          t.unit = op.unit;
          for (int k = 0; k < op.nco; ++k) {
            t.co_k[k] = op.co_k[k];
            t.co_v[k] = op.co_v[k];
          }
          if (op.nco || op.code == OP_QUAD || op.code == OP_QLITE) tp.needs_jit = 1;
          if (op.code == OP_SCALE) {
            if (ncoef + 2 > kTMaxCoef) return false;
            tp.coef[ncoef] = hp.coef[op.coef];
            tp.coef[ncoef + 1] = hp.coef[op.coef + 1];
            t.coef = (int16_t)ncoef;
            ncoef += 2;
          }
        }
      }
      if (one_q) {
        const int sl = op.r0;
        cur1q->st[sl] = op.code == OP_H ? 1 : (op.code == OP_X ? 2 : 3);
        if (op.code == OP_MAT) {
          if (ncoef + 8 > kTMaxCoef) return false;
          for (int q = 0; q < 8; ++q) tp.coef[ncoef + q] = hp.coef[op.coef + q];
          cur1q->cf[sl] = (int16_t)ncoef;
          ncoef += 8;
        }
      }
    }
    T.op_end = (int16_t)nsteps;
  }
  return true;
}

// Quadratic-form eligibility and pair factors of every OP_DIAG op of a pass
// (qk_internal.h QuadOp), from the host plan's table gates.
std::vector<QuadOp> quad_ops(const HostPlan& hp, const TmaParams& tp) {
  std::vector<QuadOp> out(kTMaxOps);
  std::unordered_map<int64_t, int> by_out;
  for (size_t t = 0; t < hp.tables.size(); ++t) by_out[hp.tables[t].out] = (int)t;
  std::unordered_map<int64_t, const std::vector<double>*> qdata;
  for (auto& qc : hp.qcopy) qdata[qc.first] = &qc.second;
  for (int ph = 0; ph < tp.nphases; ++ph)
    for (int o = tp.ph[ph].op_begin; o < tp.ph[ph].op_end; ++o) {
      const TOp& op = tp.ops[o];
      if ((op.code == OP_QUAD || op.code == OP_QLITE) && !getenv("QK_NO_PJ_CONST")) {
        auto it = qdata.find(op.table);
        if (it == qdata.end()) continue;
        const int NO = op.code == OP_QUAD ? tp.nbits - tp.C : 0;
        const QuadLayout L = quad_layout(tp.C, tp.M, NO);
        const std::vector<double>& d = *it->second;
        if ((size_t)(L.pj + 2 * (1 << tp.M)) > d.size()) continue;
        QuadOp q;
        q.npj = 1 << tp.M;
        for (int j = 0; j < q.npj; ++j) {
          q.pj[j][0] = d[L.pj + 2 * j];
          q.pj[j][1] = d[L.pj + 2 * j + 1];
        }
        out[o] = q;
        continue;
      }
      if (op.code != OP_DIAG) continue;
      auto it = by_out.find(op.table);
      if (it == by_out.end()) continue;
      const TableDesc& td = hp.tables[it->second];
      QuadOp q;
      for (int a = 0; a < 16; ++a) q.pf[a][0] = 1.0, q.pf[a][1] = 0.0;
      int slot_of_bit[32];
      for (int b = 0; b < 32; ++b) slot_of_bit[b] = -1;
      for (int sl = 0; sl < tp.M; ++sl) {
        const uint32_t pr = op.pr[1 << sl];
        if (pr && !(pr & (pr - 1))) slot_of_bit[__builtin_ctz(pr)] = sl;
      }
      bool ok = true;
      for (int g = td.g0; g < td.g0 + td.ng && ok; ++g) {
        const TableGate& tg = hp.tgates[g];
        int rs[13], nrs = 0;
        for (int j = 0; j < tg.nt; ++j)
          if (tg.slot[j] >= 0 && tg.slot[j] < 32 && slot_of_bit[tg.slot[j]] >= 0) rs[nrs++] = slot_of_bit[tg.slot[j]];
        if (nrs <= 1) continue;
        if (tg.nt != 2) {
          ok = false;
          break;
        }
        const double* e = &hp.entries[2 * tg.entries];
        const cplx e0(e[0], e[1]), e1(e[2], e[3]), e2(e[4], e[5]), e3(e[6], e[7]);
        const cplx pfv = e3 * e0 / (e1 * e2);
        const int sa = std::min(rs[0], rs[1]), sb = std::max(rs[0], rs[1]);
        const cplx cur(q.pf[sa * 4 + sb][0], q.pf[sa * 4 + sb][1]);
        const cplx nv = cur * pfv;
        q.pf[sa * 4 + sb][0] = nv.real();
        q.pf[sa * 4 + sb][1] = nv.imag();
      }
      q.ok = ok;
      q.inv2 = 1.0 / (td.scale * td.scale + td.scale_im * td.scale_im);
      out[o] = q;
    }
  return out;
}

// jit_source is a pure function of the pass structure: reloading a program
// (or a program sharing pass structures) reuses the generated source instead
// of rebuilding ~100 KB of text per pass (3.8 ms for QAOA30's 24 passes).
// Key: the TmaParams bytes without the tensor map and device pointers.
// environment switches the generator (and tma_smem_bytes / jit_pairs) reads
const char* const kGenEnv[] = {"QK_JIT_PREFETCH", "QK_JIT_HOIST", "QK_JIT_EARLY", "QK_JIT_SW128", "QK_NO_CORDER",
                               "QK_NO_SLICES", "QK_SLICE_RUN", "QK_X_FENCE", "QK_SMAX", "QK_NG2", "QK_CONS",
                               "QK_EXP_SKIP", "QK_JIT_MAXNREG", "QK_NO_TSTORE", "QK_PAIR", "QK_QHOIST"};

// A pass structure's built kernel variants (process-wide): key = its TMA
// parameters without pointers and tensor map, its OP_QUAD data, the switches
std::string tma_key(const TmaParams& tp) {
  TmaParams k = tp;
  memset(&k.map, 0, sizeof k.map);
  k.tabs = nullptr;
  k.state = nullptr;
  k.out = nullptr;
  return std::string(reinterpret_cast<const char*>(&k), sizeof k);
}
struct PassJit {
  int variant;
  void* kern;
  std::vector<long long> toff;
  std::vector<double> coef;
};
struct PassJitMemo {
  std::string tkey;  // tuning key (hash of the structure's first source)
  std::vector<PassJit> vars;
};
std::mutex g_pj_mu;
std::unordered_map<std::string, std::unique_ptr<PassJitMemo>> g_pass_jit;
std::string pass_jit_key(const TmaParams& tp, const std::vector<QuadOp>& quad, const char* venv) {
  std::string key = tma_key(tp);
  for (const QuadOp& q : quad) key.append(reinterpret_cast<const char*>(&q), sizeof q);
  for (const char* e : kGenEnv) {
    const char* v = getenv(e);
    key.push_back('|');
    if (v) key.append(v);
  }
  key += venv ? std::string("|v") + venv : std::string("|all");
  return key;
}
const PassJitMemo* pass_jit_find(const std::string& key) {
  if (getenv("QK_JIT_NOCACHE")) return nullptr;
  std::lock_guard<std::mutex> lk(g_pj_mu);
  auto it = g_pass_jit.find(key);
  return it == g_pass_jit.end() ? nullptr : it->second.get();
}
const PassJitMemo* pass_jit_store(const std::string& key, PassJitMemo&& m) {
  std::lock_guard<std::mutex> lk(g_pj_mu);
  auto& slot = g_pass_jit[key];
  if (!slot) slot.reset(new PassJitMemo(std::move(m)));  // entries live for the process (kernels do too)
  return slot.get();
}

bool jit_source_cached(const TmaParams& tp, std::string* src, std::vector<long long>* toff,
                       std::vector<double>* coef, int variant = 0, const std::vector<QuadOp>* quad = nullptr) {
  struct Val {
    bool ok;
    std::string src;
    std::vector<long long> toff;
    std::vector<double> coef;
  };
  static std::mutex mu;
  static std::unordered_map<std::string, Val> cache;
  std::string key = tma_key(tp);
  key.push_back((char)variant);
  // (the quadratic ops' data: pair factors for variant bit 2, and the pj
  // constants every variant passes as parameters)
  if (quad)
    for (const QuadOp& q : *quad) key.append(reinterpret_cast<const char*>(&q), sizeof q);
  for (const char* e : kGenEnv) {
    const char* v = getenv(e);
    key.push_back('|');
    if (v) key.append(v);
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end() && !getenv("QK_JIT_NOCACHE")) {
      *src = it->second.src;
      *toff = it->second.toff;
      *coef = it->second.coef;
      return it->second.ok;
    }
  }
  Val v;
  v.ok = jit_source(tp, &v.src, &v.toff, &v.coef, variant, quad);
  const bool ok = v.ok;
  *src = v.src;
  *toff = v.toff;
  *coef = v.coef;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(std::move(key), std::move(v));
  return ok;
}

// ---- variant autotuning ----------------------------------------------------
// Process-wide per pass structure (key = its first variant's source): device
// ms of every variant seen so far and, once all are timed, the fastest.
struct TuneRec {
  std::vector<int> variants;
  std::vector<double> ms;  // fastest timing so far (< 0: not timed yet)
  std::vector<int> cnt;    // timings so far
  int best = -1;
};
// every variant is timed this many times (its fastest counts), so one noisy
// run does not decide (QK_TUNE_ROUNDS)
int tune_rounds() {
  static const int r = getenv("QK_TUNE_ROUNDS") ? std::max(1, atoi(getenv("QK_TUNE_ROUNDS"))) : 2;
  return r;
}
std::mutex g_tune_mu;
std::unordered_map<std::string, TuneRec> g_tune;

// Point pass p at its tuned variant, or (tuning = true, before a run) at the
// next variant still to time. Returns true if p is timed in this run.
bool tune_pick(qk_sim* s, int p, bool tuning) {
  if (p >= (int)s->pass_var.size() || s->pass_var[p].size() < 2) return false;
  if ((int)s->tuning.size() < (int)s->pass_var.size()) s->tuning.assign(s->pass_var.size(), -1);
  s->tuning[p] = -1;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  TuneRec& tr = g_tune[s->pass_key[p]];
  if (tr.variants.empty())
    for (auto& v : s->pass_var[p]) {
      tr.variants.push_back(v.variant);
      tr.ms.push_back(-1.0);
      tr.cnt.push_back(0);
    }
  int pick = -1;
  if (tr.best >= 0) {
    pick = tr.best;
  } else if (tuning && !getenv("QK_NO_TUNE")) {
    int least = INT32_MAX;
    for (size_t k = 0; k < tr.cnt.size(); ++k)
      if (tr.cnt[k] < least) {
        least = tr.cnt[k];
        pick = tr.variants[k];
      }
  }
  if (pick < 0) pick = tr.variants[0];
  for (size_t k = 0; k < s->pass_var[p].size(); ++k)
    if (s->pass_var[p][k].variant == pick) {
      s->pass_jit[p] = s->pass_var[p][k].kern;
      s->jit_blob[p] = s->pass_var[p][k].blob;
      if (tr.best < 0 && tuning && !getenv("QK_NO_TUNE")) s->tuning[p] = (int)k;
      return s->tuning[p] >= 0;
    }
  return false;
}

void tune_record(qk_sim* s, int p, double ms) {
  const int k = s->tuning[p];
  const int variant = s->pass_var[p][k].variant;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  TuneRec& tr = g_tune[s->pass_key[p]];
  double best_ms = 1e300;
  int best = -1;
  for (size_t i = 0; i < tr.variants.size(); ++i)
    if (tr.variants[i] == variant) {
      tr.ms[i] = tr.cnt[i] ? std::min(tr.ms[i], ms) : ms;
      ++tr.cnt[i];
    }
  for (size_t i = 0; i < tr.variants.size(); ++i) {
    if (tr.cnt[i] < tune_rounds()) return;  // still variants to time
    if (tr.ms[i] < best_ms) {
      best_ms = tr.ms[i];
      best = tr.variants[i];
    }
  }
  tr.best = best;
  if (getenv("QK_DUMP_TUNE")) {
    fprintf(stderr, "tune: pass %d best variant %d (", p, best);
    for (size_t i = 0; i < tr.variants.size(); ++i) fprintf(stderr, " v%d %.3f ms", tr.variants[i], tr.ms[i]);
    fprintf(stderr, " )\n");
  }
}

void plan_overlap(qk_sim* s);

int upload_plan_dry(qk_sim* s);

std::atomic<uint64_t> g_plan_gen{1};

int upload_plan(qk_sim* s) {
  if (s->dry) return upload_plan_dry(s);
  HostPlan& hp = s->hp;
  std::vector<char> buf;
  const size_t o_pass = push_section(buf, hp.passes);
  const size_t o_phase = push_section(buf, hp.phases);
  const size_t o_ops = push_section(buf, hp.ops);
  const size_t o_coef = push_section(buf, hp.coef);
  const size_t o_sqs = push_section(buf, hp.sqs);
  const size_t o_tab = push_section(buf, hp.tables);
  const size_t o_tg = push_section(buf, hp.tgates);
  const size_t o_ent = push_section(buf, hp.entries);
  buf.resize(buf.size() + 256);
  if (s->blob_bytes < buf.size()) {
    if (s->blob) cudaFree(s->blob);
    s->blob = nullptr;
    s->blob_bytes = 0;
    CUDA_TRY(cudaMalloc(&s->blob, buf.size()));
    s->blob_bytes = buf.size();
  }
  char* base = (char*)s->blob;
  CUDA_TRY(cudaMemcpyAsync(base, buf.data(), buf.size(), cudaMemcpyHostToDevice, s->stream));
  // plan identity for the graph replay (graph_key): the same plan uploaded
  // again to the same addresses keeps a captured graph valid
  s->prog_gen = s->nbits <= 24 ? (uint64_t)std::hash<std::string_view>()(std::string_view(buf.data(), buf.size()))
                               : ++g_plan_gen;
  s->d_pass = (PassDesc*)(base + o_pass);
  s->d_phase = (PhaseDesc*)(base + o_phase);
  s->d_ops = (OpDesc*)(base + o_ops);
  s->d_coef = (double*)(base + o_coef);
  s->d_sqs = (SqsDesc*)(base + o_sqs);
  const size_t pool_bytes = (size_t)std::max<int64_t>(hp.pool, 1) * 16;
  if (s->pool_bytes < pool_bytes) {
    if (s->d_pool) cudaFree(s->d_pool);
    s->d_pool = nullptr;
    s->pool_bytes = 0;
    CUDA_TRY(cudaMalloc(&s->d_pool, pool_bytes));
    s->pool_bytes = pool_bytes;
  }
  s->tma.clear();
  s->lazy_map1.clear();
  s->pass_tma.assign(hp.passes.size(), -1);
  std::vector<const std::vector<int>*> pass_dest(hp.passes.size(), nullptr), pass_x(hp.passes.size(), nullptr),
      pass_tile(hp.passes.size(), nullptr);
  for (auto& ip : s->iplan) {
    ip.permuted = 0;
    if (ip.type == QK_INS_BLOCK && ip.npass > 0 && !ip.dest.empty()) {
      pass_dest[ip.pass0 + ip.npass - 1] = &ip.dest;
      pass_x[ip.pass0 + ip.npass - 1] = &ip.xspec;
    }
    if (ip.type == QK_INS_BLOCK && ip.npass == 1 && !ip.tile.empty()) pass_tile[ip.pass0] = &ip.tile;
  }
  for (size_t p = 0; p < hp.passes.size(); ++p) {
    TmaParams tp;
    if (make_tma(s, hp.passes[p], tp, pass_dest[p], pass_x[p], pass_tile[p])) {
      s->pass_tma[p] = (int)s->tma.size();
      s->tma.push_back(tp);
      s->lazy_map1.emplace_back();
      if (tp.lazy && s->bufs[1] && !encode_lazy_map(tp, s->bufs[1], &s->lazy_map1.back()))
        return fail(QK_ECUDA, "tensor map unavailable");
    }
  }
  for (auto& ip : s->iplan)
    if (ip.type == QK_INS_BLOCK && ip.npass > 0 && !ip.dest.empty() && ip.tile.empty()) {
      ip.permuted = s->pass_tma[ip.pass0 + ip.npass - 1] >= 0;
      // the planner already relabeled the qubits for this pass: it must run
      if (!ip.permuted) return fail(QK_ESIM, "internal: fused pass is not executable on the TMA path");
    }
  // the last pass that writes data carries the fused norm, unless a
  // cross-process exchange follows it (that changes this shard's norm)
  s->norm_pass = -1;
  s->norm_valid = false;
  {
    int last = -1;
    for (auto& ip : s->iplan) {
      if (ip.type == QK_INS_BLOCK && ip.npass > 0) last = ip.pass0 + ip.npass - 1;
      if (ip.type == QK_INS_CSQS && ip.sqs == -2) last = -2;
    }
    // (temporary one-block plans of the kernel-level entry points run with an
    // empty iplan, so `last` always indexes this plan's passes)
    if (last >= 0 && last < (int)s->pass_tma.size() && s->pass_tma[last] >= 0 &&
        !s->tma[s->pass_tma[last]].xbits && !getenv("QK_NO_FUSED_NORM")) {
      TmaParams& tq = s->tma[s->pass_tma[last]];
      int ng = 0, st = 0;
      tma_smem_bytes(tq.C, tq.M, &ng, &st, tq.smax);
      const uint64_t grid = tq.nchunks < (uint64_t)s->num_sms ? tq.nchunks : (uint64_t)s->num_sms;
      // the partials buffer holds 4096 doubles and the kernel's reduction area 16 groups
      if (ng <= 16 && grid * (uint64_t)ng <= 4096) {
        tq.norm = 1;
        s->norm_pass = last;
        s->nrm_parts = (int)grid * ng;
      }
    }
  }
  // specialise TMA passes of large states (compile cost amortised; cached per structure)
  s->pass_jit.assign(hp.passes.size(), nullptr);
  s->jit_blob.assign(hp.passes.size(), {});
  const char* jenv = getenv("QK_JIT");
  const int jit_min = jenv ? atoi(jenv) : 20;   // QK_JIT=<min address bits>; QK_NO_JIT disables
  if (!jit_available() && !getenv("QK_NO_JIT") && s->nbits >= jit_min) {
    static bool warned = false;
    if (!warned)
      fprintf(stderr,
              "qkb200: NVRTC (libnvrtc.so.12) not found: the specialised block passes, diagonal folding and the "
              "lazy layout are off; large states run on the generic interpreter (about 2x slower)\n");
    warned = true;
  }
  if (jit_available() && s->nbits >= jit_min) {
    const auto tj0 = std::chrono::steady_clock::now();
    // Up to sixteen variants per pass (bit 1: no hoisted table, bit 2: quadratic
    // table groups, bit 4: OP_QUAD factors computed after the stage wait
    // instead of ahead in a pending slot (passes without OP_QUAD: more
    // OP_QLITE factors hoisted into registers), bit 8: TMA-store epilogue for lazy
    // passes); identical sources are built once. QK_JIT_VARIANT=v pins one,
    // otherwise the first runs time every variant and keep the fastest per
    // pass structure (process-wide, tune_pick / tune_record). A pass structure
    // seen before (same parameters, same switches) reuses its kernels.
    const char* venv = getenv("QK_JIT_VARIANT");
    s->tuning.assign(hp.passes.size(), -1);
    s->pass_var.assign(hp.passes.size(), {});
    s->pass_key.assign(hp.passes.size(), std::string());
    std::vector<std::string> pkeys(hp.passes.size());
    std::vector<const PassJitMemo*> hits(hp.passes.size(), nullptr);
    std::vector<std::string> srcs;
    std::vector<int> src_pass, src_var;
    std::vector<std::vector<long long>> toffs;
    std::vector<std::vector<double>> coefs;
    for (size_t p = 0; p < hp.passes.size(); ++p) {
      if (s->pass_tma[p] < 0) continue;
      std::vector<QuadOp> quad = quad_ops(hp, s->tma[s->pass_tma[p]]);
      pkeys[p] = pass_jit_key(s->tma[s->pass_tma[p]], quad, venv);
      if ((hits[p] = pass_jit_find(pkeys[p]))) continue;
      std::vector<std::string> seen;
      for (int variant = 0; variant < 16; ++variant) {
        if (venv && variant != atoi(venv)) continue;
        std::string src;
        std::vector<long long> toff;
        std::vector<double> coef;
        if (!jit_source_cached(s->tma[s->pass_tma[p]], &src, &toff, &coef, variant, &quad)) continue;
        if (std::find(seen.begin(), seen.end(), src) != seen.end()) continue;
        seen.push_back(src);
        if (const char* dd = getenv("QK_JIT_DUMP")) {
          const std::string path = std::string(dd) + "/pass" + std::to_string(p) + "_v" + std::to_string(variant) + ".cu";
          if (FILE* f = fopen(path.c_str(), "w")) {
            fwrite(src.data(), 1, src.size(), f);
            fclose(f);
          }
        }
        srcs.push_back(std::move(src));
        src_pass.push_back((int)p);
        src_var.push_back(variant);
        toffs.push_back(std::move(toff));
        coefs.push_back(std::move(coef));
      }
    }
    const auto tj1 = std::chrono::steady_clock::now();
    std::vector<void*> handles;
    jit_build(srcs, &handles);
    if (getenv("QK_DUMP_LOAD"))
      fprintf(stderr, "load: jit_source %.3f ms (%zu kernels), jit_build %.3f ms\n",
              std::chrono::duration<double, std::milli>(tj1 - tj0).count(), srcs.size(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tj1).count());
    {  // new pass structures: their built variants (the tuning key: the first source's hash)
      std::map<int, PassJitMemo> fresh;
      for (size_t i = 0; i < srcs.size(); ++i) {
        PassJitMemo& m = fresh[src_pass[i]];
        if (m.tkey.empty()) m.tkey = std::to_string(std::hash<std::string>{}(srcs[i])) + "_" + std::to_string(srcs[i].size());
        if (handles[i]) m.vars.push_back({src_var[i], handles[i], toffs[i], coefs[i]});
      }
      for (auto& kv : fresh) hits[kv.first] = pass_jit_store(pkeys[kv.first], std::move(kv.second));
    }
    for (size_t p = 0; p < hp.passes.size(); ++p) {
      if (!hits[p]) continue;
      s->pass_key[p] = hits[p]->tkey;
      const TmaParams& tq = s->tma[s->pass_tma[p]];
      for (const PassJit& v : hits[p]->vars) {
        // QkJitParams: map[16 words] | tabs | state | out | nchunks | nrm | split | toff[ntab+1] |
        // coef[ncoef+1] | smap[16 words] (64-B aligned: the last 16 words of the blob)
        const size_t smap_off = (16 + 6 + v.toff.size() + 1 + v.coef.size() + 1 + 7) & ~(size_t)7;
        std::vector<uint64_t> blob(smap_off + 16, 0);
        blob[16] = (uint64_t)(uintptr_t)s->d_pool;
        blob[19] = tq.xbits ? tq.nchunks >> tq.xbits : tq.nchunks;  // cluster mode: supertiles
        blob[20] = (uint64_t)(uintptr_t)s->d_nrm;
        blob[21] = 0;                                                 // split word (launch_pass_part)
        for (size_t k = 0; k < v.toff.size(); ++k) blob[22 + k] = (uint64_t)v.toff[k];
        const size_t co = 22 + v.toff.size() + 1;
        for (size_t k = 0; k < v.coef.size(); ++k) memcpy(&blob[co + k], &v.coef[k], 8);
        s->pass_var[p].push_back({v.variant, v.kern, std::move(blob)});
        if (!s->pass_jit[p]) {
          s->pass_jit[p] = v.kern;
          s->jit_blob[p] = s->pass_var[p].back().blob;
        }
      }
    }
    for (size_t p = 0; p < hp.passes.size(); ++p) tune_pick(s, (int)p, false);
  }
  if (s->norm_pass >= 0 && !s->pass_jit[s->norm_pass]) s->norm_pass = -1;  // the interpreter sums nothing
  // strided-tile passes exist only as specialised kernels: without one the
  // generic register-tiled pass runs them (arbitrary chunk bits, in place)
  for (size_t p = 0; p < hp.passes.size(); ++p)
    if (s->pass_tma[p] >= 0 && s->tma[s->pass_tma[p]].needs_jit && !(p < s->pass_jit.size() && s->pass_jit[p]))
      return fail(QK_ESIM, "folded diagonal block needs the specialised kernel (NVRTC)");
  for (size_t p = 0; p < hp.passes.size(); ++p) {  // the generic kernels have no OP_QUAD
    const PassDesc& pd = hp.passes[p];
    bool quad = false;
    for (int ph = 0; ph < pd.nphases; ++ph) {
      const PhaseDesc& D = hp.phases[pd.phase0 + ph];
      for (int o = D.op_begin; o < D.op_end; ++o) quad = quad || hp.ops[o].code == OP_QUAD || hp.ops[o].code == OP_QLITE;
    }
    if (quad && !(s->pass_tma[p] >= 0 && p < s->pass_jit.size() && s->pass_jit[p]))
      return fail(QK_ESIM, "quadratic diagonal pass needs the specialised kernel (NVRTC)");
  }
  for (size_t p = 0; p < hp.passes.size(); ++p)
    if (s->pass_tma[p] >= 0 && s->tma[s->pass_tma[p]].lazy && !(p < s->pass_jit.size() && s->pass_jit[p])) {
      const TmaParams& tq = s->tma[s->pass_tma[p]];
      for (int x = 0; x < tq.C; ++x)  // the generic pass cannot permute the tile on store
        if (tq.dpos[x] != tq.tbit[x]) return fail(QK_ESIM, "lazy pass needs the specialised kernel (NVRTC)");
      s->pass_tma[p] = -1;
    }
  if (getenv("QK_DUMP_TABLES"))
    for (size_t p = 0; p < hp.passes.size(); ++p) {
      if (s->pass_tma[p] < 0) continue;
      const TmaParams& tq = s->tma[s->pass_tma[p]];
      fprintf(stderr, "pass %zu C=%d M=%d phases=%d smax=%d tbit=", p, tq.C, tq.M, tq.nphases, tq.smax);
      for (int k = 0; k < tq.C; ++k) fprintf(stderr, "%d,", tq.tbit[k]);
      fprintf(stderr, "\n");
      for (int ph = 0; ph < tq.nphases; ++ph)
        for (int o = tq.ph[ph].op_begin; o < tq.ph[ph].op_end; ++o) {
          const TOp& op = tq.ops[o];
          if (op.code != OP_DIAG) {
            fprintf(stderr, "   ph%d op%d code=%d\n", ph, o, op.code);
            continue;
          }
          int bits = -1;
          for (auto& td : hp.tables)
            if (td.out == op.table) bits = td.bits;
          fprintf(stderr, "   ph%d op%d DIAG bits=%d nco=%d co_k=", ph, o, bits, op.nco);
          for (int k = 0; k < op.nco; ++k) fprintf(stderr, "%d,", op.co_k[k]);
          fprintf(stderr, "\n");
        }
    }
  if (getenv("QK_DUMP_PLAN"))
    for (size_t i = 0; i < s->iplan.size(); ++i) {
      const InstrPlan& ip = s->iplan[i];
      if (ip.type != QK_INS_BLOCK) continue;
      for (int p = ip.pass0; p < ip.pass0 + ip.npass; ++p) {
        fprintf(stderr, "instr %zu pass %d C=%d phases=%d tma=%d jit=%d x=%d tile=", i, p, hp.passes[p].C,
                hp.passes[p].nphases, s->pass_tma[p] >= 0, p < (int)s->pass_jit.size() && s->pass_jit[p] != nullptr,
                s->pass_tma[p] >= 0 ? s->tma[s->pass_tma[p]].xbits : 0);
        for (int t : ip.tile) fprintf(stderr, "%d,", t);
        fprintf(stderr, "\n");
      }
    }
  plan_overlap(s);
  // OP_QUAD / OP_QLITE data: one H2D copy of the pool span they occupy (the
  // gaps are table regions, which the table build below writes), instead of
  // one pageable copy per op (QFT20: 18 copies)
  const auto tq0 = std::chrono::steady_clock::now();
  bool qdone = hp.qcopy.empty();
  if (!qdone) {
    size_t lo = SIZE_MAX, hi = 0, tot = 0;
    for (auto& q : hp.qcopy) {
      lo = std::min(lo, (size_t)(2 * q.first));
      hi = std::max(hi, (size_t)(2 * q.first) + q.second.size());
      tot += q.second.size();
    }
    if ((hi - lo) * sizeof(double) <= ((size_t)4 << 20) && hi - lo <= 2 * tot + 8192) {
      std::vector<double> img(hi - lo, 0.0);
      for (auto& q : hp.qcopy) std::copy(q.second.begin(), q.second.end(), img.begin() + (2 * q.first - lo));
      CUDA_TRY(cudaMemcpyAsync(s->d_pool + lo, img.data(), img.size() * sizeof(double), cudaMemcpyHostToDevice,
                               s->stream));
      qdone = true;
    }
  }
  if (!hp.tables.empty()) {
    int rc = launch_build_tables((const TableDesc*)(base + o_tab), (int)hp.tables.size(),
                                 (const TableGate*)(base + o_tg), (const double*)(base + o_ent),
                                 s->d_pool, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "table build launch failed: %s", cudaGetErrorString((cudaError_t)rc));
  }
  if (!qdone)
    for (auto& q : hp.qcopy)
      CUDA_TRY(cudaMemcpyAsync(s->d_pool + 2 * q.first, q.second.data(), q.second.size() * sizeof(double),
                               cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (getenv("QK_DUMP_LOAD"))
    fprintf(stderr, "load: quad data %zu ops (%s), tables and sync %.3f ms\n", hp.qcopy.size(),
            hp.qcopy.empty() ? "none" : "one copy or per op",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
  return QK_OK;
}

// qk_plan_dry: the TMA parameters and specialised sources of every pass,
// written to s->dry_dir (pass<p>_v<variant>.cu) with a one-line summary per
// pass on stderr; nothing touches a device.
int upload_plan_dry(qk_sim* s) {
  HostPlan& hp = s->hp;
  g_dry_maps = true;
  s->tma.clear();
  s->pass_tma.assign(hp.passes.size(), -1);
  std::vector<const std::vector<int>*> pass_dest(hp.passes.size(), nullptr), pass_x(hp.passes.size(), nullptr),
      pass_tile(hp.passes.size(), nullptr);
  for (auto& ip : s->iplan) {
    if (ip.type == QK_INS_BLOCK && ip.npass > 0 && !ip.dest.empty()) {
      pass_dest[ip.pass0 + ip.npass - 1] = &ip.dest;
      pass_x[ip.pass0 + ip.npass - 1] = &ip.xspec;
    }
    if (ip.type == QK_INS_BLOCK && ip.npass == 1 && !ip.tile.empty()) pass_tile[ip.pass0] = &ip.tile;
  }
  for (size_t p = 0; p < hp.passes.size(); ++p) {
    TmaParams tp;
    if (make_tma(s, hp.passes[p], tp, pass_dest[p], pass_x[p], pass_tile[p])) {
      s->pass_tma[p] = (int)s->tma.size();
      s->tma.push_back(tp);
    }
  }
  g_dry_maps = false;
  for (size_t p = 0; p < hp.passes.size(); ++p) {
    const PassDesc& pd = hp.passes[p];
    int cnt[16] = {0};
    for (int ph = 0; ph < pd.nphases; ++ph) {
      const PhaseDesc& D = hp.phases[pd.phase0 + ph];
      for (int o = D.op_begin; o < D.op_end; ++o) cnt[hp.ops[o].code & 15]++;
    }
    fprintf(stderr, "dry pass %zu: C=%d phases=%d tma=%d H=%d MAT=%d CX=%d DIAG=%d QUAD=%d QLITE=%d tile=", p, pd.C,
            pd.nphases, s->pass_tma[p] >= 0, cnt[OP_H], cnt[OP_MAT], cnt[OP_CX], cnt[OP_DIAG], cnt[OP_QUAD],
            cnt[OP_QLITE]);
    if (pass_tile[p])
      for (int t : *pass_tile[p]) fprintf(stderr, "%d,", t);
    fprintf(stderr, "\n");
    if (s->pass_tma[p] < 0 || s->dry_dir.empty()) continue;
    std::vector<QuadOp> quad = quad_ops(hp, s->tma[s->pass_tma[p]]);
    for (int variant = 0; variant < 16; ++variant) {
      std::string src;
      std::vector<long long> toff;
      std::vector<double> coef;
      if (!jit_source_cached(s->tma[s->pass_tma[p]], &src, &toff, &coef, variant, &quad)) continue;
      const std::string path = s->dry_dir + "/pass" + std::to_string(p) + "_v" + std::to_string(variant) + ".cu";
      if (FILE* f = fopen(path.c_str(), "w")) {
        fwrite(src.data(), 1, src.size(), f);
        fclose(f);
      }
    }
  }
  return QK_OK;
}

void replay_perm(qk_sim* s) {
  s->final_perm.resize(s->n);
  for (int i = 0; i < s->n; ++i) s->final_perm[i] = i;
  for (auto& ins : s->prog) {
    if (ins.type == QK_INS_BLOCK) continue;
    std::vector<int> a = ins.a, b = ins.b;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    for (size_t k = 0; k < a.size() && k < b.size(); ++k) std::swap(s->final_perm[a[k]], s->final_perm[b[k]]);
  }
}

int check_csqs(const qk_sim* s, const std::vector<int>& local_set, const std::vector<int>& rank_set) {
  // simulator.py:184-194
  const int local = s->L, S = (int)local_set.size();
  std::vector<int> srt = local_set;
  std::sort(srt.begin(), srt.end());
  bool top = true;
  for (int i = 0; i < S; ++i)
    if (srt[i] != local - S + i) top = false;
  if (!top) {
    std::string l = "(";
    for (int i = 0; i < S; ++i) l += std::to_string(local_set[i]) + (S == 1 ? "," : (i + 1 < S ? ", " : ""));
    l += ")";
    return fail(QK_ESIM, "cross-rank local set %s is not top-of-local", l.c_str());
  }
  if ((int)rank_set.size() != S) return fail(QK_ESIM, "cross-rank swap sets differ in size");
  for (int q : rank_set)
    if (q < local || q >= s->n) return fail(QK_ESIM, "rank bit %d outside [%d, %d)", q, local, s->n);
  if (s->b < S) return fail(QK_ESIM, "buffer of 2^%d too small for %d swap pairs", s->b, S);
  return QK_OK;
}

// Conservative plan-time check that a single-pass block runs on the TMA path
// (a fused pass must: the swaps it absorbs have no other executor).
bool lay_identity(const std::vector<int>& l) {
  for (size_t q = 0; q < l.size(); ++q)
    if (l[q] != (int)q) return false;
  return true;
}

// Two rounds of disjoint bit swaps (SQS, applied in order) that bring the data
// of layout `lay` (reference bit q at physical bit lay[q]) back to the
// reference layout. An SQS on physical bits (x, y) turns lay into tau o lay, so
// we need tau2 o tau1 = pi = lay^-1; on every cycle (a_0 .. a_{m-1}) of pi the
// reflections a_i <-> a_{-i} and a_i <-> a_{1-i} compose to pi.
void restore_rounds(const std::vector<int>& lay, std::vector<std::pair<int, int>> rounds[2]) {
  const int n = (int)lay.size();
  std::vector<int> pi(n);
  for (int q = 0; q < n; ++q) pi[lay[q]] = q;
  std::vector<char> seen(n, 0);
  for (int a = 0; a < n; ++a) {
    if (seen[a] || pi[a] == a) continue;
    std::vector<int> cyc;
    for (int x = a; !seen[x]; x = pi[x]) {
      seen[x] = 1;
      cyc.push_back(x);
    }
    const int m = (int)cyc.size();
    for (int i = 0; i < m; ++i) {
      const int j1 = (m - i) % m, j2 = ((1 - i) % m + m) % m;
      if (i < j1) rounds[0].push_back({cyc[i], cyc[j1]});
      if (i < j2) rounds[1].push_back({cyc[i], cyc[j2]});
    }
  }
}

bool tma_plan_ok(const HostPlan& hp, int pass, int nbits, int cmax = 12) {
  if (getenv("QK_NO_TMA")) return false;
  const PassDesc& pd = hp.passes[pass];
  if (getenv("QK_TMA13")) cmax = 13;
  if (pd.M < 3 || pd.M > kMaxTM || pd.C < 9 || pd.C > cmax || pd.nphases > kTMaxPh || nbits > 34) return false;
  if (pd.nouter != nbits - pd.C) return false;
  const int ob = hp.phases[pd.phase0].op_begin, oe = hp.phases[pd.phase0 + pd.nphases - 1].op_end;
  int ncoef = 0;
  for (int o = ob; o < oe; ++o) ncoef += hp.ops[o].code == OP_MAT ? 8 : (hp.ops[o].code == OP_SCALE ? 2 : 0);
  return oe - ob <= kTMaxOps && ncoef <= kTMaxCoef;
}

// ---- cross-block pass scheduling (lazy layout, every swap in-handle) --------
// The optimizer cut the circuit into blocks of <= c qubits with SQS between
// them (optimizer.py); in the lazy layout a swap costs nothing, so the
// only cost left is one HBM sweep per block. Here the program is rewritten on
// "wires" (a wire = a start position, followed through every swap) and cut
// again into passes over tiles of up to `cap` physical bits: a pass applies
// every non-diagonal gate whose wires are all in its tile and whose
// predecessors ran, and every diagonal gate whose predecessors ran (the
// diagonal ones need no tile: OP_QUAD applies a quadratic phase over all
// address bits). Dependencies: two gates sharing a wire are ordered unless
// both are diagonal. The tile of a pass is chosen greedily (the wire that lets
// the most gates run, ties to the earliest waiting gate), with the wires on
// the row bits 0..rowbits-1 always in it; each pass's store permutation puts
// wires of the next pass (a lookahead choice) on those row bits. QAOA30 c12
// (51 blocks, 24 passes after folding) runs in 13 passes, QFT33 c10 in 4.
// Results equal the block order's up to rounding: only commuting gates move.
//
// Shards (ntot > nb): positions >= nb are rank bits held by other shards. A
// CSQS that pairs local bits with such rank bits moves wires in and out of
// the shard, so it is a barrier: the gates before it are cut into passes
// (segment by segment), the CSQS is emitted with the wire of every position
// just before it (`xw`), and the next segment's passes see the wires it
// brought in. A CSQS whose rank bits are all held here is a relabel.
bool reblock(const std::vector<InstrH>& prog, int nb, int cap, int rowbits, std::vector<InstrH>* out,
             std::vector<int>* p2w_final, int ntot = -1, const std::vector<int>* init_pos = nullptr) {
  if (ntot < nb) ntot = nb;
  if (ntot > 64 || cap > nb) return false;
  std::vector<int> p2w(ntot);
  for (int q = 0; q < ntot; ++q) p2w[q] = q;
  struct Bar {
    size_t gate0;            // first gate after the barrier
    const InstrH* ins;
    std::vector<int> xw;     // position -> wire just before it
  };
  std::vector<Bar> bars;
  struct WG {
    const GateH* g;
    uint64_t wm;
    bool diag;
    std::vector<int> w;  // wire of every target
  };
  std::vector<WG> G;
  for (const InstrH& ins : prog) {
    if (ins.type == QK_INS_BLOCK) {
      for (const GateH& g : ins.gates) {
        WG x{&g, 0, is_diag(g.kind), {}};
        for (int t : g.t) {
          if (t < 0 || t >= nb) return false;
          x.wm |= 1ull << p2w[t];
          x.w.push_back(p2w[t]);
        }
        if (x.diag && !quad_gate(g)) return false;
        if (!x.diag && popc(x.wm) > cap - rowbits) return false;
        G.push_back(x);
      }
    } else {
      std::vector<int> sa = ins.a, sb = ins.b;
      if (sa.size() != sb.size()) return false;
      bool outside = false;
      for (int q : sa)
        if (q < 0 || q >= nb) return false;
      for (int q : sb) {
        if (q < 0 || q >= ntot) return false;
        outside = outside || q >= nb;
      }
      if (outside && ins.type != QK_INS_CSQS) return false;
      if (outside) bars.push_back({G.size(), &ins, p2w});
      std::sort(sa.begin(), sa.end());
      std::sort(sb.begin(), sb.end());
      for (size_t k = 0; k < sa.size(); ++k) std::swap(p2w[sa[k]], p2w[sb[k]]);
    }
  }
  *p2w_final = p2w;
  const int NS = (int)bars.size() + 1;  // segments
  auto seg_of_gate = [&](size_t i) {
    int sg = 0;
    while (sg < (int)bars.size() && bars[sg].gate0 <= i) ++sg;
    return sg;
  };
  // non-diagonal gates and their non-diagonal predecessors (through diagonal gates)
  std::vector<int> nd;                       // gate index of every non-diagonal gate
  std::vector<std::vector<uint64_t>> pre;    // predecessor bitsets over nd
  std::vector<std::vector<int>> ddep(G.size());  // diagonal gate -> nd predecessors
  {
    std::vector<int> last(ntot, -1);
    std::vector<std::vector<int>> dd(ntot);
    for (size_t i = 0; i < G.size(); ++i) {
      if (G[i].diag) {
        std::vector<int> deps;
        for (int w = 0; w < ntot; ++w)
          if ((G[i].wm >> w & 1) && last[w] >= 0) deps.push_back(last[w]);
        for (int w = 0; w < ntot; ++w)
          if (G[i].wm >> w & 1) dd[w].insert(dd[w].end(), deps.begin(), deps.end());
        ddep[i] = deps;
      } else {
        std::vector<int> p;
        for (int w = 0; w < ntot; ++w)
          if (G[i].wm >> w & 1) {
            if (last[w] >= 0) p.push_back(last[w]);
            p.insert(p.end(), dd[w].begin(), dd[w].end());
          }
        const int k = (int)nd.size();
        nd.push_back((int)i);
        pre.emplace_back();
        for (int x : p) {
          if ((int)pre[k].size() <= x / 64) pre[k].resize(x / 64 + 1, 0);
          pre[k][x / 64] |= 1ull << (x % 64);
        }
        for (int w = 0; w < ntot; ++w)
          if (G[i].wm >> w & 1) {
            last[w] = k;
            dd[w].clear();
          }
      }
    }
  }
  const int N = (int)nd.size();
  int first_open = 0;  // every gate before it is done (closure scans start here)
  const int kFront = getenv("QK_REBLOCK_FRONT") ? atoi(getenv("QK_REBLOCK_FRONT")) : 64;
  std::vector<int> nseg(N);
  for (int k = 0; k < N; ++k) nseg[k] = seg_of_gate((size_t)nd[k]);
  int cur_seg = 0;
  const size_t NW = (size_t)N / 64 + 1;
  std::vector<uint64_t> done(NW, 0);
  auto isdone = [&](const std::vector<uint64_t>& d, int k) { return (d[k / 64] >> (k % 64)) & 1; };
  // the non-diagonal gates a tile S can run now (in program order)
  // (a wire is blocked once a gate on it cannot run: every later gate on it
  // depends on that one, so the scan stops when all tile wires are blocked)
  auto closure = [&](uint64_t S, std::vector<uint64_t>& now, int* cnt) {
    now = done;
    int c = 0;
    uint64_t blocked = 0;
    for (int k = first_open; k < N; ++k) {
      if (nseg[k] != cur_seg || isdone(now, k)) continue;
      const uint64_t wm = G[nd[k]].wm;
      bool ok = !(wm & ~S) && !(wm & blocked);
      for (size_t w = 0; w < pre[k].size() && ok; ++w) ok = !(pre[k][w] & ~now[w]);
      if (!ok) {
        blocked |= wm;
        if ((blocked & S) == S) break;
        continue;
      }
      now[k / 64] |= 1ull << (k % 64);
      ++c;
    }
    *cnt = c;
  };
  std::vector<int> wire_at(nb);  // physical bit -> wire (the layout the passes see)
  for (int q = 0; q < nb; ++q) wire_at[q] = q;
  if (init_pos)  // initial placement: wire w at physical bit (*init_pos)[w]
    for (int w = 0; w < nb; ++w) wire_at[(*init_pos)[w]] = w;
  auto choose = [&](uint64_t forced) {
    uint64_t S = forced;
    std::vector<int> pend(ntot, INT32_MAX);
    for (int k = N - 1; k >= 0; --k)
      if (nseg[k] == cur_seg && !isdone(done, k))
        for (int w = 0; w < ntot; ++w)
          if (G[nd[k]].wm >> w & 1) pend[w] = k;
    // candidates: the wires of the first open gates (the frontier); a wire
    // whose first open gate lies further on cannot unblock more than these
    uint64_t front = 0;
    {
      int seen = 0;
      for (int k = first_open; k < N && seen < kFront; ++k)
        if (nseg[k] == cur_seg && !isdone(done, k)) {
          front |= G[nd[k]].wm;
          ++seen;
        }
    }
    std::vector<uint64_t> tmp;
    while (popc(S) < cap) {
      int best = -1, bc = -1;
      for (int x = 0; x < nb; ++x) {
        const int w = wire_at[x];
        if ((S >> w & 1) || pend[w] == INT32_MAX || !(front >> w & 1)) continue;
        int c = 0;
        closure(S | (1ull << w), tmp, &c);
        if (c > bc || (c == bc && pend[w] < pend[best])) {
          bc = c;
          best = w;
        }
      }
      if (best < 0) break;
      S |= 1ull << best;
    }
    return S;
  };
  std::vector<int> npass(N, -1);
  std::vector<uint64_t> tiles;
  std::vector<std::vector<int>> rows_after;
  uint64_t forced = 0;
  for (int r = 0; r < rowbits; ++r) forced |= 1ull << wire_at[r];
  std::vector<int> seg_first(NS, 0), seg_last(NS, -1);
  std::vector<char> seg_diag(NS, 0);
  for (size_t i = 0; i < G.size(); ++i)
    if (G[i].diag) seg_diag[seg_of_gate(i)] = 1;
  for (cur_seg = 0; cur_seg < NS; ++cur_seg) {
  seg_first[cur_seg] = (int)tiles.size();
  int left = 0;
  for (int k = 0; k < N; ++k) left += nseg[k] == cur_seg;
  if (!left && seg_diag[cur_seg] && (NS > 1 || N == 0)) {  // diagonal gates only: one pass over the row bits
    tiles.push_back(forced);
    rows_after.push_back(std::vector<int>(wire_at.begin(), wire_at.begin() + rowbits));
  }
  while (left > 0) {
    const uint64_t S = choose(forced);
    std::vector<uint64_t> now;
    int c = 0;
    closure(S, now, &c);
    if (!c) return false;
    for (int k = 0; k < N; ++k)
      if (isdone(now, k) && !isdone(done, k)) npass[k] = (int)tiles.size();
    done = now;
    while (first_open < N && isdone(done, first_open)) ++first_open;
    left -= c;
    tiles.push_back(S);
    // row bits after this pass: wires the next pass (lookahead) wants that the
    // tile holds; rows whose wire the next pass wants keep it
    std::vector<int> rows(rowbits);
    for (int r = 0; r < rowbits; ++r) rows[r] = wire_at[r];
    if (left > 0) {
      const uint64_t S2 = choose(0);
      std::vector<char> keep(rowbits, 0);
      uint64_t placed = 0;
      for (int r = 0; r < rowbits; ++r)
        if (S2 >> rows[r] & 1) keep[r] = 1, placed |= 1ull << rows[r];
      uint64_t cand = S & S2 & ~placed;
      for (int r = 0; r < rowbits && cand; ++r) {
        if (keep[r]) continue;
        const int w = __builtin_ctzll(cand);
        cand &= cand - 1;
        rows[r] = w;
      }
    } else if (cur_seg < (int)bars.size()) {
      // the segment's last pass: wires that leave at the barrier come off the
      // row bits (an exchange over bits 0..2 moves 16-B pieces)
      uint64_t leave = 0, onrow = 0;
      for (size_t k = 0; k < bars[cur_seg].ins->b.size(); ++k) {
        std::vector<int> sa = bars[cur_seg].ins->a, sb = bars[cur_seg].ins->b;
        std::sort(sa.begin(), sa.end());
        std::sort(sb.begin(), sb.end());
        if (sb[k] >= nb) leave |= 1ull << bars[cur_seg].xw[sa[k]];
      }
      for (int r = 0; r < rowbits; ++r) onrow |= 1ull << rows[r];
      uint64_t cand = S & ~leave & ~onrow;
      for (int r = 0; r < rowbits && cand; ++r) {
        if (!(leave >> rows[r] & 1)) continue;
        const int w = __builtin_ctzll(cand);
        cand &= cand - 1;
        rows[r] = w;
      }
    }
    rows_after.push_back(rows);
    // the layout after the pass: only the row assignment matters here
    std::vector<int> pos(ntot, -1);
    for (int q = 0; q < nb; ++q) pos[wire_at[q]] = q;
    for (int r = 0; r < rowbits; ++r) {
      const int w = rows[r], from = pos[w], displaced = wire_at[r];
      wire_at[r] = w;
      wire_at[from] = displaced;
      pos[w] = r;
      pos[displaced] = from;
    }
    forced = 0;
    for (int r = 0; r < rowbits; ++r) forced |= 1ull << wire_at[r];
  }
  seg_last[cur_seg] = (int)tiles.size() - 1;
  if (cur_seg < (int)bars.size()) {
    // the barrier's wire moves: a held pair swaps the two bits' wires, an
    // outside pair brings the rank position's wire onto the local bit
    const Bar& br = bars[cur_seg];
    std::vector<int> sa = br.ins->a, sb = br.ins->b;
    std::sort(sa.begin(), sa.end());
    std::sort(sb.begin(), sb.end());
    std::vector<int> pos(ntot, -1);
    for (int x = 0; x < nb; ++x) pos[wire_at[x]] = x;
    for (size_t k = 0; k < sa.size(); ++k) {
      const int wa = br.xw[sa[k]], wb = br.xw[sb[k]];
      const int xa = pos[wa];
      if (xa < 0) return false;
      if (sb[k] < nb) {
        const int xb = pos[wb];
        if (xb < 0) return false;
        wire_at[xa] = wb;
        wire_at[xb] = wa;
      } else {
        wire_at[xa] = wb;
      }
    }
    forced = 0;
    for (int r = 0; r < rowbits; ++r) forced |= 1ull << wire_at[r];
  }
  }
  if (tiles.empty()) {  // only diagonal gates: one pass over the row bits
    tiles.push_back(forced);
    rows_after.push_back(std::vector<int>(wire_at.begin(), wire_at.begin() + rowbits));
    seg_last[0] = 0;
  }
  // pass of every gate: non-diagonal from the schedule, diagonal = the latest
  // pass among its predecessors (0 if none)
  std::vector<int> gpass(G.size(), 0);
  for (int k = 0; k < N; ++k) gpass[nd[k]] = npass[k];
  for (size_t i = 0; i < G.size(); ++i)
    if (G[i].diag) {
      for (int k : ddep[i]) gpass[i] = std::max(gpass[i], npass[k]);
      gpass[i] = std::max(gpass[i], seg_first[seg_of_gate(i)]);
      if (seg_last[seg_of_gate(i)] < gpass[i]) return false;
    }
  // Latest pass a diagonal gate may run in: that of its first non-diagonal
  // successor on any of its wires (the last pass if none). A pass's tail —
  // the diagonal gates no later non-diagonal gate of the pass touches —
  // moves to the next pass when every gate of it would be tail there too:
  // it then joins that pass's tail run instead of costing a run of its own
  // (QAOA: the next layer's phases among a pass's own wires stop being a
  // 12-bit table in front of the store).
  {
    const int P = (int)tiles.size();
    std::vector<int> latest(G.size(), P - 1);
    for (size_t i = 0; i < G.size(); ++i) latest[i] = std::min(latest[i], seg_last[seg_of_gate(i)]);
    std::vector<int> next_nd(ntot, -1);  // scanning backwards: next non-diagonal gate per wire
    for (int i = (int)G.size() - 1; i >= 0; --i) {
      if (G[i].diag) {
        for (int w = 0; w < ntot; ++w)
          if ((G[i].wm >> w & 1) && next_nd[w] >= 0) latest[i] = std::min(latest[i], gpass[next_nd[w]]);
      } else {
        for (int w = 0; w < ntot; ++w)
          if (G[i].wm >> w & 1) next_nd[w] = i;
      }
    }
    if (!getenv("QK_NO_TAIL_MOVE"))
      for (int p = 0; p + 1 < P; ++p) {
        std::vector<int> tail;
        uint64_t later = 0;  // wires of non-diagonal gates of pass p after the scan point
        bool all = true;
        for (int i = (int)G.size() - 1; i >= 0; --i) {
          if (gpass[i] != p) continue;
          if (!G[i].diag) {
            later |= G[i].wm;
            continue;
          }
          if (G[i].wm & later) continue;  // a later gate of the pass needs it first
          tail.push_back(i);
          all = all && latest[i] > p + 1;
        }
        if (all)
          for (int i : tail) gpass[i] = p + 1;
      }
  }
  std::vector<InstrH> passes(tiles.size());
  for (size_t p = 0; p < tiles.size(); ++p) {
    InstrH& b = passes[p];
    b.type = QK_INS_BLOCK;
    b.rb = 1;
    for (int w = 0; w < ntot; ++w)
      if (tiles[p] >> w & 1) b.tile_w.push_back(w);
    b.rows_next = rows_after[p];
  }
  // gates in program order, each diagonal one moved down to just before the
  // first later non-diagonal gate of its pass that shares a wire (the end if
  // none), so the kernels see few, large diagonal runs
  std::vector<std::vector<int>> pg(tiles.size());
  for (size_t i = 0; i < G.size(); ++i) pg[gpass[i]].push_back((int)i);
  for (size_t p = 0; p < tiles.size(); ++p) {
    const std::vector<int>& v = pg[p];
    std::vector<int> tail;
    std::vector<std::vector<int>> before(v.size());
    for (size_t a = 0; a < v.size(); ++a) {
      if (!G[v[a]].diag) continue;
      size_t dl = v.size();
      for (size_t c2 = a + 1; c2 < v.size(); ++c2)
        if (!G[v[c2]].diag && (G[v[c2]].wm & G[v[a]].wm)) {
          dl = c2;
          break;
        }
      (dl == v.size() ? tail : before[dl]).push_back(v[a]);
    }
    std::vector<int> order;
    for (size_t a = 0; a < v.size(); ++a) {
      for (int i : before[a]) order.push_back(i);
      if (!G[v[a]].diag) order.push_back(v[a]);
    }
    order.insert(order.end(), tail.begin(), tail.end());
    for (int i : order) {
      GateH g = *G[i].g;
      g.t = G[i].w;
      passes[p].gates.push_back(std::move(g));
    }
  }
  // passes in order, each barrier after the last pass of its segment
  out->clear();
  size_t bi = 0;
  auto flush_bars = [&](int upto) {
    while (bi < bars.size() && seg_last[bi] <= upto) {
      InstrH c = *bars[bi].ins;
      c.rb = 1;
      c.xw = bars[bi].xw;
      out->push_back(std::move(c));
      ++bi;
    }
  };
  flush_bars(-1);
  for (size_t p = 0; p < passes.size(); ++p) {
    out->push_back(std::move(passes[p]));
    flush_bars((int)p);
  }
  flush_bars(INT32_MAX);
  return true;
}

// The schedule is a pure function of the program and its arguments; loading
// the same circuit again (every end-to-end step does) reuses it, like the
// generated pass sources. Process-wide, bounded.
void pack_prog(const std::vector<InstrH>& prog, std::vector<int32_t>* wp, std::vector<double>* pp);
bool reblock_memo(const std::vector<InstrH>& prog, int nb, int cap, int rowbits, std::vector<InstrH>* out,
                  std::vector<int>* p2w_final, int ntot, const std::vector<int>* init_pos) {
  if (getenv("QK_NO_PLAN_MEMO")) return reblock(prog, nb, cap, rowbits, out, p2w_final, ntot, init_pos);
  std::vector<int32_t> w;
  std::vector<double> pr;
  pack_prog(prog, &w, &pr);
  std::string key(reinterpret_cast<const char*>(w.data()), w.size() * 4);
  key.append(reinterpret_cast<const char*>(pr.data()), pr.size() * 8);
  const int args[4] = {nb, cap, rowbits, ntot};
  key.append(reinterpret_cast<const char*>(args), sizeof args);
  if (init_pos) key.append(reinterpret_cast<const char*>(init_pos->data()), init_pos->size() * sizeof(int));
  struct Memo {
    bool ok;
    std::vector<InstrH> out;
    std::vector<int> p2w;
  };
  static std::mutex mu;
  static std::map<std::string, Memo> memo;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) {
      *out = it->second.out;
      *p2w_final = it->second.p2w;
      return it->second.ok;
    }
  }
  const bool ok = reblock(prog, nb, cap, rowbits, out, p2w_final, ntot, init_pos);
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() > 64) memo.clear();
  memo[key] = Memo{ok, ok ? *out : std::vector<InstrH>(), ok ? *p2w_final : std::vector<int>()};
  return ok;
}

// Whole-plan memo (host side only: the device tables, tensor maps and
// kernels are still built by upload_plan for every load). Key: the packed
// program, the handle's shape and every QK_* switch of the environment.
struct PlanMemo {
  HostPlan hp;
  std::vector<InstrPlan> iplan;
  std::vector<int> plan_lay0, lay_final;
  bool oop_sqs = false, reblocked = false;
};
std::mutex g_plan_mu;
std::map<std::string, PlanMemo> g_plan_memo;

std::string plan_key(const qk_sim* s, bool try_reblock) {
  std::vector<int32_t> w;
  std::vector<double> pr;
  pack_prog(s->prog, &w, &pr);
  std::string key(reinterpret_cast<const char*>(w.data()), w.size() * 4);
  key.append(reinterpret_cast<const char*>(pr.data()), pr.size() * 8);
  const int shape[12] = {s->n, s->r, s->b, s->L, s->nbits, s->count, s->rank_lo, (int)s->gbg, s->bufs[1] != nullptr,
                         (int)try_reblock, (int)jit_available(), (int)s->dry};
  key.append(reinterpret_cast<const char*>(shape), sizeof shape);
  std::vector<std::string> env;
  for (char** e = environ; e && *e; ++e)
    if (!strncmp(*e, "QK_", 3)) env.push_back(*e);
  std::sort(env.begin(), env.end());
  for (auto& e : env) key += "|" + e;
  return key;
}

int compile_program_impl(qk_sim* s, bool try_reblock, bool* reblocked) {
  const auto tc0 = std::chrono::steady_clock::now();
  struct PlanTimer {
    std::chrono::steady_clock::time_point t0;
    ~PlanTimer() {
      if (getenv("QK_DUMP_LOAD"))
        fprintf(stderr, "load: compile_program total %.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  } plan_timer{tc0};
  s->hp.clear();
  s->iplan.clear();
  const bool memo_on = !getenv("QK_NO_PLAN_MEMO");
  const std::string pkey = memo_on ? plan_key(s, try_reblock) : std::string();
  if (memo_on) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plan_memo.find(pkey);
    if (it != g_plan_memo.end()) {
      s->hp = it->second.hp;
      s->iplan = it->second.iplan;
      s->plan_lay0 = it->second.plan_lay0;
      s->lay_final = it->second.lay_final;
      s->oop_sqs = it->second.oop_sqs;
      *reblocked = it->second.reblocked;
    }
  }
  if (!s->iplan.empty() || !s->hp.passes.empty()) {
    replay_perm(s);
    const auto tq0 = std::chrono::steady_clock::now();
    const int urc = upload_plan(s);
    if (getenv("QK_DUMP_LOAD"))
      fprintf(stderr, "load: plan memo hit, upload_plan %.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
    return urc;
  }
  std::string emsg;
  const int nb = s->nbits;
  // Relabeling mode (needs the second buffer): every block runs with the same
  // chunk width Cg over address bits [0, Cg); a plan-time map sigma (reference
  // position -> address bit) absorbs SQS runs into the preceding block's
  // out-of-place store. The store's destination layout keeps the next chunk
  // contiguous and puts >= 5 qubits that stay in the chunk on the lowest
  // address bits, so every warp still writes whole 512-B runs.
  int Cg = 0;
  bool relabel = s->bufs[1] && !s->gbg && !getenv("QK_NO_FUSE") && !getenv("QK_NO_TMA");
  bool all_chunked = true;
  for (auto& ins : s->prog) {
    if (ins.type != QK_INS_BLOCK || ins.gates.empty()) continue;
    const int w = block_chunk_width(ins, s->L);
    if (!w) relabel = all_chunked = false;
    Cg = std::max(Cg, w);
  }
  if (Cg < 9 || Cg > 12 || Cg > nb) relabel = false;
  // cluster-exchange fusion needs the load-time specialised kernels
  const char* jenv = getenv("QK_JIT");
  const bool xfuse = relabel && !getenv("QK_NO_XFUSE") && jit_available() && nb >= (jenv ? atoi(jenv) : 20);
  const bool fold = relabel && !getenv("QK_NO_FOLD") && jit_available() && nb >= (jenv ? atoi(jenv) : 20);
  std::vector<int> sigma(nb);
  for (int q = 0; q < nb; ++q) sigma[q] = q;
  // Lazy in-place mode (no second buffer, e.g. 33 qubits on one B200): SQS and
  // in-handle CSQS only relabel (sigma); a block runs as one strided-tile pass
  // over its targets' current physical bits plus bits 0..2 (128-B rows), stored
  // back in place. The handle keeps the end layout (lay_final), maps every
  // readback through it and restores the reference layout before writers.
  // It also replaces relabeling when every chunk is <= 10 qubits (the tiles
  // then stay <= 13 bits; QFT30: 0.112 s lazy vs 0.132 s relabeled).
  const bool lazy_ok = !s->gbg && !getenv("QK_NO_LAZY") && !getenv("QK_NO_TMA") && jit_available() &&
                       nb >= (jenv ? atoi(jenv) : 20) && nb >= 16;
  // It also takes chunks of 11-12 qubits: a block whose tile would exceed 13
  // bits first gets one SQS pass that brings its qubits onto bits 0..11
  // (emit_fixup). The in-tile store permutations keep that rare: QAOA30 needs
  // one fix-up and no other swap pass (0.18 s, against 0.26 s relabeled with
  // 10 SQS passes and 4.3 -> 1.8 s for QAOA33 in place, which ran its swaps).
  const bool lazy = lazy_ok && all_chunked && (!s->bufs[1] || relabel) &&
                    (Cg <= 10 || (Cg <= 12 && !getenv("QK_NO_LAZY12")));
  if (lazy) relabel = false;
  // cross-block pass scheduling (reblock): lazy layout, every swap inside
  // the handle, every diagonal gate quadratic; checked up front so the
  // reference's errors (swap ranges, CSQS contract) still come from the loop
  std::vector<InstrH> rprog;
  std::vector<int> rb_p2w;
  *reblocked = false;
  if (try_reblock && lazy && !getenv("QK_NO_FOLD")) {
    bool ok = true;
    for (auto& ins : s->prog) {
      if (ins.type == QK_INS_SQS) {
        for (int q : ins.a) ok = ok && q >= 0 && q < s->L;
        for (int q : ins.b) ok = ok && q >= 0 && q < s->L;
      } else if (ins.type == QK_INS_CSQS) {
        ok = ok && check_csqs(s, ins.a, ins.b) == QK_OK;
        // rank bits held by other shards: a barrier of the schedule (QK_NO_XREBLOCK: block order)
        for (int q : ins.b) ok = ok && (q < nb || !getenv("QK_NO_XREBLOCK"));
      }
    }
    const char* cenv = getenv("QK_REBLOCK_CAP");
    const auto trb = std::chrono::steady_clock::now();
    // row bits forced into every tile: 3 (128-B rows); QK_ROWBITS=4 (dev) gives 256-B row segments
    const int rowb = getenv("QK_ROWBITS") ? atoi(getenv("QK_ROWBITS")) : 3;
    const bool rbok = ok && reblock_memo(s->prog, nb, cenv ? atoi(cenv) : 12, rowb, &rprog, &rb_p2w, s->n, nullptr);
    if (getenv("QK_DUMP_LOAD"))
      fprintf(stderr, "load: reblock %.3f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - trb).count());
    if (rbok) {
      // worth it only with fewer sweeps than the block order (one per block
      // that is not diagonal-only; those fold into the pass before)
      size_t sweeps = 0, passes = 0;
      for (auto& ins : s->prog) {
        if (ins.type != QK_INS_BLOCK || ins.gates.empty()) continue;
        bool dg = true;
        for (auto& g : ins.gates) dg = dg && is_diag(g.kind);
        sweeps += !dg;
      }
      for (auto& ins : rprog) passes += ins.type == QK_INS_BLOCK;
      *reblocked = passes < std::max<size_t>(sweeps, 1) || getenv("QK_REBLOCK");
    }
  }
  // First-use placement: a run from |0...0> may start in any layout, so the
  // wires go to physical bits in the order the schedule first puts them in a
  // tile. The zero support then grows from the bottom: each early pass reads
  // and writes only the prefix its wires span (QFT/BV/H circuits whose first
  // gates sit on high qubits get the same cheap early passes as QAOA).
  s->plan_lay0.clear();
  if (*reblocked && !getenv("QK_NO_ZPLACE")) {
    std::vector<int> pos(nb, -1), order;
    for (const InstrH& ins : rprog)
      if (ins.type == QK_INS_BLOCK)
        for (int w : ins.tile_w)
          if (w < nb && pos[w] < 0) {
            pos[w] = (int)order.size();
            order.push_back(w);
          }
    for (int w = 0; w < nb; ++w)
      if (pos[w] < 0) {
        pos[w] = (int)order.size();
        order.push_back(w);
      }
    bool ident_pos = true;
    for (int w = 0; w < nb; ++w) ident_pos = ident_pos && pos[w] == w;
    std::vector<InstrH> rprog2;
    std::vector<int> p2w2;
    const char* cenv2 = getenv("QK_REBLOCK_CAP");
    const int rowb2 = getenv("QK_ROWBITS") ? atoi(getenv("QK_ROWBITS")) : 3;
    if (!ident_pos && reblock_memo(s->prog, nb, cenv2 ? atoi(cenv2) : 12, rowb2, &rprog2, &p2w2, s->n, &pos)) {
      size_t n1 = 0, n2 = 0;
      for (auto& ins : rprog) n1 += ins.type == QK_INS_BLOCK;
      for (auto& ins : rprog2) n2 += ins.type == QK_INS_BLOCK;
      if (n2 <= n1) {
        rprog.swap(rprog2);
        rb_p2w.swap(p2w2);
        s->plan_lay0 = pos;
        for (int q = 0; q < nb; ++q) sigma[q] = pos[q];
      }
    }
  }
  // reblocked: sigma is indexed by wire; wires of other shards' rank bits sit outside (-1)
  if (*reblocked && s->n > nb) {
    sigma.resize(s->n);
    for (int w = nb; w < s->n; ++w) sigma[w] = -1;
  }
  const std::vector<InstrH>& prog = *reblocked ? rprog : s->prog;
  const auto tloop = std::chrono::steady_clock::now();
  auto emit_restore = [&]() {
    std::vector<std::pair<int, int>> rounds[2];
    restore_rounds(sigma, rounds);
    for (auto& rd : rounds) {
      if (rd.empty()) continue;
      std::vector<int> A, B;
      for (auto& pr : rd) {
        A.push_back(pr.first);
        B.push_back(pr.second);
      }
      InstrPlan rp;
      rp.type = QK_INS_SQS;
      rp.synthetic = 1;
      rp.sqs = compile_sqs(s->hp, A, B, nb, true);
      rp.bytes = 32.0 * std::ldexp(1.0, nb) * (1.0 - std::ldexp(1.0, -(int)A.size()));
      s->iplan.push_back(std::move(rp));
      for (int& v : sigma)
        for (auto& pr : rd) {
          if (v == pr.first) { v = pr.second; break; }
          if (v == pr.second) { v = pr.first; break; }
        }
    }
    return lay_identity(sigma);
  };
  // one SQS pass moving the physical bits `need` (a block's qubits) onto
  // bits [0, lo): each one above pairs with a free bit below
  auto emit_fixup = [&](const std::vector<int>& need, int lo) {
    std::vector<char> in(nb, 0);
    for (int p : need) in[p] = 1;
    std::vector<int> A, B;
    int f = 0;
    for (int p : need) {
      if (p < lo) continue;
      while (f < lo && in[f]) ++f;
      if (f >= lo) return false;
      A.push_back(p);
      B.push_back(f);
      in[f] = 1;
      ++f;
    }
    if (A.empty()) return true;
    InstrPlan rp;
    rp.type = QK_INS_SQS;
    rp.synthetic = 1;
    rp.sqs = compile_sqs(s->hp, A, B, nb, true);
    rp.bytes = 32.0 * std::ldexp(1.0, nb) * (1.0 - std::ldexp(1.0, -(int)A.size()));
    s->iplan.push_back(std::move(rp));
    for (int& v : sigma)
      for (size_t k = 0; k < A.size(); ++k) {
        if (v == A[k]) { v = B[k]; break; }
        if (v == B[k]) { v = A[k]; break; }
      }
    return true;
  };
  std::vector<int> ident(nb);
  for (int q = 0; q < nb; ++q) ident[q] = q;
  std::vector<char> fused(prog.size(), 0);
  auto diag_block = [&](const InstrH& b) {
    if (b.type != QK_INS_BLOCK || b.gates.empty()) return false;
    for (auto& g : b.gates) {
      if (!is_diag(g.kind)) return false;
      for (int t : g.t)
        if (t < 0 || t >= nb) return false;
    }
    return true;
  };
  const bool lazy_fold = lazy && !getenv("QK_NO_FOLD");
  const bool fold_eager = !s->gbg && !getenv("QK_NO_FOLD") && jit_available() && nb >= (jenv ? atoi(jenv) : 20);
  const bool merge_sqs = !relabel && !lazy && !getenv("QK_NO_SQS_MERGE");
  std::vector<int> folded_into(prog.size(), -1);  // lazy mode: diagonal block -> absorbing pass
  auto remap = [&](const InstrH& ins) {
    InstrH m = ins;
    for (auto& g : m.gates)
      for (int& t : g.t) t = sigma[t];
    return m;
  };
  for (size_t ii = 0; ii < prog.size(); ++ii) {
    auto& ins = prog[ii];
    InstrPlan ip;
    ip.type = ins.type;
    // eager mode: a run of swaps (diagonal blocks folded away in between) is
    // composed on the host and executed as at most two SQS passes, since any
    // bit permutation is a product of two involutions (restore_rounds)
    if (merge_sqs && !lay_identity(sigma) && ins.type != QK_INS_SQS &&
        !(ins.type == QK_INS_BLOCK && (folded_into[ii] >= 0 || ins.gates.empty())) && !emit_restore())
      return fail(QK_ESIM, "internal: swap run merge failed");
    if (ins.type == QK_INS_BLOCK && folded_into[ii] >= 0) {
      ip.fused_by = folded_into[ii];  // applied by an earlier pass (no kernel)
      s->iplan.push_back(std::move(ip));
      continue;
    }
    if (ins.type == QK_INS_BLOCK && lazy && !ins.gates.empty()) {
      {
        // a tile over 13 bits (or more strided runs than the TMA view takes):
        // bring the block's qubits down first
        std::vector<char> inP(nb, 0);
        std::vector<int> P;
        if (ins.rb) {
          for (int w : ins.tile_w)
            if (!inP[sigma[w]]) {
              inP[sigma[w]] = 1;
              P.push_back(sigma[w]);
            }
        } else {
          for (auto& g : ins.gates)
            for (int t : g.t)
              if (t >= 0 && t < nb && !inP[sigma[t]]) {
                inP[sigma[t]] = 1;
                P.push_back(sigma[t]);
              }
        }
        int c3 = 0;
        for (int p = 0; p < nb; ++p) c3 += inP[p] || p < 3;
        std::vector<int> T3;
        for (int p = 0; p < nb; ++p)
          if (inP[p] || p < 3 || (c3 < 10 && p < 10)) T3.push_back(p);
        uint8_t tb3[16] = {0};
        for (size_t x = 0; x < T3.size() && x < 16; ++x) tb3[x] = (uint8_t)T3[x];
        TileDims td3{};
        const bool fits = T3.size() <= 13 && tile_dims(tb3, (int)T3.size(), nb, &td3, 3);
        if (!fits && (Cg > 10 || ins.rb) && !getenv("QK_NO_FIXUP")) {
          std::sort(P.begin(), P.end());
          if (!emit_fixup(P, std::min(nb, std::max(12, (int)P.size()))))
            return fail(QK_ESIM, "internal: layout fix-up failed");
        }
      }
      InstrH mapped = remap(ins);
      std::vector<char> inT(nb, 0);
      int maxt = -1;
      for (auto& g : mapped.gates)
        for (int t : g.t) {
          if (t < 0 || t >= nb) return fail(QK_ESIM, "gate target %d beyond local range", t);
          if (ins.rb) continue;  // the scheduler's tile: diagonal targets may stay outside
          inT[t] = 1;
          maxt = std::max(maxt, t);
        }
      for (int w : ins.tile_w) inT[sigma[w]] = 1;
      // row bits: 0..2 (128-B rows); when that makes a 13-bit tile (one
      // 128-KiB stage) and 0..1 keeps it at 12, take 64-B rows and 3 stages,
      // unless the tile spans many 2-MiB pages (address bits >= 17): its 1024
      // rows then miss the TLB and half-size rows double that cost per byte
      // (H33: 50 ms with 8 pages, 118 ms with 1024 pages, 88 ms at 128-B rows)
      int rows = 3;
      {
        int c3 = 0, c2b = 0, pagebits = 0;
        for (int p = 0; p < nb; ++p) {
          c3 += inT[p] || p < 3;
          c2b += inT[p] || p < 2;
          pagebits += inT[p] && p >= 17;
        }
        // dense 2x2 gates keep the 13-bit tile: its 512 consumer threads hide
        // the FP64 chains the 256-thread 12-bit pass exposes (U33: 124 vs 90 ms)
        bool dense = false;
        for (auto& g : mapped.gates) dense = dense || g.kind == QK_U || g.kind == QK_RX || g.kind == QK_RY;
        if (c3 > 12 && c2b <= 12 && pagebits <= 4 && !dense && !getenv("QK_NO_ROW64")) rows = 2;
      }
      for (int p = 0; p < rows; ++p) inT[p] = 1;
      int cnt = 0;
      for (char c2 : inT) cnt += c2;
      // pad with the lowest free bits to 10 (QK_PAD: padding the small last
      // passes of the schedule to 12 measured mixed: BV33 -2.2 ms, QFT33 +4.7 ms)
      const int pad = getenv("QK_PAD") ? atoi(getenv("QK_PAD")) : 10;
      for (int p = 0; p < nb && cnt < pad; ++p)
        if (!inT[p]) inT[p] = 1, ++cnt;
      std::vector<int> T;
      for (int p = 0; p < nb; ++p)
        if (inT[p]) T.push_back(p);
      const bool contiguous = T.back() == (int)T.size() - 1 && T.size() <= 12 && !lazy_fold;
      TileDims tdchk{};
      uint8_t tb8[16] = {0};
      for (size_t x = 0; x < T.size() && x < 16; ++x) tb8[x] = (uint8_t)T[x];
      if (cnt <= 13 && !contiguous && tile_dims(tb8, cnt, nb, &tdchk, inT[2] ? 3 : 2)) {
        // Store permutation inside the tile (in place, same address set):
        // qubits the next block needs move onto bits 0..2, so its tile only
        // has to add what is missing (10 bits instead of 13 when all fit).
        std::vector<int> dphys = ident;
        std::vector<int> sig2 = sigma;
        size_t jj = ii + 1;
        bool ok = true;
        for (; jj < prog.size(); ++jj) {
          const InstrH& nx = prog[jj];
          if (nx.type == QK_INS_BLOCK) {
            if (!nx.gates.empty() && !(lazy_fold && diag_block(nx))) break;
            continue;
          }
          bool in_local = true;
          for (int q : nx.a) in_local = in_local && q >= 0 && q < nb;
          for (int q : nx.b) in_local = in_local && q >= 0 && q < nb;
          if (!in_local) {
            ok = false;
            break;
          }
          std::vector<int> sa = nx.a, sb = nx.b;
          std::sort(sa.begin(), sa.end());
          std::sort(sb.begin(), sb.end());
          for (size_t k = 0; k < sa.size(); ++k) std::swap(sig2[sa[k]], sig2[sb[k]]);
        }
        if (ins.rb && !getenv("QK_NO_LAZY_PERM")) {
          // the scheduler's rows: rows_next on bits 0.., then the next pass's
          // tile wires, then the rest, each group in ascending bit order,
          // onto the tile's bits in ascending order
          std::vector<char> used(nb, 0), nxt(nb, 0), leave(nb, 0);
          if (jj < prog.size())
            for (int w : prog[jj].tile_w) nxt[sigma[w]] = 1;
          if (jj < prog.size() && prog[jj].type == QK_INS_CSQS && prog[jj].rb) {
            // a barrier next: the wires it sends away go to the highest tile
            // bits, so the exchange moves long contiguous runs
            const InstrH& bx = prog[jj];
            std::vector<int> sa = bx.a, sb = bx.b;
            std::sort(sa.begin(), sa.end());
            std::sort(sb.begin(), sb.end());
            for (size_t k = 0; k < sa.size(); ++k)
              if (sb[k] >= nb && sigma[bx.xw[sa[k]]] >= 0) leave[sigma[bx.xw[sa[k]]]] = 1;
          }
          std::vector<int> srcs;
          bool rows_ok = true;
          for (int w : ins.rows_next) {
            const int p0 = sigma[w];
            rows_ok = rows_ok && inT[p0] && !used[p0];
            if (!rows_ok) break;
            used[p0] = 1;
            srcs.push_back(p0);
          }
          if (rows_ok && (int)srcs.size() <= (inT[2] ? 3 : 2)) {
            for (int x : T)
              if (!used[x] && nxt[x]) used[x] = 1, srcs.push_back(x);
            for (int x : T)
              if (!used[x] && !leave[x]) used[x] = 1, srcs.push_back(x);
            for (int x : T)
              if (!used[x]) used[x] = 1, srcs.push_back(x);
            dphys = ident;
            for (size_t k = 0; k < T.size(); ++k) dphys[srcs[k]] = T[k];
          }
        } else if (ok && jj < prog.size() && !getenv("QK_NO_LAZY_PERM")) {
          std::vector<char> need(nb, 0);
          for (auto& g : prog[jj].gates)
            for (int t : g.t)
              if (t >= 0 && t < nb) need[sig2[t]] = 1;
          std::vector<int> want, low;
          for (int p : T)
            if (p >= 3 && need[p]) want.push_back(p);
          for (int p = 0; p < 3; ++p)
            if (!need[p] && inT[p]) low.push_back(p);  // in place: only inside the tile
          // The qubits moved onto the row bits must be lanes of the last phase;
          // when that costs a layout-only phase, try other picks among the
          // wanted qubits (phase count of the block's own gates decides).
          std::vector<const GateH*> own;
          for (auto& g : mapped.gates) own.push_back(&g);
          auto nph = [&](const std::vector<int>& dp) {
            HostPlan tmp;
            std::string em;
            if (compile_pass(tmp, own, T, nb, 0, em, &dp, inT[2] ? 3 : 2) || tmp.passes.empty()) return 99;
            return tmp.passes.back().nphases;
          };
          // The picks take the free row bits; the other wanted qubits then
          // take the lowest remaining tile positions in order, so the next
          // tile has fewer strided runs and pages (QK_NO_PACK: rows only).
          const bool pack = !getenv("QK_NO_PACK");
          auto make = [&](const std::vector<int>& pick) {
            std::vector<int> dp = ident;
            std::vector<char> used(nb, 0), taken(nb, 0);
            size_t k = 0;
            for (int r : low)
              if (k < pick.size()) {
                dp[pick[k]] = r;
                used[pick[k]] = taken[r] = 1;
                ++k;
              }
            std::vector<int> slots, srcs;
            for (int x : T)
              if (!taken[x] && !(x < 3 && !std::count(low.begin(), low.end(), x))) slots.push_back(x);
            for (int x : T)
              if (x < 3 && !std::count(low.begin(), low.end(), x)) used[x] = 1;  // needed row bits stay
            if (pack)
              for (int x : want)
                if (!used[x]) {
                  srcs.push_back(x);
                  used[x] = 1;
                }
            for (int x : T)
              if (!used[x]) srcs.push_back(x);
            if (srcs.size() != slots.size()) {  // should not happen: rows only
              dp = ident;
              for (size_t j = 0; j < pick.size() && j < low.size(); ++j) {
                dp[low[j]] = pick[j];
                dp[pick[j]] = low[j];
              }
              return dp;
            }
            for (size_t j = 0; j < srcs.size(); ++j) dp[srcs[j]] = slots[j];
            return dp;
          };
          std::vector<std::vector<int>> cands;
          cands.push_back(want);
          cands.push_back(std::vector<int>(want.rbegin(), want.rend()));
          for (size_t k = 0; k + low.size() <= want.size() && k < 8; ++k)
            cands.push_back(std::vector<int>(want.begin() + k, want.end()));
          int best_ph = 99;
          size_t best_moves = 0;
          for (auto& c : cands) {
            const std::vector<int> dp = make(c);
            const int ph = nph(dp);
            const size_t mv = std::min(c.size(), low.size());
            // more moves first (the next tile shrinks), then fewer phases
            if (mv > best_moves || (mv == best_moves && ph < best_ph)) {
              best_ph = ph;
              best_moves = mv;
              dphys = dp;
            }
          }
        }
        // fold the diagonal-only blocks up to the next other block: their
        // qubits sit (after the lazy swaps in between) at sig3[t], i.e. at
        // dinv[sig3[t]] before this pass's store permutation dphys
        std::vector<GateH> folded;
        std::vector<size_t> folded_at;
        if (lazy_fold) {
          std::vector<int> dinv(nb);
          for (int q = 0; q < nb; ++q) dinv[dphys[q]] = q;
          std::vector<int> sig3(sigma.size(), -1);
          for (size_t q = 0; q < sigma.size(); ++q) sig3[q] = sigma[q] >= 0 ? dphys[sigma[q]] : -1;
          for (size_t j = ii + 1; j < prog.size(); ++j) {
            const InstrH& nx = prog[j];
            if (nx.type == QK_INS_BLOCK) {
              if (nx.gates.empty()) continue;
              if (!diag_block(nx)) break;
              bool local = true;
              for (auto& g : nx.gates)
                for (int t : g.t) local = local && t >= 0 && t < (int)sig3.size() && sig3[t] >= 0;
              if (!local) break;
              for (auto& g : nx.gates) {
                GateH m = g;
                for (int& t : m.t) t = dinv[sig3[t]];
                folded.push_back(m);
              }
              folded_at.push_back(j);
              continue;
            }
            bool in_local = true;
            for (int q : nx.a) in_local = in_local && q >= 0 && q < nb;
            for (int q : nx.b) in_local = in_local && q >= 0 && q < nb;
            if (!in_local) break;
            std::vector<int> sa = nx.a, sb = nx.b;
            std::sort(sa.begin(), sa.end());
            std::sort(sb.begin(), sb.end());
            for (size_t k = 0; k < sa.size(); ++k) std::swap(sig3[sa[k]], sig3[sb[k]]);
          }
        }
        std::vector<const GateH*> gs;
        for (auto& g : mapped.gates) gs.push_back(&g);
        for (auto& g : folded) gs.push_back(&g);
        ip.pass0 = (int)s->hp.passes.size();
        int rc = compile_pass(s->hp, gs, T, nb, 0, emsg, &dphys, inT[2] ? 3 : 2, ins.rb != 0);
        if (ins.rb && !rc && !tma_plan_ok(s->hp, ip.pass0, nb, 13))
          return fail(QK_ESIM, "reblock: pass %d does not fit the specialised kernel", ip.pass0);
        if (!rc && !folded.empty() && !tma_plan_ok(s->hp, ip.pass0, nb, 13)) {
          // too many ops for one specialised pass: the folded blocks run on their own
          s->hp.passes.resize(ip.pass0);
          folded.clear();
          folded_at.clear();
          gs.resize(mapped.gates.size());
          rc = compile_pass(s->hp, gs, T, nb, 0, emsg, &dphys, inT[2] ? 3 : 2);
        }
        if (!rc && !tma_plan_ok(s->hp, ip.pass0, nb, 13) && dphys != ident) {
          // the generic pass will run it: no in-tile store permutation
          s->hp.passes.resize(ip.pass0);
          dphys = ident;
          rc = compile_pass(s->hp, gs, T, nb, 0, emsg, &dphys, inT[2] ? 3 : 2);
        }
        if (rc) return fail(rc, "%s", emsg.c_str());
        ip.npass = (int)s->hp.passes.size() - ip.pass0;
        ip.bytes = 32.0 * std::ldexp(1.0, nb) * ip.npass;
        ip.tile = T;
        ip.dest = dphys;
        for (int& v : sigma)
          if (v >= 0) v = dphys[v];
        for (size_t j : folded_at) folded_into[j] = (int)s->iplan.size();
        s->iplan.push_back(std::move(ip));
        continue;
      }
      // contiguous chunk: the standard pass; a tile the TMA view cannot take: restore first
      if (ins.rb) return fail(QK_ESIM, "reblock: tile of pass %zu does not fit the TMA view", ii);
      if (!contiguous && !emit_restore()) return fail(QK_ESIM, "internal: layout restore failed");
    }
    if (ins.type == QK_INS_BLOCK) {
      InstrH mapped = remap(ins);
      if (relabel && !ins.gates.empty()) {
        // longest run of following SQS that still leaves >= 5 lane positions
        std::vector<int> best_d;
        size_t best_j = ii + 1;
        std::vector<int> P(nb);  // P[q]: reference position whose data lands on q
        for (int q = 0; q < nb; ++q) P[q] = q;
        // Diagonal-only blocks inside the run are folded into this pass: a
        // diagonal gate is one multiply per amplitude whichever bits it reads,
        // so it needs no chunk of its own (targets mapped back through the
        // swaps before it; bits outside this chunk add a per-chunk table term).
        std::vector<GateH> folded;
        for (size_t j = ii + 1; j < prog.size(); ++j) {
          const InstrH& nx = prog[j];
          if (nx.type == QK_INS_BLOCK && fold && !nx.gates.empty()) {
            bool diag = true;
            for (auto& g : nx.gates) {
              diag = diag && is_diag(g.kind);
              for (int t : g.t) diag = diag && t >= 0 && t < nb;
            }
            if (!diag) break;
            for (auto& g : nx.gates) {
              GateH m = g;
              for (int& t : m.t) t = P[t];
              folded.push_back(m);
            }
            best_j = j + 1;
            continue;
          }
          if (!(nx.type == QK_INS_SQS && !nx.a.empty())) break;
          std::vector<int> a = prog[j].a, b = prog[j].b;
          bool ok = true;
          for (int q : a) ok = ok && q >= 0 && q < s->L;
          for (int q : b) ok = ok && q >= 0 && q < s->L;
          if (!ok) break;
          std::sort(a.begin(), a.end());
          std::sort(b.begin(), b.end());
          std::vector<int> P2 = P;  // after this swap, q holds what P said pi(q) held
          for (size_t k = 0; k < a.size(); ++k) std::swap(P2[a[k]], P2[b[k]]);
          // source addresses of the next chunk's qubits
          std::vector<char> in_next(nb, 0);
          for (int q = 0; q < Cg; ++q) in_next[sigma[P2[q]]] = 1;
          std::vector<int> stay, incoming, rest;
          for (int a2 = 0; a2 < nb; ++a2) {
            if (in_next[a2] && a2 < Cg) stay.push_back(a2);
            else if (in_next[a2]) incoming.push_back(a2);
            else rest.push_back(a2);
          }
          // >= 5 qubits that stay in the chunk go to destination bits 0..4, so
          // every warp writes whole 512-B runs (128-B runs scattered at 64-KiB
          // strides measured slower than a separate SQS pass)
          if (stay.size() < 5) {
            if (getenv("QK_DUMP_PLAN")) fprintf(stderr, "relabel: swap run stops at instr %zu with %zu staying\n", j, stay.size());
            break;
          }
          std::vector<int> d(nb);
          int pos = 0;
          for (int x : stay) d[x] = pos++;
          for (int x : incoming) d[x] = pos++;
          for (int x : rest) d[x] = pos++;
          P = P2;
          best_d = d;
          best_j = j + 1;
        }
        // No run keeps 5 chunk qubits on the lanes (e.g. QAOA's full 12-qubit
        // chunk swaps): fuse the first swap run through a cluster exchange.
        // X = 3 incoming qubits become the cluster rank (spectators) and land
        // on destination bits 0..2, so the gathered stores are 128-B runs and
        // the next chunk is contiguous again.
        std::vector<int> xspec;
        if (best_d.empty() && folded.empty() && xfuse) {
          std::vector<int> P2(nb);
          for (int q = 0; q < nb; ++q) P2[q] = q;
          size_t j = ii + 1;
          for (; j < prog.size() && prog[j].type == QK_INS_SQS && !prog[j].a.empty(); ++j) {
            std::vector<int> a = prog[j].a, b = prog[j].b;
            bool ok = true;
            for (int q : a) ok = ok && q >= 0 && q < s->L;
            for (int q : b) ok = ok && q >= 0 && q < s->L;
            if (!ok) break;
            std::sort(a.begin(), a.end());
            std::sort(b.begin(), b.end());
            for (size_t k = 0; k < a.size(); ++k) std::swap(P2[a[k]], P2[b[k]]);
          }
          if (j > ii + 1) {
            std::vector<char> in_next(nb, 0);
            for (int q = 0; q < Cg; ++q) in_next[sigma[P2[q]]] = 1;
            std::vector<int> incoming, stay, other_in, leaving, rest;
            for (int a2 = 0; a2 < nb; ++a2) {
              if (in_next[a2] && a2 >= Cg) incoming.push_back(a2);
              else if (in_next[a2]) stay.push_back(a2);
              else if (a2 < Cg) leaving.push_back(a2);
              else rest.push_back(a2);
            }
            const int X = 3;
            if ((int)incoming.size() >= X) {
              std::vector<int> d(nb);
              int pos = 0;
              for (int k = 0; k < X; ++k) {
                xspec.push_back(incoming[k]);
                d[incoming[k]] = pos++;
              }
              for (int x : stay) d[x] = pos++;
              for (size_t k = X; k < incoming.size(); ++k) d[incoming[k]] = pos++;
              for (int x : leaving) d[x] = pos++;
              for (int x : rest) d[x] = pos++;
              P = P2;
              best_d = d;
              best_j = j;
            }
          }
        }
        if (!best_d.empty() || !folded.empty()) {
          ip.dest = best_d;
          ip.xspec = xspec;
          const size_t hp_passes = s->hp.passes.size();
          int rc;
          if (folded.empty()) {
            rc = compile_block(s->hp, mapped, s->L, nb, ip, emsg, 10, Cg);
          } else {
            // one pass over [0, Cg): the block's gates, then the folded diagonal ones
            std::vector<GateH> fm = folded;
            for (auto& g : fm)
              for (int& t : g.t) t = sigma[t];
            std::vector<const GateH*> gs;
            for (auto& g : mapped.gates) gs.push_back(&g);
            for (auto& g : fm) gs.push_back(&g);
            std::vector<int> Q;
            for (int p = 0; p < Cg; ++p) Q.push_back(p);
            ip.pass0 = (int)hp_passes;
            rc = compile_pass(s->hp, gs, Q, nb, 0, emsg, best_d.empty() ? nullptr : &best_d);
            ip.npass = (int)s->hp.passes.size() - ip.pass0;
            ip.bytes = 32.0 * std::ldexp(1.0, nb) * ip.npass;
          }
          if (rc) return fail(rc, "%s", emsg.c_str());
          // The cluster exchange moves 7/8 of every chunk over DSMEM (~20 B/clk
          // per SM), so an exchange pass costs ~1.6x a plain pass whatever its
          // gates: it beats block + separate SQS only for single-phase blocks.
          const bool x_ok = xspec.empty() || getenv("QK_XFUSE_ALL") ||
                            (ip.npass == 1 && s->hp.passes[hp_passes].nphases == 1);
          if (ip.npass == 1 && x_ok && tma_plan_ok(s->hp, (int)hp_passes, nb)) {
            if (!best_d.empty()) {  // only folded diagonal blocks: the layout stays
              std::vector<int> ns(nb);
              for (int q = 0; q < nb; ++q) ns[q] = best_d[sigma[P[q]]];
              sigma = ns;
            }
            for (size_t j = ii + 1; j < best_j; ++j) fused[j] = 1;
            ip.fused_by = -1;
            s->iplan.push_back(std::move(ip));
            const int block_idx = (int)s->iplan.size() - 1;
            for (size_t j = ii + 1; j < best_j; ++j) {
              InstrPlan fp;
              fp.type = prog[j].type;  // SQS, or a folded diagonal block (no pass)
              fp.fused_by = block_idx;
              s->iplan.push_back(std::move(fp));
            }
            ii = best_j - 1;
            continue;
          }
          // not fusable after all: recompile in place (drop the permuted pass)
          s->hp.passes.resize(hp_passes);
          ip.dest.clear();
          ip.xspec.clear();
        }
      }
      // Eager mode (swaps executed as passes, e.g. QAOA c12 in place): the
      // diagonal-only blocks up to the next other block still fold into this
      // pass, their targets mapped back through the swaps in between.
      const int w_own = block_chunk_width(ins, s->L);
      if (!relabel && !lazy && fold_eager && !ins.gates.empty() && w_own >= 9 && w_own <= 12) {
        std::vector<int> P(nb);
        for (int q = 0; q < nb; ++q) P[q] = q;
        std::vector<GateH> folded;
        std::vector<size_t> folded_at;
        for (size_t j = ii + 1; j < prog.size(); ++j) {
          const InstrH& nx = prog[j];
          if (nx.type == QK_INS_BLOCK) {
            if (nx.gates.empty()) continue;
            if (!diag_block(nx)) break;
            for (auto& g : nx.gates) {
              GateH m = g;
              for (int& t : m.t) t = P[t];
              folded.push_back(m);
            }
            folded_at.push_back(j);
            continue;
          }
          bool in_local = true;
          for (int q : nx.a) in_local = in_local && q >= 0 && q < s->L;
          for (int q : nx.b) in_local = in_local && q >= 0 && q < s->L;
          if (nx.type != QK_INS_SQS || !in_local) break;  // CSQS: stop folding there
          std::vector<int> sa = nx.a, sb = nx.b;
          std::sort(sa.begin(), sa.end());
          std::sort(sb.begin(), sb.end());
          for (size_t k = 0; k < sa.size(); ++k) std::swap(P[sa[k]], P[sb[k]]);
        }
        if (!folded.empty()) {
          std::vector<const GateH*> gs;
          for (auto& g : mapped.gates) gs.push_back(&g);
          for (auto& g : folded) gs.push_back(&g);
          std::vector<int> Q;
          for (int p = 0; p < w_own; ++p) Q.push_back(p);
          ip.pass0 = (int)s->hp.passes.size();
          int rc = compile_pass(s->hp, gs, Q, nb, 0, emsg);
          if (!rc && tma_plan_ok(s->hp, ip.pass0, nb)) {
            ip.npass = (int)s->hp.passes.size() - ip.pass0;
            ip.bytes = 32.0 * std::ldexp(1.0, nb) * ip.npass;
            for (size_t j : folded_at) folded_into[j] = (int)s->iplan.size();
            s->iplan.push_back(std::move(ip));
            continue;
          }
          s->hp.passes.resize(ip.pass0);  // too many ops: no fold
        }
      }
      int rc = compile_block(s->hp, mapped, s->L, nb, ip, emsg, 10, relabel ? Cg : 0);
      if (rc) return fail(rc, "%s", emsg.c_str());
    } else if (ins.type == QK_INS_SQS) {
      for (int q : ins.a)
        if (q < 0 || q >= s->L)
          return fail(QK_EINVAL, "swap bit %d out of range for %d local qubits", q, s->L);
      for (int q : ins.b)
        if (q < 0 || q >= s->L)
          return fail(QK_EINVAL, "swap bit %d out of range for %d local qubits", q, s->L);
      std::vector<int> a, b;
      for (int q : ins.a) a.push_back(sigma[q]);
      for (int q : ins.b) b.push_back(sigma[q]);
      // keep the sorted-pair semantics of the reference: pair sorted(A)[k] with sorted(B)[k]
      std::vector<int> sa = ins.a, sb = ins.b;
      std::sort(sa.begin(), sa.end());
      std::sort(sb.begin(), sb.end());
      a.clear();
      b.clear();
      for (size_t k = 0; k < sa.size(); ++k) {
        a.push_back(sigma[sa[k]]);
        b.push_back(sigma[sb[k]]);
      }
      if (lazy || merge_sqs) {
        // relabel only: sigma'[sa_k] = sigma[sb_k] and vice versa
        for (size_t k = 0; k < sa.size(); ++k) std::swap(sigma[sa[k]], sigma[sb[k]]);
        ip.lazy = 1;
        ip.bytes = 0;
        s->iplan.push_back(std::move(ip));
        continue;
      }
      ip.sqs = ins.a.empty() ? -1 : compile_sqs(s->hp, a, b, nb, true);
      ip.bytes = 32.0 * std::ldexp(1.0, nb) * (1.0 - std::ldexp(1.0, -(int)ins.a.size()));
    } else {
      int rc = check_csqs(s, ins.a, ins.b);
      if (rc) return rc;
      // rank bits held inside this handle become plain address bits
      const int held_rank_bits = nb - s->L;
      if (ins.rb) {
        // a barrier of the cross-block schedule: exchange on the layout as it
        // is (position q holds wire xw[q] at physical bit sigma[xw[q]]), then
        // the wires move: held pairs swap bits, incoming wires take the bits
        // of the outgoing ones
        std::vector<int> xl(nb);
        for (int q = 0; q < nb; ++q) {
          xl[q] = sigma[ins.xw[q]];
          if (xl[q] < 0) return fail(QK_ESIM, "internal: reblocked exchange on a non-local wire");
        }
        ip.a = ins.a;
        ip.b = ins.b;
        ip.csqs_s = (int)ins.a.size();
        ip.sqs = -2;
        ip.xlay = xl;
        int so = 0;
        for (int q : ins.b) so += q - s->L >= held_rank_bits;
        ip.bytes = 16.0 * std::ldexp(1.0, s->L) * s->count * (1.0 - std::ldexp(1.0, -so));
        std::vector<int> sa = ins.a, sb = ins.b;
        std::sort(sa.begin(), sa.end());
        std::sort(sb.begin(), sb.end());
        std::vector<int> ns = sigma;
        for (size_t k = 0; k < sa.size(); ++k) {
          const int wa = ins.xw[sa[k]], wb = ins.xw[sb[k]];
          ns[wb] = sigma[wa];
          ns[wa] = sb[k] < nb ? sigma[wb] : -1;
        }
        sigma = ns;
        if (getenv("QK_DUMP_PLAN")) {
          fprintf(stderr, "reblocked csqs: exchanged local positions at physical bits");
          for (int q : ins.a) fprintf(stderr, " %d", xl[q]);
          fprintf(stderr, "\n");
        }
        s->iplan.push_back(std::move(ip));
        continue;
      }
      bool local_only = true;
      for (int q : ins.b)
        if (q - s->L >= held_rank_bits) local_only = false;
      ip.a = ins.a;
      ip.b = ins.b;
      ip.csqs_s = (int)ins.a.size();
      if (local_only && lazy) {
        std::vector<int> sa = ins.a, sb = ins.b;
        std::sort(sa.begin(), sa.end());
        std::sort(sb.begin(), sb.end());
        for (size_t k = 0; k < sa.size(); ++k) std::swap(sigma[sa[k]], sigma[sb[k]]);
        ip.lazy = 1;
        ip.bytes = 0;
        s->iplan.push_back(std::move(ip));
        continue;
      }
      const bool strided_x = !getenv("QK_NO_STRIDED_XRS");
      if (!local_only && lazy && !strided_x && !lay_identity(sigma) && !emit_restore())
        return fail(QK_ESIM, "internal: layout restore failed");
      if (local_only) {
        std::vector<int> sa = ins.a, sb = ins.b;
        std::sort(sa.begin(), sa.end());
        std::sort(sb.begin(), sb.end());
        std::vector<int> a, b;
        for (size_t k = 0; k < sa.size(); ++k) {
          a.push_back(sigma[sa[k]]);
          b.push_back(sigma[sb[k]]);
        }
        ip.sqs = ins.a.empty() ? -1 : compile_sqs(s->hp, a, b, nb, true);
        ip.bytes = 32.0 * std::ldexp(1.0, nb) * (1.0 - std::ldexp(1.0, -(int)ins.a.size()));
      } else {
        ip.sqs = -2;  // cross-process exchange over the current layout (strided segments)
        ip.xlay = sigma;
        {  // algorithmic NVLink bytes sent by this shard: 16 B x 2^L x (1 - 2^-S) per partition
          int so = 0;
          for (int q : ins.b) so += q - s->L >= held_rank_bits;
          ip.bytes = 16.0 * std::ldexp(1.0, s->L) * s->count * (1.0 - std::ldexp(1.0, -so));
        }
        bool id = true;
        for (int q = 0; q < nb; ++q) id = id && sigma[q] == q;
        if (!id && !strided_x) {
          std::vector<int> d(nb);
          for (int q = 0; q < nb; ++q) d[sigma[q]] = q;
          InstrPlan rp;
          rp.type = QK_INS_BLOCK;
          rp.dest = d;
          InstrH empty;
          empty.type = QK_INS_BLOCK;
          int rc2 = compile_block(s->hp, empty, s->L, nb, rp, emsg, 10, Cg);
          if (rc2 || rp.npass != 1) return fail(QK_ESIM, "internal: layout restore pass failed");
          rp.synthetic = 1;
          s->iplan.push_back(std::move(rp));
          for (int q = 0; q < nb; ++q) sigma[q] = q;
          ip.xlay = sigma;
        }
      }
    }
    s->iplan.push_back(std::move(ip));
  }
  if (getenv("QK_DUMP_LOAD"))
    fprintf(stderr, "load: pass planning %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tloop).count());
  if (merge_sqs && !lay_identity(sigma) && !emit_restore()) return fail(QK_ESIM, "internal: swap run merge failed");
  // lazy and relabel modes: the handle keeps the end layout (readbacks map
  // through it, writers and the next run restore it); QK_RELABEL_RESTORE
  // restores it with a final permuted pass instead
  if (*reblocked) {  // sigma is indexed by wire: final position q holds wire rb_p2w[q]
    std::vector<int> ns(nb);
    for (int q = 0; q < nb; ++q) ns[q] = sigma[rb_p2w[q]];
    sigma = ns;
  }
  s->oop_sqs = relabel;
  s->lay_final = ident;
  if (lazy || (relabel && !getenv("QK_RELABEL_RESTORE"))) {
    s->lay_final = sigma;
    for (int q = 0; q < nb; ++q) sigma[q] = q;
  }
  bool is_ident = lay_identity(sigma);
  if (!is_ident) {
    std::vector<int> d(nb);
    for (int q = 0; q < nb; ++q) d[sigma[q]] = q;
    InstrPlan ip;
    ip.type = QK_INS_BLOCK;
    ip.dest = d;
    InstrH empty;
    empty.type = QK_INS_BLOCK;
    int rc = compile_block(s->hp, empty, s->L, nb, ip, emsg, 10, Cg);
    if (rc || ip.npass != 1) return fail(QK_ESIM, "internal: layout restore pass failed");
    ip.synthetic = 1;
    s->iplan.push_back(std::move(ip));
  }
  replay_perm(s);
  if (getenv("QK_DUMP_PLAN")) {
    int bi = 0;
    for (auto& ip : s->iplan) {
      if (ip.type == QK_INS_BLOCK) {
        for (int p = ip.pass0; p < ip.pass0 + ip.npass; ++p) {
          const PassDesc& pd = s->hp.passes[p];
          int cnt[16] = {0};
          for (int ph = 0; ph < pd.nphases; ++ph) {
            const PhaseDesc& D = s->hp.phases[pd.phase0 + ph];
            for (int o = D.op_begin; o < D.op_end; ++o) cnt[s->hp.ops[o].code]++;
          }
          fprintf(stderr, "block %d pass %d: C=%d M=%d phases=%d H=%d X=%d MAT=%d CX=%d SWAP=%d DIAG=%d SCALE=%d\n", bi,
                  p, pd.C, pd.M, pd.nphases, cnt[0], cnt[1], cnt[2], cnt[3], cnt[4], cnt[5], cnt[6]);
        }
        ++bi;
      } else if (ip.sqs >= 0) {
        const SqsDesc& d = s->hp.sqs[ip.sqs];
        fprintf(stderr, "swap: nv=%d w=%d nouter=%d in-tile=%d outer=%d\n", d.nv, d.w, d.nouter, d.nvp, d.nop);
      }
    }
    for (auto& t : s->hp.tables) fprintf(stderr, "table: bits=%d gates=%d\n", t.bits, t.ng);
    int nf = 0, ns = 0;
    for (auto& ip : s->iplan) {
      nf += ip.fused_by >= 0;
      ns += ip.type == QK_INS_SQS;
    }
    fprintf(stderr, "relabel=%d Cg=%d fused SQS %d of %d\n", (int)relabel, Cg, nf, ns);
  }
  if (memo_on) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    if (g_plan_memo.size() > 32) g_plan_memo.clear();
    g_plan_memo[pkey] = PlanMemo{s->hp, s->iplan, s->plan_lay0, s->lay_final, s->oop_sqs, *reblocked};
  }
  const auto tq0 = std::chrono::steady_clock::now();
  const int urc = upload_plan(s);
  if (getenv("QK_DUMP_LOAD"))
    fprintf(stderr, "load: upload_plan %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
  return urc;
}

int compile_program(qk_sim* s) {
  bool rb = false;
  const int rc = compile_program_impl(s, !getenv("QK_NO_REBLOCK"), &rb);
  if (rc == QK_OK || !rb) return rc;
  if (getenv("QK_DUMP_PLAN")) fprintf(stderr, "reblock: plan failed (%s), block order instead\n", g_err.c_str());
  return compile_program_impl(s, false, &rb);
}

int ensure_events(qk_sim* s, size_t n) {
  while (s->events.size() < n) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    s->events.push_back(e);
  }
  return QK_OK;
}

// split != 0: one part of a specialised pass (qk_jit.cpp qk_insert: the chunks
// whose split bits hold the given values), never on a fresh state
int launch_pass(qk_sim* s, int p, uint64_t first = 0, uint64_t count_override = 0, uint64_t split = 0) {
  const bool tma_pass = s->allow_tma && !first && !count_override && p < (int)s->pass_tma.size() && s->pass_tma[p] >= 0;
  // a fresh state is read only by a TMA pass (it writes every chunk) through a
  // view whose in-bounds part is the written prefix
  CUtensorMap fmap;
  const int zb = s->zbits;
  const bool from_fresh = !split && zb < s->nbits && (s->fresh ? s->cur == 0 : true) && tma_pass &&
                          !getenv("QK_NO_FRESH") &&
                          fresh_map(s, s->tma[s->pass_tma[p]], zb, s->bufs[s->cur], &fmap);
  if (split && !(tma_pass && p < (int)s->pass_jit.size() && s->pass_jit[p]))
    return fail(QK_ESIM, "internal: split launch of a pass without a specialised kernel");
  if (!from_fresh) {
    if (s->fresh && getenv("QK_DUMP_PLAN"))
      fprintf(stderr, "fresh state: pass %d (tma %d) fills the whole state first\n", p, (int)tma_pass);
    int rc = ensure_full(s);
    if (rc) return rc;
  }
  if (tma_pass) {
    TmaParams& tp = s->tma[s->pass_tma[p]];
    if (from_fresh) {
      if (!tp.lazy) tp.map = fmap;
      s->fresh = false;
      s->fresh_saved += 16.0 * (double)(s->amps - (1ull << zb));
    } else if (!tp.lazy) {
      const CUtensorMap* map = state_map(s, s->cur, tp.box_rows);
      if (!map) return fail(QK_ECUDA, "tensor map unavailable");
      tp.map = *map;
    }
    // lazy passes carry their own strided views of bufs[0] / bufs[1]
    const CUtensorMap* lazy_map =
        from_fresh ? &fmap : tp.lazy ? (s->cur ? &s->lazy_map1[s->pass_tma[p]] : &tp.map) : &tp.map;
    const bool flip = tp.permuted && !tp.lazy;
    tp.state = s->bufs[s->cur];
    tp.out = flip ? s->bufs[s->cur ^ 1] : s->bufs[s->cur];
    int rc;
    if (p < (int)s->pass_jit.size() && s->pass_jit[p]) {
      void* kern = s->pass_jit[p];
      std::vector<uint64_t>* bl = &s->jit_blob[p];
      if (from_fresh && p < (int)s->pass_var.size() && getenv("QK_TSTORE_TWIN")) {
        // (dev) run a TMA-store variant's register-store twin on bounded passes
        int cur = -1;
        for (auto& v : s->pass_var[p])
          if (v.kern == kern) cur = v.variant;
        if (cur >= 0 && (cur & 8)) {
          kern = nullptr;
          for (auto& v : s->pass_var[p])
            if (v.variant == (cur ^ 8)) {
              kern = v.kern;
              bl = &v.blob;
            }
          if (!kern) return fail(QK_ESIM, "internal: no register-store twin for a bounded pass");
        }
      }
      std::vector<uint64_t>& blob = *bl;
      // zero support: chunks with an outer bit at or above the next bound
      // hold zeros and no later pass reads them: a prefix of the chunk index
      // range (outer bits ascend), so the pass runs only the chunks below it
      uint64_t nlive = 0;
      if (from_fresh && !split && !tp.norm && !tp.xbits && !flip && !getenv("QK_NO_ZSKIP") && !jit_corder(tp) &&
          !jit_pairs(tp)) {
        int hi = tp.lazy ? 0 : tp.C - 1;
        std::vector<char> in_tile(s->nbits, 0);
        if (tp.lazy)
          for (int x = 0; x < tp.C; ++x) hi = std::max(hi, (int)tp.tbit[x]), in_tile[tp.tbit[x]] = 1;
        else
          for (int x = 0; x < tp.C; ++x) in_tile[x] = 1;
        const int zb2 = std::max(zb, hi + 1);
        if (zb2 < s->nbits) {
          int nlo = 0;
          for (int b = 0; b < zb2; ++b) nlo += !in_tile[b];
          nlive = 1ull << nlo;
          s->zmem_next = zb2;
          s->fresh_saved += 16.0 * (double)(s->amps - (1ull << zb2));  // stores skipped
        }
      }
      memcpy(blob.data(), lazy_map, 128);
      {  // the unbounded view, for the TMA-store epilogue
        const CUtensorMap* full =
            tp.lazy ? (s->cur ? &s->lazy_map1[s->pass_tma[p]] : &tp.map) : &tp.map;
        memcpy(blob.data() + blob.size() - 16, full, 128);
      }
      blob[17] = (uint64_t)(uintptr_t)tp.state;
      blob[18] = (uint64_t)(uintptr_t)tp.out;
      const uint64_t nch = split ? tp.nchunks >> (split & 3) : nlive ? nlive : tp.nchunks;
      if (split) {
        blob[19] = nch;
        blob[21] = split;
      }
      if (nlive) blob[19] = nch;
      rc = tp.xbits ? jit_launch_x(kern, blob.data(), tp.C, tp.M, tp.xbits, tp.nchunks >> tp.xbits,
                                   (CUstream_st*)s->stream)
                    : jit_launch(kern, blob.data(), tp.C, tp.M, nch, s->num_sms, (CUstream_st*)s->stream,
                                 tp.smax, jit_slice_bytes(tp), jit_pairs(tp) ? 2 : 1);
      if (split || nlive) {
        blob[19] = tp.nchunks;
        blob[21] = 0;
      }
    } else {
      TmaParams tf;
      if (from_fresh && tp.lazy) {  // the generic kernel reads its view from the params
        tf = tp;
        tf.map = fmap;
      }
      rc = launch_block_tma(from_fresh && tp.lazy ? &tf : &tp, s->num_sms, (CUstream_st*)s->stream);
    }
    if (rc) return fail(QK_ECUDA, "tma block launch failed: %s", cudaGetErrorString((cudaError_t)rc));
    if (flip) {
      s->cur ^= 1;
      s->state = s->bufs[s->cur];
    }
    // zero support: the pass's gates and in-tile permutation touch only its
    // tile bits (a permuted store of the relabeled mode may move any bit)
    s->zmem = s->zmem_next;  // what the pass left unwritten (64: it wrote every chunk)
    s->zmem_next = 64;
    if (split || flip || tp.xbits || s->zbits >= s->nbits || getenv("QK_NO_ZBOUND")) {
      s->zbits = 64;
    } else {
      int hi = tp.lazy ? 0 : tp.C - 1;
      if (tp.lazy)
        for (int x = 0; x < tp.C; ++x) hi = std::max(hi, (int)tp.tbit[x]);
      s->zbits = std::max(s->zbits, hi + 1);
    }
    return QK_OK;
  }
  s->zbits = 64;
  PassDesc h = s->hp.passes[p];
  if (count_override) h.ncta = count_override;
  int rc = launch_block_pass(s->state, &h, s->d_pass + p, s->d_phase, s->d_ops, s->d_coef, s->d_pool, first,
                             (CUstream_st*)s->stream);
  if (rc) return fail(QK_ECUDA, "block launch failed: %s", cudaGetErrorString((cudaError_t)rc));
  return QK_OK;
}

int exchange_cross(qk_sim* s, const InstrPlan& ip);

bool fused_away(const qk_sim* s, const InstrPlan& ip) {
  return ip.lazy || (ip.fused_by >= 0 && s->iplan[ip.fused_by].permuted);
}

// Multi-process CSQS plan (simulator.py:179-235 semantics, output independent
// of B). Pairs whose rank bit lies inside the shard are a local permutation;
// the others select peer shards. CSQS local bits are the top S local bits
// (checked), so the out-of-shard pairs use the top `so` local bits and every
// exchange is one contiguous segment per partition: segment y of shard x <->
// segment x of shard y. The lower shard of a pair moves the first half, the
// higher one the second half, so both NVLink directions carry equal traffic and
// every amplitude pair is swapped exactly once.
struct Seg {
  uint64_t my_off, peer, peer_off, len;
};

int csqs_plan(int n, int r, int count, int shard, const std::vector<int>& local_set,
              const std::vector<int>& rank_set, std::vector<Seg>& segs, std::vector<int>& in_a,
              std::vector<int>& in_b, std::vector<int>* group = nullptr) {
  const int L = n - r;
  const int held = __builtin_ctz((unsigned)count);
  std::vector<int> loc = local_set, rk = rank_set;
  std::sort(loc.begin(), loc.end());
  std::sort(rk.begin(), rk.end());
  std::vector<int> out_a, out_b;
  for (size_t k = 0; k < loc.size(); ++k) {
    if (rk[k] - L < held) {
      in_a.push_back(loc[k]);
      in_b.push_back(rk[k]);
    } else {
      out_a.push_back(loc[k]);
      out_b.push_back(rk[k]);
    }
  }
  const int so = (int)out_a.size();
  if (!so) return QK_OK;
  for (int k = 0; k < so; ++k)
    if (out_a[k] != L - so + k) return fail(QK_ESIM, "cross-shard local bits must be the top local bits");
  std::vector<int> sbit(so);
  for (int k = 0; k < so; ++k) sbit[k] = out_b[k] - L - held;
  const uint64_t part = 1ull << L;
  const uint64_t run = part >> so;
  int x = 0;
  for (int k = 0; k < so; ++k) x |= ((shard >> sbit[k]) & 1) << k;
  if (group)
    for (int y = 0; y < (1 << so); ++y) {  // every shard this one exchanges with (symmetric)
      if (y == x) continue;
      int peer = shard;
      for (int k = 0; k < so; ++k) peer = (peer & ~(1 << sbit[k])) | (((y >> k) & 1) << sbit[k]);
      group->push_back(peer);
    }
  for (int pi = 0; pi < count; ++pi) {
    for (int y = 0; y < (1 << so); ++y) {
      if (y == x) continue;
      int peer = shard;
      for (int k = 0; k < so; ++k) {
        peer &= ~(1 << sbit[k]);
        peer |= ((y >> k) & 1) << sbit[k];
      }
      const uint64_t my_off = pi * part + (uint64_t)y * run;
      const uint64_t peer_off = pi * part + (uint64_t)x * run;
      if (run > 1) {
        const uint64_t half = run / 2;
        const uint64_t o = shard < peer ? 0 : half;
        segs.push_back({my_off + o, (uint64_t)peer, peer_off + o, half});
      } else if (shard < peer) {
        segs.push_back({my_off, (uint64_t)peer, peer_off, 1});
      }
    }
  }
  return QK_OK;
}

// ---- exchange overlap ------------------------------------------------------

// split word of part f (cpos: chunk-index bits of the split bits, in bit order of f)
uint64_t ovl_word(const int* cpos, int k, int f, bool acc) {
  std::vector<std::pair<int, int>> pv;
  for (int b = 0; b < k; ++b) pv.push_back({cpos[b], (f >> b) & 1});
  std::sort(pv.begin(), pv.end());
  uint64_t w = (uint64_t)k;
  for (int b = 0; b < k; ++b) {
    w |= (uint64_t)pv[b].first << (2 + 6 * b);
    w |= (uint64_t)pv[b].second << (20 + b);
  }
  if (acc) w |= 1ull << 23;
  return w;
}

// Pass before a pipelined exchange: part by part, each followed by an event
// the exchange of that part waits on (comm stream).
int ovl_pre(qk_sim* s, int p, int j) {
  const InstrPlan& ip = s->iplan[j];
  for (int f = 0; f < (1 << ip.ovl_k); ++f) {
    int rc = launch_pass(s, p, 0, 0, ovl_word(ip.ovl_cp, ip.ovl_k, f, p == s->norm_pass && f > 0));
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(s->ev_part[f], s->stream));
  }
  s->ovl_live = j;
  return QK_OK;
}

// Pass after it: part f as soon as part f of the exchange is done.
int ovl_post(qk_sim* s, int p, int j) {
  const InstrPlan& ip = s->iplan[j];
  for (int f = 0; f < (1 << ip.ovl_k); ++f) {
    CUDA_TRY(cudaStreamWaitEvent(s->stream, s->ev_x[f], 0));
    int rc = launch_pass(s, p, 0, 0, ovl_word(ip.ovl_cq, ip.ovl_k, f, p == s->norm_pass && f > 0));
    if (rc) return rc;
  }
  s->ovl_live = -1;
  return QK_OK;
}

// The exchange on the comm stream, part by part: wait for that part of the
// pass before, meet the exchange group (device barrier), swap the part's
// amplitudes of every segment, meet again, release the pass after.
int exchange_overlapped(qk_sim* s, const InstrPlan& ip, size_t i) {
  std::vector<Seg> segs;
  std::vector<int> in_a, in_b, group;
  int rc = csqs_plan(s->n, s->r, s->count, s->shard, ip.a, ip.b, segs, in_a, in_b, &group);
  if (rc) return rc;
  cudaStream_t cs = s->comm;
  auto phys = [&](int q) { return ip.xlay.empty() ? q : ip.xlay[q]; };
  auto lay_of = [&](uint64_t a) {
    uint64_t b = 0;
    for (int q = 0; q < s->nbits; ++q) b |= ((a >> q) & 1ull) << phys(q);
    return b;
  };
  std::vector<unsigned long long*> rflags;
  for (int p : group) rflags.push_back(s->peer_flags[p]);
  auto meet = [&]() -> int {
    std::vector<unsigned long long> ep;
    for (int p : group) ep.push_back(++s->pair_epoch[p]);
    if (launch_peer_barrier(s->flags, rflags.data(), group.data(), ep.data(), (int)group.size(), s->shard, s->d_err,
                            (CUstream_st*)cs))
      return fail(QK_ECUDA, "peer barrier launch failed");
    return QK_OK;
  };
  for (int f = 0; f < (1 << ip.ovl_k); ++f) {
    CUDA_TRY(cudaStreamWaitEvent(cs, s->ev_part[f], 0));
    if (f == 0) CUDA_TRY(cudaEventRecord(s->events[2 * i], cs));
    rc = meet();
    if (rc) return rc;
    uint64_t fixed = 0;
    for (int b = 0; b < ip.ovl_k; ++b) fixed |= (uint64_t)((f >> b) & 1) << ip.ovl_f[b];
    for (auto& sg : segs) {
      double* peer_state = (s->cur ? s->peers1 : s->peers)[sg.peer];
      const int k = __builtin_ctzll(sg.len);
      std::vector<int> pos;
      for (int q = 0; q < k; ++q) {
        const int pq = phys(q);
        if (pq != ip.ovl_f[0] && (ip.ovl_k < 2 || pq != ip.ovl_f[1])) pos.push_back(pq);
      }
      std::sort(pos.begin(), pos.end());
      rc = launch_swap_strided(s->state + 2 * (lay_of(sg.my_off) | fixed),
                               peer_state + 2 * (lay_of(sg.peer_off) | fixed), sg.len >> ip.ovl_k, pos.data(),
                               (int)pos.size(), (CUstream_st*)cs);
      if (rc) return fail(QK_ECUDA, "peer exchange failed");
    }
    rc = meet();
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(s->ev_x[f], cs));
  }
  CUDA_TRY(cudaEventRecord(s->events[2 * i + 1], cs));
  return QK_OK;
}

// Which CSQS can be pipelined (after the kernels are known): one partition
// per shard, no in-shard pairs, in-place specialised passes on both sides,
// and QK_OVL_BITS (default 1) split bits that lie outside both tiles, outside
// the exchanged bits and among the free bits of every exchanged segment. A
// pass serves one exchange only.
void plan_overlap(qk_sim* s) {
  const size_t np = s->hp.passes.size();
  s->ovl_by_p.assign(np, -1);
  s->ovl_by_q.assign(np, -1);
  s->ovl_live = -1;
  for (auto& ip : s->iplan) ip.ovl_p = ip.ovl_q = -1;
  const int want = getenv("QK_OVL_BITS") ? atoi(getenv("QK_OVL_BITS")) : 1;
  // on by default when the peers are other GPUs (the exchange then runs over
  // NVLink while the passes use HBM); members sharing one GPU share its HBM
  // and measured slower pipelined (QFT33 R=1 on one B200: 0.85 vs 0.77 s)
  const bool on = getenv("QK_OVERLAP") ? true : s->overlap != 0;
  if (!on || getenv("QK_NO_OVERLAP") || want < 1 || want > 2 || s->nshards <= 1 || s->count != 1) return;
  // in place (lazy strided tile, or contiguous chunk without a permuted store)
  auto ok_pass = [&](int p) {
    if (p < 0 || p >= (int)np || s->pass_tma[p] < 0 || p >= (int)s->pass_jit.size() || !s->pass_jit[p]) return false;
    const TmaParams& tq = s->tma[s->pass_tma[p]];
    return !tq.xbits && (tq.lazy || !tq.permuted);
  };
  // chunk-index bit of physical bit e in pass p (-1: e is a tile bit)
  auto cidx = [&](int p, int e) {
    const TmaParams& tq = s->tma[s->pass_tma[p]];
    if (!tq.lazy) return e < tq.C ? -1 : e - tq.C;  // contiguous chunk: bits 0..C-1
    int below = 0;
    for (int k = 0; k < tq.C; ++k) {
      if (tq.tbit[k] == e) return -1;
      below += tq.tbit[k] < e;
    }
    return e - below;
  };
  for (size_t j = 0; j < s->iplan.size(); ++j) {
    InstrPlan& ip = s->iplan[j];
    if (ip.type != QK_INS_CSQS || ip.sqs != -2) continue;
    const int so = (int)ip.a.size();
    int P = -1, Q = -1;
    for (int k = (int)j - 1; k >= 0; --k) {
      const InstrPlan& q = s->iplan[k];
      if (q.type == QK_INS_BLOCK && q.npass > 0) { P = q.pass0 + q.npass - 1; break; }
      if ((q.type == QK_INS_BLOCK && q.npass == 0) || (q.type != QK_INS_BLOCK && fused_away(s, q))) continue;
      break;
    }
    for (size_t k = j + 1; k < s->iplan.size(); ++k) {
      const InstrPlan& q = s->iplan[k];
      if (q.type == QK_INS_BLOCK && q.npass > 0) { Q = q.pass0; break; }
      if ((q.type == QK_INS_BLOCK && q.npass == 0) || (q.type != QK_INS_BLOCK && fused_away(s, q))) continue;
      break;
    }
    if (getenv("QK_DUMP_PLAN")) fprintf(stderr, "overlap? csqs %zu: P=%d ok=%d Q=%d ok=%d\n", j, P, (int)ok_pass(P), Q, (int)ok_pass(Q));
    if (!ok_pass(P) || !ok_pass(Q) || P == Q || s->ovl_by_p[P] >= 0 || s->ovl_by_q[P] >= 0 || s->ovl_by_p[Q] >= 0)
      continue;
    // free reference bits of every segment: 0 .. L-so-2 (the lower/higher shard
    // halves take bit L-so-1); prefer the highest physical positions
    std::vector<int> cand;
    for (int q = 0; q + so + 1 < s->L; ++q) {
      const int e = ip.xlay.empty() ? q : ip.xlay[q];
      if (cidx(P, e) >= 0 && cidx(Q, e) >= 0 && cidx(P, e) < 64 && cidx(Q, e) < 64) cand.push_back(e);
    }
    std::sort(cand.rbegin(), cand.rend());
    if ((int)cand.size() < want) continue;
    const int k = want;
    if ((s->tma[s->pass_tma[P]].nchunks >> k) < (uint64_t)s->num_sms ||
        (s->tma[s->pass_tma[Q]].nchunks >> k) < (uint64_t)s->num_sms)
      continue;  // every part keeps a full grid (the fused-norm partial slots)
    ip.ovl_k = k;
    for (int b = 0; b < k; ++b) {
      ip.ovl_f[b] = cand[b];
      ip.ovl_cp[b] = cidx(P, cand[b]);
      ip.ovl_cq[b] = cidx(Q, cand[b]);
    }
    ip.ovl_p = P;
    ip.ovl_q = Q;
    s->ovl_by_p[P] = (int)j;
    s->ovl_by_q[Q] = (int)j;
    if (getenv("QK_DUMP_PLAN"))
      fprintf(stderr, "overlap: csqs %zu pipelined with passes %d / %d in %d parts (split bit %d)\n", j, P, Q, 1 << k,
              cand[0]);
  }
}

int run_instr(qk_sim* s, const InstrPlan& ip, bool* skipped = nullptr, size_t idx = (size_t)-1) {
  if (ip.type != QK_INS_BLOCK && fused_away(s, ip)) return QK_OK;
  // a swap of |0...0> (fresh after reset, every shard alike) is the identity:
  // bitswap(0) = 0 for SQS and CSQS (simulator.py:81-88, 179-235)
  if (ip.type != QK_INS_BLOCK && s->fresh && !getenv("QK_NO_FRESH")) {
    if (skipped) *skipped = true;
    return QK_OK;
  }
  if (ip.type != QK_INS_BLOCK) {
    int rc = ensure_full(s);  // (drops the zero support: the swap moves data)
    if (rc) return rc;
  }
  if (ip.type == QK_INS_BLOCK) {
    for (int p = ip.pass0; p < ip.pass0 + ip.npass; ++p) {
      const int jp = p < (int)s->ovl_by_p.size() ? s->ovl_by_p[p] : -1;
      const int jq = p < (int)s->ovl_by_q.size() ? s->ovl_by_q[p] : -1;
      const bool timed = p < (int)s->tuning.size() && s->tuning[p] >= 0;
      if (timed) CUDA_TRY(cudaEventRecord(s->tune_ev[2 * p], s->stream));
      int rc;
      if (jq >= 0 && s->ovl_live == jq) rc = ovl_post(s, p, jq);
      else if (jp >= 0 && !s->fresh) rc = ovl_pre(s, p, jp);  // (a fresh pre-pass runs whole)
      else rc = launch_pass(s, p);
      if (rc) return rc;
      if (timed) CUDA_TRY(cudaEventRecord(s->tune_ev[2 * p + 1], s->stream));
    }
    return QK_OK;
  }
  if (ip.sqs >= 0) {
    int rc = -2;
    if (getenv("QK_SQS_BULK") && s->nbits >= 16)  // bulk-copy variant: 512-B copies are TMA-op bound
      rc = launch_sqs_bulk(s->state, &s->hp.sqs[ip.sqs], s->num_sms, (CUstream_st*)s->stream);
    if (rc == -2 && s->bufs[1] && s->oop_sqs && !getenv("QK_SQS_INPLACE")) {
      // relabeled programs own a second buffer: permute into it and flip
      rc = launch_sqs_oop(s->state, s->bufs[s->cur ^ 1], &s->hp.sqs[ip.sqs], (CUstream_st*)s->stream);
      if (!rc) {
        s->cur ^= 1;
        s->state = s->bufs[s->cur];
      }
    }
    if (rc == -2) rc = launch_sqs(s->state, &s->hp.sqs[ip.sqs], s->d_sqs + ip.sqs, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "sqs launch failed: %s", cudaGetErrorString((cudaError_t)rc));
    return QK_OK;
  }
  if (ip.sqs == -2) {
    if (idx != (size_t)-1 && s->ovl_live == (int)idx) return exchange_overlapped(s, ip, idx);
    return exchange_cross(s, ip);
  }
  return QK_OK;
}

int exchange_cross(qk_sim* s, const InstrPlan& ip) {
  if (s->nshards <= 1 || (int)s->peers.size() < s->nshards)
    return fail(QK_ESIM, "cross-rank swap needs the peer shards' state (qk_ipc_open)");
  std::vector<Seg> segs;
  std::vector<int> in_a, in_b, group;
  int rc = csqs_plan(s->n, s->r, s->count, s->shard, ip.a, ip.b, segs, in_a, in_b, &group);
  if (rc) return rc;
  for (auto& sg : segs)
    if (!(s->cur ? s->peers1 : s->peers)[sg.peer])
      return fail(QK_ESIM, "peer shard %d not mapped (qk_ipc_open)", (int)sg.peer);
  // Device-side barrier (default): the shards of the exchange group meet on
  // flags in each other's memory, stream-ordered; the host never waits. The
  // host-callback barrier (two stream syncs + two host barriers) stays as a
  // debugging fallback (QK_HOST_BARRIER).
  bool dev_bar = !getenv("QK_HOST_BARRIER");
  std::vector<unsigned long long*> rflags;
  for (int p : group) {
    if (!s->peer_flags[p]) dev_bar = false;
    rflags.push_back(s->peer_flags[p]);
  }
  if (!dev_bar && !s->barrier) return fail(QK_ESIM, "cross-rank swap needs a barrier between the shards");
  auto meet = [&]() -> int {
    if (dev_bar) {
      std::vector<unsigned long long> ep;
      for (int p : group) ep.push_back(++s->pair_epoch[p]);
      if (launch_peer_barrier(s->flags, rflags.data(), group.data(), ep.data(), (int)group.size(), s->shard,
                              s->d_err, (CUstream_st*)s->stream))
        return fail(QK_ECUDA, "peer barrier launch failed");
      return QK_OK;
    }
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (s->barrier(s->barrier_ctx)) return fail(QK_ESIM, "barrier callback failed");
    return QK_OK;
  };
  rc = meet();
  if (rc) return rc;
  const bool ident_lay = ip.xlay.empty() || lay_identity(ip.xlay);
  auto lay_of = [&](uint64_t i) {
    if (ident_lay) return i;
    uint64_t j = 0;
    for (int q = 0; q < s->nbits; ++q) j |= ((i >> q) & 1ull) << ip.xlay[q];
    return j;
  };
  for (auto& sg : segs) {
    // every shard runs the same plan, so the peers' current buffer is bufs[cur] too
    double* peer_state = (s->cur ? s->peers1 : s->peers)[sg.peer];
    if (ident_lay) {
      rc = launch_swap_segments(s->state + 2 * sg.my_off, peer_state + 2 * sg.peer_off, sg.len,
                                (CUstream_st*)s->stream);
    } else {
      // lazy / relabeled layout: the segment's free reference bits 0..k-1 sit at
      // xlay[0..k-1]; enumerate them in physical order (coalesced runs)
      const int k = __builtin_ctzll(sg.len);
      std::vector<int> pos;
      for (int q = 0; q < k; ++q) pos.push_back(ip.xlay[q]);
      std::sort(pos.begin(), pos.end());
      rc = launch_swap_strided(s->state + 2 * lay_of(sg.my_off), peer_state + 2 * lay_of(sg.peer_off), sg.len,
                               pos.data(), (int)pos.size(), (CUstream_st*)s->stream);
    }
    if (rc) return fail(QK_ECUDA, "peer exchange failed");
  }
  rc = meet();
  if (rc) return rc;
  if (!in_a.empty()) {
    HostPlan tmp;
    if (!ident_lay) {  // in-shard pairs act on the bits' current positions
      std::vector<int> sa = in_a, sb = in_b;
      std::sort(sa.begin(), sa.end());
      std::sort(sb.begin(), sb.end());
      in_a.clear();
      in_b.clear();
      for (size_t k = 0; k < sa.size(); ++k) {
        in_a.push_back(ip.xlay[sa[k]]);
        in_b.push_back(ip.xlay[sb[k]]);
      }
      compile_sqs(tmp, in_a, in_b, s->nbits, true);
    } else {
      compile_sqs(tmp, in_a, in_b, s->nbits);
    }
    rc = launch_sqs(s->state, &tmp.sqs[0], nullptr, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "in-shard swap failed");
  }
  return QK_OK;
}

// after a synchronize: did a peer barrier time out?
int check_peer_error(qk_sim* s) {
  if (!s->d_err || s->nshards <= 1) return QK_OK;
  int e = 0;
  CUDA_TRY(cudaMemcpy(&e, s->d_err, sizeof e, cudaMemcpyDeviceToHost));
  if (e) return fail(QK_ESIM, "a peer shard did not reach the exchange barrier within 60 s");
  return QK_OK;
}

// Bring the state back to the reference layout (two SQS rounds at most).
int materialize(qk_sim* s, bool keep_fresh = false) {
  s->norm_valid = false;  // every caller is about to write the state
  if (!keep_fresh) {
    int rc = ensure_full(s);
    if (rc) return rc;
  }
  if (s->lay.empty() || lay_identity(s->lay)) return QK_OK;
  std::vector<std::pair<int, int>> rounds[2];
  restore_rounds(s->lay, rounds);
  for (auto& rd : rounds) {
    if (rd.empty()) continue;
    std::vector<int> A, B;
    for (auto& pr : rd) {
      A.push_back(pr.first);
      B.push_back(pr.second);
    }
    HostPlan tmp;
    compile_sqs(tmp, A, B, s->nbits, true);
    int rc = launch_sqs(s->state, &tmp.sqs[0], nullptr, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "layout restore failed: %s", cudaGetErrorString((cudaError_t)rc));
    for (int& v : s->lay)
      for (auto& pr : rd) {
        if (v == pr.first) { v = pr.second; break; }
        if (v == pr.second) { v = pr.first; break; }
      }
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (!lay_identity(s->lay)) return fail(QK_ESIM, "internal: layout restore did not reach the reference layout");
  return QK_OK;
}

// physical address (handle-local) of reference address i under the layout
uint64_t lay_addr(const qk_sim* s, uint64_t i) {
  if (s->lay.empty()) return i;
  uint64_t j = 0;
  for (int q = 0; q < s->nbits; ++q) j |= ((i >> q) & 1ull) << s->lay[q];
  return j;
}

int create_common(int n, int r, int b, int device, int rank_lo, int count, qk_sim** out, int second = -1) {
  if (!out) return fail(QK_EINVAL, "null output handle");
  *out = nullptr;
  if (n < 0 || r < 0 || r > n) return fail(QK_EINVAL, "need 0 <= R <= N, got R=%d, N=%d", r, n);
  if (b < 0 || b > n - r) return fail(QK_EINVAL, "need B <= N-R, got B=%d, N-R=%d", b, n - r);
  if (count < 1 || (count & (count - 1)) || rank_lo < 0 || rank_lo % count || rank_lo + count > (1 << r))
    return fail(QK_EINVAL, "bad shard [%d, %d) of %d ranks", rank_lo, rank_lo + count, 1 << r);
  const double required = std::ldexp(16.0, n);
  const int hb = __builtin_ctz((unsigned)count);
  const int nbits = n - r + hb;
  if (n > 62) return fail(QK_ENOMEM, "cannot allocate state: %.0f bytes required", required);
  CUDA_TRY(cudaSetDevice(device));
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  const size_t need = (size_t)16 << nbits;
  if (nbits > 40 || (double)need > 0.97 * (double)free_b)
    return fail(QK_ENOMEM, "cannot allocate state: %.0f bytes required", required);
  qk_sim* s = new qk_sim();
  s->n = n;
  s->r = r;
  s->b = b;
  s->device = device;
  s->rank_lo = rank_lo;
  s->count = count;
  s->L = n - r;
  s->nbits = nbits;
  s->amps = (size_t)1 << nbits;
  s->nshards = (1 << r) / count;
  s->shard = rank_lo / count;
  cudaError_t e = cudaMalloc(&s->bufs[0], need + kFlagBytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete s;
    return fail(QK_ENOMEM, "cannot allocate state: %.0f bytes required", required);
  }
  s->state = s->bufs[0];
  s->lay.resize(nbits);
  for (int q = 0; q < nbits; ++q) s->lay[q] = q;
  s->lay_final = s->lay;
  // second buffer for out-of-place fused block+SQS passes when it fits comfortably
  // (second: -1 decide here, 0 never, 1 always — a group decides for all its members)
  if (second != 0 && !getenv("QK_INPLACE") && (second == 1 || 2.0 * (double)need <= 0.90 * (double)free_b)) {
    if (cudaMalloc(&s->bufs[1], need) != cudaSuccess) {
      cudaGetLastError();
      s->bufs[1] = nullptr;
    }
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->comm, cudaStreamNonBlocking));
  for (int k = 0; k < 8; ++k) {
    CUDA_TRY(cudaEventCreateWithFlags(&s->ev_part[k], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&s->ev_x[k], cudaEventDisableTiming));
  }
  CUDA_TRY(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaMalloc(&s->d_partial, 148 * 8 * sizeof(double) + 256));
  CUDA_TRY(cudaMalloc(&s->d_nrm, 4096 * sizeof(double)));
  if (preload_exchange_kernels()) return fail(QK_ECUDA, "kernel preload failed");
  CUDA_TRY(cudaMalloc(&s->d_err, 256));
  CUDA_TRY(cudaMemsetAsync(s->d_err, 0, 256, s->stream));
  s->flags = (unsigned long long*)((char*)s->bufs[0] + need);
  CUDA_TRY(cudaMemsetAsync(s->flags, 0, kFlagBytes, s->stream));
  s->d_scalar = s->d_partial + 148 * 8;
  int rc = launch_fill_zero_one(s->state, s->amps, rank_lo == 0, (CUstream_st*)s->stream);
  if (rc) return fail(QK_ECUDA, "state init failed");
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->peers.assign(s->nshards, nullptr);
  s->peers1.assign(s->nshards, nullptr);
  s->peers[s->shard] = s->bufs[0];
  s->peers1[s->shard] = s->bufs[1];
  s->peer_flags.assign(s->nshards, nullptr);
  s->peer_flags[s->shard] = s->flags;
  s->pair_epoch.assign(s->nshards, 0);
  *out = s;
  return QK_OK;
}

// packed form of a program (qk_load_packed / qk_parse_text): per instruction
// its type; a block then has its gate count and per gate kind, #targets,
// targets, #params (params go to the double array); a swap has its size and
// both sets. Gate ids follow after a -1 sentinel and their count.
void pack_prog(const std::vector<InstrH>& prog, std::vector<int32_t>* wp, std::vector<double>* pp) {
  std::vector<int32_t>& w = *wp;
  std::vector<double>& p = *pp;
  for (auto& ins : prog) {
    w.push_back(ins.type);
    if (ins.type == QK_INS_BLOCK) {
      w.push_back((int32_t)ins.gates.size());
      for (auto& g : ins.gates) {
        w.push_back(g.kind);
        w.push_back((int32_t)g.t.size());
        for (int t : g.t) w.push_back(t);
        w.push_back((int32_t)g.p.size());
        p.insert(p.end(), g.p.begin(), g.p.end());
      }
    } else {
      w.push_back((int32_t)ins.a.size());
      w.insert(w.end(), ins.a.begin(), ins.a.end());
      w.insert(w.end(), ins.b.begin(), ins.b.end());
    }
  }
  std::vector<int32_t> ids;
  for (auto& ins : prog)
    if (ins.type == QK_INS_BLOCK)
      for (auto& g : ins.gates) ids.push_back((int32_t)g.gid);
  w.push_back(-1);
  w.push_back((int32_t)ids.size());
  w.insert(w.end(), ids.begin(), ids.end());
}

std::vector<InstrH> unpack(const int32_t* w, size_t nw, const double* p, size_t np, int* rc_out,
                           std::string& emsg) {
  std::vector<InstrH> out;
  size_t i = 0, pi = 0;
  *rc_out = QK_OK;
  auto bad = [&](const char* m) {
    emsg = m;
    *rc_out = QK_EINVAL;
    return std::vector<InstrH>();
  };
  while (i < nw) {
    InstrH ins;
    ins.type = w[i++];
    if (ins.type == -1) break;  // gate-id side channel of qk_parse_text
    if (i >= nw) return bad("truncated packed program");
    const int cnt = w[i++];
    if (ins.type == QK_INS_BLOCK) {
      for (int g = 0; g < cnt; ++g) {
        if (i + 2 > nw) return bad("truncated packed gate");
        GateH gh;
        gh.kind = w[i++];
        const int nt = w[i++];
        if (gh.kind < 0 || gh.kind > QK_D || nt < 1 || nt > 24 || i + nt + 1 > nw)
          return bad("bad packed gate");
        for (int k = 0; k < nt; ++k) gh.t.push_back(w[i++]);
        const int npar = w[i++];
        if (pi + npar > np) return bad("packed params exhausted");
        gh.p.assign(p + pi, p + pi + npar);
        pi += npar;
        if (gh.kind == QK_D && npar != (2 << nt)) return bad("D gate needs 2^k complex entries");
        ins.gates.push_back(std::move(gh));
      }
    } else if (ins.type == QK_INS_SQS || ins.type == QK_INS_CSQS) {
      if (i + 2 * (size_t)cnt > nw) return bad("truncated swap record");
      ins.a.assign(w + i, w + i + cnt);
      ins.b.assign(w + i + cnt, w + i + 2 * cnt);
      i += 2 * cnt;
    } else {
      return bad("unknown packed record");
    }
    out.push_back(std::move(ins));
  }
  return out;
}

// ---- one run of the loaded program, in three steps (a group handle
// interleaves its members' steps so that one host thread drives all GPUs)

int run_prepare(qk_sim* s, size_t* first_exec) {
  CUDA_TRY(cudaSetDevice(s->device));
  int rc = materialize(s, true);  // the plan starts from the reference layout
  if (rc) return rc;
  if (!s->plan_lay0.empty() && !lay_identity(s->plan_lay0) && !s->fresh) {
    // a run that does not start from |0...0>: move the data to the plan's
    // start layout (two SQS rounds, the inverse of a restore)
    std::vector<std::pair<int, int>> rounds[2];
    restore_rounds(s->plan_lay0, rounds);
    for (int r = 1; r >= 0; --r) {
      if (rounds[r].empty()) continue;
      std::vector<int> A, B;
      for (auto& pr : rounds[r]) {
        A.push_back(pr.first);
        B.push_back(pr.second);
      }
      HostPlan tmp;
      compile_sqs(tmp, A, B, s->nbits, true);
      int rc2 = launch_sqs(s->state, &tmp.sqs[0], nullptr, (CUstream_st*)s->stream);
      if (rc2) return fail(QK_ECUDA, "layout placement failed: %s", cudaGetErrorString((cudaError_t)rc2));
    }
  }
  s->fresh_saved = 0;
  *first_exec = s->iplan.size();  // the instruction whose pass read the fresh state
  s->skipped.assign(s->iplan.size(), 0);
  s->saved_i.assign(s->iplan.size(), 0.0);
  s->ovl_live = -1;
  // variant autotuning: passes whose structure is not tuned yet run their next
  // untimed variant (bit-identical results) between two events
  const size_t np = s->pass_var.size();
  bool any = false;
  for (size_t p = 0; p < np; ++p) any = tune_pick(s, (int)p, true) || any;
  if (any)
    while (s->tune_ev.size() < 2 * np) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      s->tune_ev.push_back(e);
    }
  return ensure_events(s, 2 * s->iplan.size() + 2);
}

int run_step(qk_sim* s, size_t i, size_t* first_exec) {
  CUDA_TRY(cudaSetDevice(s->device));
  if (!s->capturing) CUDA_TRY(cudaEventRecord(s->events[2 * i], s->stream));
  const bool was_fresh = s->fresh;
  const double saved0 = s->fresh_saved;
  bool skipped = false;
  const bool overlapped = s->iplan[i].type == QK_INS_CSQS && s->ovl_live == (int)i;
  int rc = run_instr(s, s->iplan[i], &skipped, i);
  if (rc) return rc;
  s->skipped[i] = skipped;
  s->saved_i[i] = s->fresh_saved - saved0;
  if (was_fresh && !s->fresh && s->fresh_saved > 0) *first_exec = i;
  // (an overlapped exchange brackets itself on the comm stream)
  if (!overlapped && !s->capturing) CUDA_TRY(cudaEventRecord(s->events[2 * i + 1], s->stream));
  else s->stat_overlapped += 1;
  return QK_OK;
}

// after the steps: wait, check the exchanges, adopt the end layout and add
// this run's per-class device times (ms) to cls and to the kernel stats
int run_finish(qk_sim* s, size_t first_exec, double cls[3]) {
  CUDA_TRY(cudaSetDevice(s->device));
  if (!s->fresh && s->zmem < s->nbits) {  // a run that never reached the top bits
    int rc = ensure_full(s);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  int rc = check_peer_error(s);
  if (rc) return rc;
  if (s->lay_final.size() == s->lay.size()) s->lay = s->lay_final;
  s->zbits = 64;  // a later run or writer starts from an unknown state
  s->norm_valid = s->norm_pass >= 0;
  for (size_t p = 0; p < s->tuning.size(); ++p)
    if (s->tuning[p] >= 0) {
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, s->tune_ev[2 * p], s->tune_ev[2 * p + 1]));
      tune_record(s, (int)p, ms);
      s->tuning[p] = -1;
    }
  const size_t ni = s->iplan.size();
  // a replay is timed as a whole and attributed to its instructions in the
  // proportions of the last eager run
  float g_ms = 0;
  double g_sum = 0;
  const bool replay = s->graph_timed;
  s->graph_timed = false;
  if (replay) {
    CUDA_TRY(cudaEventElapsedTime(&g_ms, s->events[0], s->events[1]));
    s->last_ms.resize(ni, 0.0);
    for (size_t i = 0; i < ni; ++i) g_sum += s->last_ms[i];
    s->stat_graph += 1;
  } else {
    s->last_ms.assign(ni, 0.0);
  }
  for (size_t i = 0; i < ni; ++i) {
    float ms = 0;
    if (replay) ms = g_sum > 0 ? (float)(g_ms * s->last_ms[i] / g_sum) : (i == 0 ? g_ms : 0.f);
    else CUDA_TRY(cudaEventElapsedTime(&ms, s->events[2 * i], s->events[2 * i + 1]));
    if (!replay) s->last_ms[i] = ms;
    const int c = s->iplan[i].type;
    if (getenv("QK_DUMP_TIMES"))
      fprintf(stderr, "instr %zu type %d pass0 %d passes %d permuted %d fused %d: %.3f ms\n", i, c, s->iplan[i].pass0, s->iplan[i].npass,
              (int)s->iplan[i].permuted, (int)fused_away(s, s->iplan[i]), ms);
    cls[c] += ms;
    const InstrPlan& ip = s->iplan[i];
    const bool xp = c == QK_INS_BLOCK && ip.npass > 0 && s->pass_tma[ip.pass0 + ip.npass - 1] >= 0 &&
                    s->tma[s->pass_tma[ip.pass0 + ip.npass - 1]].xbits > 0;
    const int sc = xp ? 3 : c;
    s->stat_ms[sc] += ms;
    if (fused_away(s, ip) || s->skipped[i]) continue;
    s->stat_bytes[sc] += ip.bytes - s->saved_i[i];
    s->stat_launch[sc] += c == QK_INS_BLOCK ? ip.npass : (ip.sqs != -1 ? 1 : 0);
  }
  return QK_OK;
}

bool is_group(const qk_sim* s) { return s && !s->members.empty(); }

// Group handle (qk_create_multi): member k holds ranks [k*cnt, (k+1)*cnt) on
// its device; members reach each other's HBM directly (peer access over
// NVLink), so a cross-member CSQS is the same exchange as between processes,
// with the device-side barrier and no host round trip. The host enqueues
// instruction i on every member before instruction i+1 on any, so a member's
// exchange barrier never waits on work that is not yet enqueued.
int group_run(qk_sim* g, double* timings) {
  const auto t0 = std::chrono::steady_clock::now();
  const size_t nm = g->members.size();
  std::vector<size_t> first(nm, 0);
  for (size_t k = 0; k < nm; ++k) {
    int rc = run_prepare(g->members[k], &first[k]);
    if (rc) return rc;
  }
  const size_t ni = g->members[0]->iplan.size();
  for (size_t i = 0; i < ni; ++i)
    for (size_t k = 0; k < nm; ++k) {
      int rc = run_step(g->members[k], i, &first[k]);
      if (rc) return rc;
    }
  double cls[3] = {0, 0, 0};
  for (size_t k = 0; k < nm; ++k) {
    double ck[3] = {0, 0, 0};
    int rc = run_finish(g->members[k], first[k], ck);
    if (rc) return rc;
    for (int c = 0; c < 3; ++c) cls[c] = std::max(cls[c], ck[c]);  // max over devices
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (timings) {
    timings[0] = cls[0] * 1e-3;
    timings[1] = cls[1] * 1e-3;
    timings[2] = cls[2] * 1e-3;
    timings[3] = wall;
  }
  return QK_OK;
}

// cross_rank_swap on a group handle: enqueue every member's exchange before
// waiting on any (each one's device barrier waits for the others)
int group_csqs(qk_sim* g, const int32_t* local_set, const int32_t* rank_set, int S) {
  std::vector<int> a(local_set, local_set + S), b(rank_set, rank_set + S);
  for (qk_sim* m : g->members) {
    CUDA_TRY(cudaSetDevice(m->device));
    int rc = materialize(m);
    if (rc) return rc;
    rc = check_csqs(m, a, b);
    if (rc) return rc;
  }
  if (S == 0) return QK_OK;
  qk_sim* m0 = g->members[0];
  const int held = m0->nbits - m0->L;
  bool local_only = true;
  for (int q : b)
    if (q - m0->L >= held) local_only = false;
  if (local_only) {
    for (qk_sim* m : g->members) {
      int rc = qk_csqs(m, local_set, rank_set, S);
      if (rc) return rc;
    }
    return QK_OK;
  }
  InstrPlan ip;
  ip.type = QK_INS_CSQS;
  ip.a = a;
  ip.b = b;
  ip.csqs_s = S;
  for (qk_sim* m : g->members) {
    CUDA_TRY(cudaSetDevice(m->device));
    int rc = exchange_cross(m, ip);
    if (rc) return rc;
  }
  for (qk_sim* m : g->members) {
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    int rc = check_peer_error(m);
    if (rc) return rc;
  }
  return QK_OK;
}

// ---- CUDA-graph replay of small runs
//
// A run of a small state is launch-bound (QFT20: two passes of ~15 us between
// host-side planning of zero-support views, tensor-map encodes and launches).
// Its launch sequence is a pure function of the loaded plan, the tuned
// variant picks and the host-side start state (fresh / zero-support bounds /
// buffer / layout), so the steps of the first run from a start state are
// captured into a graph (their host logic runs as in an eager run, the
// launches go into the graph) and later runs from the same start state replay
// it and re-apply the host state the steps left. Eligible: single-shard
// handles of at most 2^QK_GRAPH_BITS amplitudes (default 24), tuning complete,
// the same start state seen by the previous (eager) run,
// reference layout at the start, no per-launch profiling; QK_NO_GRAPH turns
// it off. Anything that fails during capture (a host sync, an unsupported
// call) restores the start state and runs eagerly.

bool tuning_pending(qk_sim* s) {
  if (getenv("QK_NO_TUNE")) return false;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  for (size_t p = 0; p < s->pass_var.size(); ++p) {
    if (s->pass_var[p].size() < 2) continue;
    auto it = g_tune.find(s->pass_key[p]);
    if (it == g_tune.end() || it->second.best < 0) return true;
  }
  return false;
}

bool graph_eligible(qk_sim* s) {
  static const int max_bits = getenv("QK_GRAPH_BITS") ? atoi(getenv("QK_GRAPH_BITS")) : 24;
  if (s->dry || s->nshards != 1 || s->per_launch || s->iplan.empty() || s->graph_fails > 2) return false;
  if (s->nbits > max_bits || getenv("QK_NO_GRAPH") || getenv("QK_DUMP_TIMES")) return false;
  if (!s->lay.empty() && !lay_identity(s->lay)) return false;  // a restore would sync
  for (auto& ip : s->iplan)
    if (ip.type == QK_INS_CSQS && ip.sqs == -2) return false;
  return !tuning_pending(s);
}

std::vector<int64_t> graph_key(const qk_sim* s) {
  std::string env;  // launch-time QK_* switches (QK_NO_FRESH, QK_SQS_INPLACE, ...)
  for (char** e = environ; e && *e; ++e)
    if (!strncmp(*e, "QK_", 3)) (env += *e) += '|';
  // the launches' kernels and their parameter blocks as built (jit_blob is
  // patched at launch from the run's state, which the key holds already)
  uint64_t kh = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { kh = (kh ^ v) * 1099511628211ull; };
  for (size_t p = 0; p < s->pass_jit.size(); ++p) {
    mix((uint64_t)(uintptr_t)s->pass_jit[p]);
    if (p < s->pass_var.size())
      for (auto& v : s->pass_var[p]) {
        mix((uint64_t)(uintptr_t)v.kern);
        for (uint64_t w : v.blob) mix(w);
      }
  }
  for (int t : s->pass_tma) mix((uint64_t)(int64_t)t);
  return {(int64_t)s->prog_gen, s->fresh, s->zbits,  s->zmem, s->zmem_next, s->cur, s->allow_tma,
          (int64_t)(uintptr_t)s->d_scratch, (int64_t)s->iplan.size(), (int64_t)std::hash<std::string>()(env),
          (int64_t)(uintptr_t)s->blob, (int64_t)(uintptr_t)s->d_pool, (int64_t)kh};
}

qk_sim::HostRunState host_state(const qk_sim* s) {
  qk_sim::HostRunState h;
  h.fresh = s->fresh;
  h.zbits = s->zbits;
  h.zmem = s->zmem;
  h.zmem_next = s->zmem_next;
  h.cur = s->cur;
  h.ovl_live = s->ovl_live;
  h.fresh_saved = s->fresh_saved;
  h.saved_i = s->saved_i;
  h.skipped = s->skipped;
  h.lay = s->lay;
  return h;
}

void set_host_state(qk_sim* s, const qk_sim::HostRunState& h) {
  s->fresh = h.fresh;
  s->zbits = h.zbits;
  s->zmem = h.zmem;
  s->zmem_next = h.zmem_next;
  s->cur = h.cur;
  s->state = s->bufs[s->cur];
  s->ovl_live = h.ovl_live;
  s->fresh_saved = h.fresh_saved;
  s->saved_i = h.saved_i;
  s->skipped = h.skipped;
  s->lay = h.lay;
}

// 1: not taken (run eagerly); otherwise the run's status
constexpr size_t kGraphs = 8;

int graph_run(qk_sim* s, double* timings) {
  if (!graph_eligible(s)) return 1;
  const auto t0 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaSetDevice(s->device));
  const std::vector<int64_t> key = graph_key(s);
  qk_sim::GraphEnt* ent = nullptr;
  for (auto& g : s->graphs)
    if (g.key == key) ent = &g;
  if (ent) {
    s->norm_valid = false;  // (run_prepare's materialize)
    set_host_state(s, ent->post);
  } else {
    // capture on the second run from a start state: a program loaded for one
    // run from one state stays eager
    if (std::find(s->gseen.begin(), s->gseen.end(), key) == s->gseen.end()) {
      s->gseen.push_back(key);
      if (s->gseen.size() > kGraphs) s->gseen.pop_front();
      return 1;
    }
    const qk_sim::HostRunState pre = host_state(s);
    const bool nv = s->norm_valid;
    size_t first_exec = 0;
    int rc = ensure_events(s, 2 * s->iplan.size() + 2);
    if (rc) return rc;
    s->capturing = true;
    cudaError_t e = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      rc = run_prepare(s, &first_exec);
      for (size_t i = 0; !rc && i < s->iplan.size(); ++i) rc = run_step(s, i, &first_exec);
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e2 = e == cudaSuccess ? cudaStreamEndCapture(s->stream, &g) : e;
    s->capturing = false;
    cudaGraphExec_t ex = nullptr;
    if (!rc && e2 == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) ex = nullptr;
    if (g) cudaGraphDestroy(g);
    if (!ex) {
      cudaGetLastError();
      set_host_state(s, pre);
      s->norm_valid = nv;
      s->graph_fails += 1;
      return 1;
    }
    if (s->graphs.size() >= kGraphs) {
      cudaGraphExecDestroy(s->graphs.front().exec);
      s->graphs.pop_front();
    }
    s->graphs.push_back({key, ex, host_state(s)});
    ent = &s->graphs.back();
    ent->post.first_exec = first_exec;
  }
  CUDA_TRY(cudaEventRecord(s->events[0], s->stream));
  CUDA_TRY(cudaGraphLaunch(ent->exec, s->stream));
  CUDA_TRY(cudaEventRecord(s->events[1], s->stream));
  s->graph_timed = true;
  double cls[3] = {0, 0, 0};
  int rc = run_finish(s, ent->post.first_exec, cls);
  if (rc) return rc;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (timings) {
    timings[0] = cls[0] * 1e-3;
    timings[1] = cls[1] * 1e-3;
    timings[2] = cls[2] * 1e-3;
    timings[3] = wall;
  }
  return QK_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

// a group handle forwards the call to every member (in member order)
#define QK_GROUP_ALL(call)                 \
  if (is_group(s)) {                       \
    for (qk_sim* m : s->members) {         \
      int rc_ = (call);                    \
      if (rc_) return rc_;                 \
    }                                      \
    return QK_OK;                          \
  }

extern "C" {

int qk_version(void) { return 1; }

int qk_jit_available(void) { return jit_available() ? 1 : 0; }
const char* qk_last_error(void) { return g_err.c_str(); }

int qk_device_count(int* count) {
  if (!count) return fail(QK_EINVAL, "null pointer");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail(QK_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  }
  return QK_OK;
}

int qk_create(int n, int r, int b, int device, qk_sim** out) {
  return create_common(n, r, b, device, 0, 1 << std::max(0, std::min(r, 30)), out);
}

int qk_create_shard(int n, int r, int b, int device, int rank_lo, int count, qk_sim** out) {
  return create_common(n, r, b, device, rank_lo, count, out);
}

int qk_create_multi(int n, int r, int b, const int* devs, int ndev, qk_sim** out) {
  if (!out) return fail(QK_EINVAL, "null output handle");
  *out = nullptr;
  if (!devs || ndev < 1 || (ndev & (ndev - 1))) return fail(QK_EINVAL, "device count %d must be a power of two", ndev);
  if (r < 0 || r > 30 || ndev > (1 << r))
    return fail(QK_EINVAL, "%d devices need at least log2(%d) rank qubits, got R=%d", ndev, ndev, r);
  if (n - r < 0 || n > 62) return fail(QK_EINVAL, "need 0 <= R <= N, got R=%d, N=%d", r, n);
  const int cnt = (1 << r) / ndev;
  const int nbits = n - r + __builtin_ctz((unsigned)cnt);
  const double need = std::ldexp(16.0, nbits);
  // second buffers for every member or for none (the plans must agree): each
  // device must hold 2 x (its members' states) within 90% of its free memory
  int second = getenv("QK_INPLACE") ? 0 : 1;
  std::map<int, int> per_dev;
  for (int k = 0; k < ndev; ++k) per_dev[devs[k]]++;
  for (auto& kv : per_dev) {
    CUDA_TRY(cudaSetDevice(kv.first));
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    if ((double)kv.second * need > 0.97 * (double)free_b)
      return fail(QK_ENOMEM, "cannot allocate state: %.0f bytes required", std::ldexp(16.0, n));
    if (2.0 * kv.second * need > 0.90 * (double)free_b) second = 0;
  }
  qk_sim* g = new qk_sim();
  g->n = n;
  g->r = r;
  g->b = b;
  g->device = devs[0];
  g->rank_lo = 0;
  g->count = 1 << r;
  g->L = n - r;
  g->nbits = n;
  g->amps = (size_t)1 << n;
  for (int k = 0; k < ndev; ++k) {
    qk_sim* m = nullptr;
    int rc = create_common(n, r, b, devs[k], k * cnt, cnt, &m, second);
    if (rc) {
      std::string msg = qk_last_error();
      for (qk_sim* x : g->members) qk_destroy(x);
      delete g;
      return fail(rc, "%s", msg.c_str());
    }
    g->members.push_back(m);
  }
  // direct peer access between the members' devices (NVLink), then every
  // member sees every other member's buffers and barrier flags
  for (int a = 0; a < ndev; ++a)
    for (int c = 0; c < ndev; ++c) {
      if (devs[a] == devs[c]) continue;
      int ok = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&ok, devs[a], devs[c]));
      if (!ok) {
        for (qk_sim* x : g->members) qk_destroy(x);
        delete g;
        return fail(QK_ECUDA, "device %d cannot access device %d (no peer path)", devs[a], devs[c]);
      }
      CUDA_TRY(cudaSetDevice(devs[a]));
      cudaError_t e = cudaDeviceEnablePeerAccess(devs[c], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        for (qk_sim* x : g->members) qk_destroy(x);
        delete g;
        return fail(QK_ECUDA, "peer access %d -> %d: %s", devs[a], devs[c], cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  const bool distinct = per_dev.size() == (size_t)ndev;
  for (qk_sim* m : g->members) m->overlap = distinct ? 1 : 0;
  for (int a = 0; a < ndev; ++a)
    for (int c = 0; c < ndev; ++c) {
      g->members[a]->peers[c] = g->members[c]->bufs[0];
      g->members[a]->peers1[c] = g->members[c]->bufs[1];
      g->members[a]->peer_flags[c] = g->members[c]->flags;
    }
  *out = g;
  return QK_OK;
}

int qk_destroy(qk_sim* s) {
  if (!s) return QK_OK;
  if (is_group(s)) {
    for (qk_sim* m : s->members) qk_destroy(m);
    delete s;
    return QK_OK;
  }
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (auto& g : s->graphs) cudaGraphExecDestroy(g.exec);
  for (auto e : s->events) cudaEventDestroy(e);
  for (auto e : s->tune_ev) cudaEventDestroy(e);
  for (auto e : s->marks)
    if (e) cudaEventDestroy(e);
  if (s->ipc_mapped) {
    for (size_t i = 0; i < s->peers.size(); ++i)
      if ((int)i != s->shard && s->peers[i]) cudaIpcCloseMemHandle(s->peers[i]);
    for (size_t i = 0; i < s->peers1.size(); ++i)
      if ((int)i != s->shard && s->peers1[i]) cudaIpcCloseMemHandle(s->peers1[i]);
  }
  if (s->d_err) cudaFree(s->d_err);
  if (s->bufs[0]) cudaFree(s->bufs[0]);
  if (s->bufs[1]) cudaFree(s->bufs[1]);
  if (s->blob) cudaFree(s->blob);
  if (s->d_pool) cudaFree(s->d_pool);
  if (s->d_partial) cudaFree(s->d_partial);
  if (s->d_nrm) cudaFree(s->d_nrm);
  if (s->d_scratch) cudaFree(s->d_scratch);
  if (s->comm) {
    cudaStreamSynchronize(s->comm);
    cudaStreamDestroy(s->comm);
  }
  for (int k = 0; k < 8; ++k) {
    if (s->ev_part[k]) cudaEventDestroy(s->ev_part[k]);
    if (s->ev_x[k]) cudaEventDestroy(s->ev_x[k]);
  }
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return QK_OK;
}

int qk_reset(qk_sim* s) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_reset(m));
  CUDA_TRY(cudaSetDevice(s->device));
  s->cur = 0;
  s->state = s->bufs[0];
  s->norm_valid = false;
  for (int q = 0; q < s->nbits; ++q) s->lay[q] = q;  // |0...0> is the same in every layout
  // only the first chunk is written; the rest is filled on demand (ensure_full)
  s->fresh = s->amps >= (2ull << kFreshBits) && !getenv("QK_NO_FRESH");
  s->zbits = s->fresh ? kFreshBits : 64;
  s->zmem = s->fresh ? kFreshBits : 64;
  int rc = launch_fill_zero_one(s->state, s->fresh ? (1ull << kFreshBits) : s->amps, s->rank_lo == 0,
                                (CUstream_st*)s->stream);
  if (rc) return fail(QK_ECUDA, "reset failed");
  return QK_OK;  // stream-ordered: every later entry point uses this stream
}

int qk_layout(const qk_sim* s, int* n, int* r, int* b, int* rank_lo, int* count) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (n) *n = s->n;
  if (r) *r = s->r;
  if (b) *b = s->b;
  if (rank_lo) *rank_lo = s->rank_lo;
  if (count) *count = s->count;
  return QK_OK;
}

int qk_load_text(qk_sim* s, const char* text, size_t len, int c, int* n_instr) {
  if (!s || (!text && len)) return fail(QK_EINVAL, "null argument");
  QK_GROUP_ALL(qk_load_text(m, text, len, c, n_instr));
  CUDA_TRY(cudaSetDevice(s->device));
  Parser ps;
  ps.n = s->n;
  ps.local = s->L;
  ps.c = c;
  std::vector<InstrH> prog;
  if (ps.run(text, len, &prog)) return fail(ps.code, "%s", ps.msg.c_str());
  s->prog = std::move(prog);
  s->gbg = false;
  int rc = compile_program(s);
  if (rc) return rc;
  if (n_instr) *n_instr = (int)s->prog.size();
  return QK_OK;
}

int qk_plan_dry(const char* text, size_t len, int n, int c, int second_buffer, const char* dump_dir, int* npass) {
  if ((!text && len) || n < 1 || n > 48) return fail(QK_EINVAL, "bad argument");
  qk_sim s;
  s.dry = true;
  // (dev: QK_DRY_R=r plans one shard of a 2^r-GPU job, one rank partition each)
  const int dr = getenv("QK_DRY_R") ? atoi(getenv("QK_DRY_R")) : 0;
  if (dr < 0 || dr >= n) return fail(QK_EINVAL, "bad QK_DRY_R");
  s.n = n;
  s.r = dr;
  s.L = n - dr;
  s.nbits = n - dr;
  s.amps = (size_t)1 << (n - dr);
  s.b = n - dr;
  static double fake[2];
  s.bufs[0] = &fake[0];  // never dereferenced: planning only tests them for presence
  s.bufs[1] = second_buffer ? &fake[1] : nullptr;
  s.state = s.bufs[0];
  if (dump_dir) s.dry_dir = dump_dir;
  Parser ps;
  ps.n = n;
  ps.local = n - dr;
  ps.c = c;
  if (ps.run(text, len, &s.prog)) return fail(ps.code, "%s", ps.msg.c_str());
  const int rc = compile_program(&s);
  if (npass) *npass = (int)s.hp.passes.size();
  s.bufs[0] = s.bufs[1] = s.state = nullptr;
  return rc;
}

int qk_load_packed(qk_sim* s, const int32_t* words, size_t nwords, const double* params, size_t nparams) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_load_packed(m, words, nwords, params, nparams));
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  std::string emsg;
  std::vector<InstrH> prog = unpack(words, nwords, params, nparams, &rc, emsg);
  if (rc) return fail(rc, "%s", emsg.c_str());
  s->prog = std::move(prog);
  s->gbg = false;
  return compile_program(s);
}

int qk_load_gate_by_gate(qk_sim* s, const int32_t* words, size_t nwords, const double* params,
                         size_t nparams) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (s->r != 0) return fail(QK_EINVAL, "gate-by-gate baseline runs on a single rank");
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  std::string emsg;
  std::vector<InstrH> prog = unpack(words, nwords, params, nparams, &rc, emsg);
  if (rc) return fail(rc, "%s", emsg.c_str());
  std::vector<InstrH> one_each;
  for (auto& ins : prog) {
    if (ins.type != QK_INS_BLOCK) return fail(QK_EINVAL, "gate-by-gate program holds gate blocks only");
    for (auto& g : ins.gates) {
      InstrH b;
      b.type = QK_INS_BLOCK;
      b.gates.push_back(g);
      one_each.push_back(std::move(b));
    }
  }
  s->prog = std::move(one_each);
  s->gbg = true;
  return compile_program(s);
}

int qk_program_info(const qk_sim* s, int* n_instr, int* n_blocks, int* n_sqs, int* n_csqs, int32_t* perm) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) return qk_program_info(s->members[0], n_instr, n_blocks, n_sqs, n_csqs, perm);
  int nb = 0, ns = 0, nc = 0;
  for (auto& i : s->prog) {
    nb += i.type == QK_INS_BLOCK;
    ns += i.type == QK_INS_SQS;
    nc += i.type == QK_INS_CSQS;
  }
  if (n_instr) *n_instr = (int)s->prog.size();
  if (n_blocks) *n_blocks = nb;
  if (n_sqs) *n_sqs = ns;
  if (n_csqs) *n_csqs = nc;
  if (perm)
    for (int i = 0; i < s->n; ++i) perm[i] = i < (int)s->final_perm.size() ? s->final_perm[i] : i;
  return QK_OK;
}

int qk_set_profiling(qk_sim* s, int per_launch) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_set_profiling(m, per_launch));
  s->per_launch = per_launch;
  return QK_OK;
}

int qk_run(qk_sim* s, double* timings) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) return group_run(s, timings);
  {
    const int g = graph_run(s, timings);
    if (g != 1) return g;
  }
  const auto t0 = std::chrono::steady_clock::now();
  size_t first_exec = 0;
  int rc = run_prepare(s, &first_exec);
  if (rc) return rc;
  for (size_t i = 0; i < s->iplan.size(); ++i) {
    rc = run_step(s, i, &first_exec);
    if (rc) return rc;
  }
  double cls[3] = {0, 0, 0};
  rc = run_finish(s, first_exec, cls);
  if (rc) return rc;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (timings) {
    timings[0] = cls[0] * 1e-3;
    timings[1] = cls[1] * 1e-3;
    timings[2] = cls[2] * 1e-3;
    timings[3] = wall;
  }
  return QK_OK;
}

int qk_kernel_stats(qk_sim* s, double* out, int reset) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) {  // every member runs the same passes: report member 0 (one device), reset all
    int rc = qk_kernel_stats(s->members[0], out, reset);
    for (size_t k = 1; !rc && reset && k < s->members.size(); ++k) rc = qk_kernel_stats(s->members[k], nullptr, 1);
    return rc;
  }
  if (out)
    for (int c = 0; c < 3; ++c) {
      out[2 * c] = s->stat_ms[c];
      out[2 * c + 1] = s->stat_launch[c];
      out[6 + c] = s->stat_bytes[c];
    }
  if (out) {
    out[9] = s->stat_ms[3];
    out[10] = s->stat_launch[3];
    out[11] = s->stat_bytes[3];
    out[12] = s->stat_overlapped;
    out[13] = s->stat_graph;
    out[14] = out[15] = 0;
  }
  if (reset) {
    for (int c = 0; c < 4; ++c) s->stat_ms[c] = s->stat_launch[c] = s->stat_bytes[c] = 0;
    s->stat_overlapped = 0;
    s->stat_graph = 0;
  }
  return QK_OK;
}

int qk_sumsq(qk_sim* s, double* sumsq) {
  if (!s || !sumsq) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {
    double acc = 0.0;
    for (qk_sim* m : s->members) {
      double v = 0.0;
      int rc = qk_sumsq(m, &v);
      if (rc) return rc;
      acc += v;
    }
    *sumsq = acc;
    return QK_OK;
  }
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  // the run's last pass already summed what it stored (any later swap only permutes)
  int rc = s->norm_valid && !getenv("QK_NO_FUSED_NORM")
               ? launch_sum_final(s->d_nrm, s->nrm_parts, s->d_scalar, (CUstream_st*)s->stream)
               : launch_sumsq(s->state, s->amps, s->d_partial, s->d_scalar, (CUstream_st*)s->stream);
  if (rc) return fail(QK_ECUDA, "norm launch failed");
  CUDA_TRY(cudaMemcpyAsync(sumsq, s->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

int qk_read_physical(qk_sim* s, int part, uint64_t off, uint64_t count, double* reim) {
  if (!s || (!reim && count)) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {
    const int cnt = s->members[0]->count;
    if (part < 0 || part >= s->count) return fail(QK_EINVAL, "read outside partition");
    return qk_read_physical(s->members[part / cnt], part % cnt, off, count, reim);
  }
  const uint64_t psize = 1ull << s->L;
  if (part < 0 || part >= s->count || off + count > psize || off > psize)
    return fail(QK_EINVAL, "read outside partition");
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  if (count && !lay_identity(s->lay)) {
    // lazy layout: gather through the bit permutation (reference index i -> lay_addr(i))
    std::vector<int> pm(s->nbits);
    for (int q = 0; q < s->nbits; ++q) pm[s->lay[q]] = q;
    const uint64_t chunk = 1u << 22;
    int rc = ensure_scratch(s, chunk * 16);
    if (rc) return rc;
    for (uint64_t b = 0; b < count; b += chunk) {
      const uint64_t m = std::min(chunk, count - b);
      rc = launch_gather_logical(s->state, pm.data(), s->nbits, part * psize + off + b, m, (double*)s->d_scratch,
                                 (CUstream_st*)s->stream);
      if (rc) return fail(QK_ECUDA, "layout gather failed");
      CUDA_TRY(cudaMemcpyAsync(reim + 2 * b, s->d_scratch, m * 16, cudaMemcpyDeviceToHost, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    return QK_OK;
  }
  if (count)
    CUDA_TRY(cudaMemcpyAsync(reim, s->state + 2 * (part * psize + off), count * 16, cudaMemcpyDeviceToHost,
                             s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

int qk_write_physical(qk_sim* s, int part, uint64_t off, uint64_t count, const double* reim) {
  if (!s || (!reim && count)) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {
    const int cnt = s->members[0]->count;
    if (part < 0 || part >= s->count) return fail(QK_EINVAL, "write outside partition");
    return qk_write_physical(s->members[part / cnt], part % cnt, off, count, reim);
  }
  const uint64_t psize = 1ull << s->L;
  if (part < 0 || part >= s->count || off + count > psize || off > psize)
    return fail(QK_EINVAL, "write outside partition");
  { int mrc = materialize(s); if (mrc) return mrc; }  // writes address the reference layout
  CUDA_TRY(cudaSetDevice(s->device));
  if (count)
    CUDA_TRY(cudaMemcpyAsync(s->state + 2 * (part * psize + off), reim, count * 16, cudaMemcpyHostToDevice,
                             s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

int qk_gather(qk_sim* s, const uint64_t* idx, uint64_t count, double* reim) {
  if (!s || (count && (!idx || !reim))) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {  // split by owning member, gather, scatter back
    std::vector<std::vector<uint64_t>> sel(s->members.size()), pos(s->members.size());
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t k = idx[i] >> s->members[0]->nbits;
      if (k >= s->members.size()) return fail(QK_EINVAL, "index %llu not held by this handle", (unsigned long long)idx[i]);
      sel[k].push_back(idx[i]);
      pos[k].push_back(i);
    }
    std::vector<double> buf;
    for (size_t k = 0; k < s->members.size(); ++k) {
      if (sel[k].empty()) continue;
      buf.resize(2 * sel[k].size());
      int rc = qk_gather(s->members[k], sel[k].data(), sel[k].size(), buf.data());
      if (rc) return rc;
      for (size_t j = 0; j < sel[k].size(); ++j) {
        reim[2 * pos[k][j]] = buf[2 * j];
        reim[2 * pos[k][j] + 1] = buf[2 * j + 1];
      }
    }
    return QK_OK;
  }
  if (!count) return QK_OK;
  const uint64_t lo = (uint64_t)s->rank_lo << s->L;
  for (uint64_t i = 0; i < count; ++i)
    if (idx[i] < lo || idx[i] - lo >= s->amps) return fail(QK_EINVAL, "index %llu not held by this handle",
                                                          (unsigned long long)idx[i]);
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  const uint64_t chunk = 1u << 22;
  int rc = ensure_scratch(s, chunk * 24);
  if (rc) return rc;
  uint64_t* d_idx = (uint64_t*)s->d_scratch;
  double* d_out = (double*)((char*)s->d_scratch + chunk * 8);
  std::vector<uint64_t> rel(std::min(count, chunk));
  for (uint64_t b = 0; b < count; b += chunk) {
    const uint64_t m = std::min(chunk, count - b);
    for (uint64_t i = 0; i < m; ++i) rel[i] = lay_addr(s, idx[b + i] - lo);
    CUDA_TRY(cudaMemcpyAsync(d_idx, rel.data(), m * 8, cudaMemcpyHostToDevice, s->stream));
    rc = launch_gather(s->state, d_idx, m, d_out, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "gather failed");
    CUDA_TRY(cudaMemcpyAsync(reim + 2 * b, d_out, m * 16, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  return QK_OK;
}

int qk_read_logical(qk_sim* s, const int32_t* perm, const uint64_t* lidx, uint64_t count, double* reim) {
  if (!s || !perm || (count && (!lidx || !reim))) return fail(QK_EINVAL, "null argument");
  std::vector<uint64_t> phys(count);
  for (uint64_t i = 0; i < count; ++i) {
    if (s->n < 64 && (lidx[i] >> s->n)) return fail(QK_EINVAL, "logical index %llu out of range",
                                                    (unsigned long long)lidx[i]);
    uint64_t p = 0;
    for (int pos = 0; pos < s->n; ++pos) p |= ((lidx[i] >> perm[pos]) & 1ull) << pos;
    phys[i] = p;
  }
  return qk_gather(s, phys.data(), count, reim);
}

int qk_overlap_product(qk_sim* s, const int32_t* perm, const double* factors, double* out) {
  if (!s || !factors || !out) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {
    double acc[2] = {0.0, 0.0};
    for (qk_sim* m : s->members) {
      double v[2];
      int rc = qk_overlap_product(m, perm, factors, v);
      if (rc) return rc;
      acc[0] += v[0];
      acc[1] += v[1];
    }
    out[0] = acc[0];
    out[1] = acc[1];
    return QK_OK;
  }
  std::vector<int> pm(s->n);
  for (int q = 0; q < s->n; ++q) pm[q] = perm ? perm[q] : q;
  {
    std::vector<int> seen(s->n, 0);
    for (int q = 0; q < s->n; ++q) {
      if (pm[q] < 0 || pm[q] >= s->n || seen[pm[q]]) return fail(QK_EINVAL, "permutation is not a bijection");
      seen[pm[q]] = 1;
    }
  }
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  // factor of memory bit p: reference bit q with lay[q] == p -> logical qubit pm[q]
  std::vector<cplx> mf(40 * 2, cplx(1.0, 0.0));
  for (int p = 0; p < 40; ++p) mf[2 * p + 1] = cplx(0.0, 0.0);
  for (int q = 0; q < s->nbits; ++q) {
    const double* f = factors + 4 * pm[q];
    const int p = s->lay.empty() ? q : s->lay[q];
    mf[2 * p] = std::conj(cplx(f[0], f[1]));
    mf[2 * p + 1] = std::conj(cplx(f[2], f[3]));
  }
  cplx cst(1.0, 0.0);
  const uint64_t base = (uint64_t)s->rank_lo << s->L;
  for (int q = s->nbits; q < s->n; ++q) {
    const double* f = factors + 4 * pm[q];
    cst *= ((base >> q) & 1) ? std::conj(cplx(f[2], f[3])) : std::conj(cplx(f[0], f[1]));
  }
  std::vector<cplx> tabs(4096);
  for (int g = 0; g < 4; ++g)
    for (int v = 0; v < 1024; ++v) {
      cplx t(1.0, 0.0);
      for (int b = 0; b < 10; ++b) t *= mf[2 * (10 * g + b) + ((v >> b) & 1)];
      tabs[1024 * g + v] = t;
    }
  int rc = ensure_scratch(s, (size_t)overlap_scratch_bytes() + 4096 * 16);
  if (rc) return rc;
  double* d_tabs = (double*)s->d_scratch;
  double* d_work = d_tabs + 2 * 4096;
  CUDA_TRY(cudaMemcpyAsync(d_tabs, tabs.data(), 4096 * 16, cudaMemcpyHostToDevice, s->stream));
  rc = launch_overlap(s->state, s->amps, d_tabs, d_work, (CUstream_st*)s->stream);
  if (rc) return fail(QK_ECUDA, "overlap launch failed");
  double res[2];
  CUDA_TRY(cudaMemcpyAsync(res, d_work + 2 * 148 * 8, 16, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  const cplx o = cst * cplx(res[0], res[1]);
  out[0] = o.real();
  out[1] = o.imag();
  return QK_OK;
}

int qk_read_logical_range(qk_sim* s, const int32_t* perm, uint64_t start, uint64_t count, double* reim) {
  if (!s || !perm || (count && !reim)) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) {
    if (s->n < 64 && (start + count > (1ull << s->n) || start > (1ull << s->n)))
      return fail(QK_EINVAL, "logical range out of bounds");
    std::vector<uint64_t> phys(count);
    for (uint64_t i = 0; i < count; ++i) {
      const uint64_t l = start + i;
      uint64_t p = 0;
      for (int q = 0; q < s->n; ++q) p |= ((l >> perm[q]) & 1ull) << q;
      phys[i] = p;
    }
    return qk_gather(s, phys.data(), count, reim);
  }
  if (s->count != (1 << s->r)) return fail(QK_EINVAL, "logical range readback needs the whole state");
  if (s->n < 64 && (start + count > (1ull << s->n) || start > (1ull << s->n)))
    return fail(QK_EINVAL, "logical range out of bounds");
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  const uint64_t chunk = 1u << 22;
  int rc = ensure_scratch(s, chunk * 16);
  if (rc) return rc;
  std::vector<int> pm(s->n);
  for (int pos = 0; pos < s->n; ++pos) pm[pos < s->nbits ? s->lay[pos] : pos] = perm[pos];
  for (uint64_t b = 0; b < count; b += chunk) {
    const uint64_t m = std::min(chunk, count - b);
    rc = launch_gather_logical(s->state, pm.data(), s->n, start + b, m, (double*)s->d_scratch,
                               (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "logical gather failed");
    CUDA_TRY(cudaMemcpyAsync(reim + 2 * b, s->d_scratch, m * 16, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  return QK_OK;
}

static int reblock_packed_impl(const int32_t* words, size_t nwords, const double* params, size_t nparams, int n,
                               int nlocal, int cap, int32_t* out_words, size_t* out_nwords, double* out_params,
                               size_t* out_nparams, int32_t* p2w, int* npass) {
  if (!words || !out_nwords || !out_nparams || !npass || n < 1 || n > 64 || nlocal < 1 || nlocal > n)
    return fail(QK_EINVAL, "bad argument");
  int rc = 0;
  std::string emsg;
  std::vector<InstrH> prog = unpack(words, nwords, params, nparams, &rc, emsg);
  if (rc) return fail(rc, "%s", emsg.c_str());
  std::vector<InstrH> out;
  std::vector<int> pw;
  if (!reblock(prog, nlocal, cap, 3, &out, &pw, n)) {
    *npass = 0;
    return QK_OK;
  }
  // a barrier (cross-shard CSQS) goes out as its outgoing and incoming wires
  for (auto& ins : out)
    if (ins.type == QK_INS_CSQS && !ins.xw.empty()) {
      std::vector<int> sa = ins.a, sb = ins.b;
      std::sort(sa.begin(), sa.end());
      std::sort(sb.begin(), sb.end());
      for (size_t k = 0; k < sa.size(); ++k) {
        ins.a[k] = ins.xw[sa[k]];
        ins.b[k] = ins.xw[sb[k]];
      }
    }
  std::vector<int32_t> w;
  std::vector<double> p;
  pack_prog(out, &w, &p);
  if (out_words) {
    if (*out_nwords < w.size() || *out_nparams < p.size()) return fail(QK_EINVAL, "buffers too small");
    memcpy(out_words, w.data(), w.size() * 4);
    if (!p.empty()) memcpy(out_params, p.data(), p.size() * 8);
    if (p2w)
      for (int q = 0; q < n; ++q) p2w[q] = pw[q];
  }
  *out_nwords = w.size();
  *out_nparams = p.size();
  int np = 0;
  for (auto& ins : out) np += ins.type == QK_INS_BLOCK;
  *npass = np;
  return QK_OK;
}

int qk_reblock_packed(const int32_t* words, size_t nwords, const double* params, size_t nparams, int n, int cap,
                      int32_t* out_words, size_t* out_nwords, double* out_params, size_t* out_nparams,
                      int32_t* p2w, int* npass) {
  return reblock_packed_impl(words, nwords, params, nparams, n, n, cap, out_words, out_nwords, out_params,
                             out_nparams, p2w, npass);
}

int qk_reblock_shard(const int32_t* words, size_t nwords, const double* params, size_t nparams, int n, int nlocal,
                     int cap, int32_t* out_words, size_t* out_nwords, double* out_params, size_t* out_nparams,
                     int32_t* p2w, int* npass) {
  return reblock_packed_impl(words, nwords, params, nparams, n, nlocal, cap, out_words, out_nwords, out_params,
                             out_nparams, p2w, npass);
}

int qk_parse_text(const char* text, size_t len, int n, int local, int c, int32_t* words, size_t* nwords,
                  double* params, size_t* nparams, int* err_line) {
  if (!nwords || !nparams || (!text && len)) return fail(QK_EINVAL, "null argument");
  Parser ps;
  ps.n = n;
  ps.local = local;
  ps.c = c;
  std::vector<InstrH> prog;
  if (ps.run(text, len, &prog)) {
    if (err_line) *err_line = ps.line_no;
    return fail(ps.code, "%s", ps.msg.c_str());
  }
  std::vector<int32_t> w;
  std::vector<double> p;
  pack_prog(prog, &w, &p);
  if (words) {
    if (*nwords < w.size() || *nparams < p.size()) return fail(QK_EINVAL, "buffers too small");
    memcpy(words, w.data(), w.size() * 4);
    if (!p.empty()) memcpy(params, p.data(), p.size() * 8);
  }
  *nwords = w.size();
  *nparams = p.size();
  return QK_OK;
}

int qk_apply_block(qk_sim* s, int part, const int32_t* words, size_t nwords, const double* params,
                   size_t nparams, int c, uint64_t row_start, uint64_t row_stop) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) {
    const int cnt = s->members[0]->count;
    if (part < 0 || part >= s->count) return fail(QK_EINVAL, "bad partition %d", part);
    return qk_apply_block(s->members[part / cnt], part % cnt, words, nwords, params, nparams, c, row_start, row_stop);
  }
  { int mrc = materialize(s); if (mrc) return mrc; }
  if (part < 0 || part >= s->count) return fail(QK_EINVAL, "bad partition %d", part);
  if (c < 1 || c > s->L) return fail(QK_EINVAL, "bad chunk width %d", c);
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  std::string emsg;
  std::vector<InstrH> prog = unpack(words, nwords, params, nparams, &rc, emsg);
  if (rc) return fail(rc, "%s", emsg.c_str());
  if (prog.size() != 1 || prog[0].type != QK_INS_BLOCK) return fail(QK_EINVAL, "expected one gate block");
  static const char* names[] = {"H", "X", "U", "CX", "CP", "SWAP", "RX", "RY", "RZ", "RZZ", "D"};
  for (auto& g : prog[0].gates)
    for (int t : g.t)
      if (t >= c) {
        std::string tg = "(";
        for (size_t k = 0; k < g.t.size(); ++k)
          tg += std::to_string(g.t[k]) + (g.t.size() == 1 ? "," : (k + 1 < g.t.size() ? ", " : ""));
        tg += ")";
        return fail(QK_ESIM, "gate %s %s does not fit width %d", names[g.kind], tg.c_str(), c);
      }
  const uint64_t rows = 1ull << (s->L - c);
  if (row_stop > rows) row_stop = rows;
  if (row_start >= row_stop) return QK_OK;
  // chunk = [0, c) of the partition, outer = [c, L): CTA index == row
  HostPlan keep = std::move(s->hp);
  std::vector<InstrPlan> keep_ip = std::move(s->iplan);
  s->hp.clear();
  s->iplan.clear();
  std::vector<int> Q;
  for (int p = 0; p < c; ++p) Q.push_back(p);
  std::vector<const GateH*> gs;
  for (auto& g : prog[0].gates) gs.push_back(&g);
  rc = compile_pass(s->hp, gs, Q, s->L, 0, emsg);
  if (rc) {
    s->hp = std::move(keep);
    s->iplan = std::move(keep_ip);
    return fail(rc, "%s", emsg.c_str());
  }
  rc = upload_plan(s);
  if (!rc && !s->hp.passes.empty()) {
    double* saved = s->state;
    s->state = s->state + 2 * ((uint64_t)part << s->L);
    s->allow_tma = false;
    rc = launch_pass(s, 0, row_start, row_stop - row_start);
    s->allow_tma = true;
    s->state = saved;
    if (!rc) {
      cudaError_t e = cudaStreamSynchronize(s->stream);
      if (e != cudaSuccess) rc = fail(QK_ECUDA, "%s", cudaGetErrorString(e));
    }
  }
  s->hp = std::move(keep);
  s->iplan = std::move(keep_ip);
  int rc2 = upload_plan(s);
  return rc ? rc : rc2;
}

int qk_apply_gate_full(qk_sim* s, const int32_t* words, size_t nwords, const double* params, size_t nparams) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_apply_gate_full(m, words, nwords, params, nparams));
  { int mrc = materialize(s); if (mrc) return mrc; }
  CUDA_TRY(cudaSetDevice(s->device));
  int rc;
  std::string emsg;
  std::vector<InstrH> prog = unpack(words, nwords, params, nparams, &rc, emsg);
  if (rc) return fail(rc, "%s", emsg.c_str());
  if (prog.size() != 1 || prog[0].type != QK_INS_BLOCK) return fail(QK_EINVAL, "expected one gate block");
  HostPlan keep = std::move(s->hp);
  std::vector<InstrPlan> keep_ip = std::move(s->iplan);
  s->hp.clear();
  s->iplan.clear();
  InstrPlan ip;
  // force the memory-level grouping by compiling gate by gate as singleton blocks
  rc = QK_OK;
  for (auto& g : prog[0].gates) {
    InstrH one;
    one.type = QK_INS_BLOCK;
    one.gates.push_back(g);
    rc = compile_block(s->hp, one, s->L, s->nbits, ip, emsg);
    if (rc) break;
  }
  if (rc) {
    s->hp = std::move(keep);
    s->iplan = std::move(keep_ip);
    return fail(rc, "%s", emsg.c_str());
  }
  rc = upload_plan(s);
  for (size_t p = 0; !rc && p < s->hp.passes.size(); ++p) rc = launch_pass(s, (int)p);
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) rc = fail(QK_ECUDA, "%s", cudaGetErrorString(e));
  }
  s->hp = std::move(keep);
  s->iplan = std::move(keep_ip);
  int rc2 = upload_plan(s);
  return rc ? rc : rc2;
}

int qk_sqs(qk_sim* s, int part, const int32_t* out_set, const int32_t* in_set, int k, int cl,
           uint64_t start, uint64_t stop) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) {
    const int cnt = s->members[0]->count;
    if (part < 0 || part >= s->count) return fail(QK_EINVAL, "bad partition %d", part);
    return qk_sqs(s->members[part / cnt], part % cnt, out_set, in_set, k, cl, start, stop);
  }
  { int mrc = materialize(s); if (mrc) return mrc; }
  if (part < 0 || part >= s->count) return fail(QK_EINVAL, "bad partition %d", part);
  std::vector<int> a(out_set, out_set + k), b(in_set, in_set + k);
  for (int q : a)
    if (q < 0 || q >= s->L) return fail(QK_EINVAL, "swap bit %d out of range for %d local qubits", q, s->L);
  for (int q : b)
    if (q < 0 || q >= s->L) return fail(QK_EINVAL, "swap bit %d out of range for %d local qubits", q, s->L);
  for (int x : a)
    for (int y : b)
      if (x == y) return fail(QK_EINVAL, "bit sets overlap");
  CUDA_TRY(cudaSetDevice(s->device));
  const uint64_t size = 1ull << s->L;
  if (stop > size) stop = size;
  double* base = s->state + 2 * ((uint64_t)part << s->L);
  if (k == 0 || start >= stop) return QK_OK;
  if (start == 0 && stop == size) {
    HostPlan tmp;
    compile_sqs(tmp, a, b, s->L);
    int rc = ensure_scratch(s, sizeof(SqsDesc));
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(s->d_scratch, &tmp.sqs[0], sizeof(SqsDesc), cudaMemcpyHostToDevice, s->stream));
    rc = launch_sqs(base, &tmp.sqs[0], (const SqsDesc*)s->d_scratch, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "sqs launch failed");
  } else {
    std::vector<int> P, Qo;
    shift_pairs(a, b, cl, s->L, P, Qo);
    std::vector<int> sa = a, sb = b;
    std::sort(sa.begin(), sa.end());
    std::sort(sb.begin(), sb.end());
    std::vector<int> sp = P, sq = Qo;
    std::sort(sp.begin(), sp.end());
    std::sort(sq.begin(), sq.end());
    int rc = launch_sqs_range(base, start, stop, sp.data(), sq.data(), (int)sp.size(), sa.data(), sb.data(), k,
                              (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "sqs range launch failed");
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

int qk_csqs(qk_sim* s, const int32_t* local_set, const int32_t* rank_set, int S) {
  if (!s) return fail(QK_EINVAL, "null handle");
  if (is_group(s)) return group_csqs(s, local_set, rank_set, S);
  { int mrc = materialize(s); if (mrc) return mrc; }
  std::vector<int> a(local_set, local_set + S), b(rank_set, rank_set + S);
  int rc = check_csqs(s, a, b);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(s->device));
  if (S == 0) return QK_OK;
  InstrPlan ip;
  ip.type = QK_INS_CSQS;
  ip.a = a;
  ip.b = b;
  ip.csqs_s = S;
  const int held = s->nbits - s->L;
  bool local_only = true;
  for (int q : b)
    if (q - s->L >= held) local_only = false;
  if (!local_only) {
    rc = exchange_cross(s, ip);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    rc = check_peer_error(s);
    if (rc) return rc;
  } else {
    HostPlan tmp;
    compile_sqs(tmp, a, b, s->nbits);
    rc = ensure_scratch(s, sizeof(SqsDesc));
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(s->d_scratch, &tmp.sqs[0], sizeof(SqsDesc), cudaMemcpyHostToDevice, s->stream));
    rc = launch_sqs(s->state, &tmp.sqs[0], (const SqsDesc*)s->d_scratch, (CUstream_st*)s->stream);
    if (rc) return fail(QK_ECUDA, "csqs launch failed");
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

int qk_csqs_plan(int n, int r, int count, int shard, const int32_t* local_set, const int32_t* rank_set, int S,
                 uint64_t* segs, size_t* nseg, int32_t* local_pairs, int* nlocal) {
  if (!nseg || !nlocal || (S && (!local_set || !rank_set))) return fail(QK_EINVAL, "null argument");
  if (r < 0 || r > n || count < 1 || (count & (count - 1)) || count > (1 << r) || shard < 0 ||
      shard >= (1 << r) / count)
    return fail(QK_EINVAL, "bad shard layout");
  std::vector<Seg> sg;
  std::vector<int> in_a, in_b;
  int rc = csqs_plan(n, r, count, shard, std::vector<int>(local_set, local_set + S),
                     std::vector<int>(rank_set, rank_set + S), sg, in_a, in_b);
  if (rc) return rc;
  if (segs) {
    if (*nseg < sg.size()) return fail(QK_EINVAL, "segment buffer too small");
    for (size_t i = 0; i < sg.size(); ++i) {
      segs[4 * i] = sg[i].my_off;
      segs[4 * i + 1] = sg[i].peer;
      segs[4 * i + 2] = sg[i].peer_off;
      segs[4 * i + 3] = sg[i].len;
    }
  }
  if (local_pairs)
    for (size_t k = 0; k < in_a.size(); ++k) {
      local_pairs[k] = in_a[k];
      local_pairs[in_a.size() + k] = in_b[k];
    }
  *nseg = sg.size();
  *nlocal = (int)in_a.size();
  return QK_OK;
}

int qk_ipc_handle(qk_sim* s, void* handle128) {
  if (!s || !handle128) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) return fail(QK_EINVAL, "a multi-device handle maps its members itself");
  CUDA_TRY(cudaSetDevice(s->device));
  { int frc = ensure_full(s); if (frc) return frc; }
  unsigned char* out = static_cast<unsigned char*>(handle128);
  memset(out, 0, 128);
  for (int b = 0; b < 2; ++b) {
    if (!s->bufs[b]) continue;
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, s->bufs[b]));
    memcpy(out + 64 * b, &h, sizeof h);
  }
  return QK_OK;
}

int qk_ipc_open(qk_sim* s, int peer, const void* handle128) {
  if (!s || !handle128) return fail(QK_EINVAL, "null argument");
  if (is_group(s)) return fail(QK_EINVAL, "a multi-device handle maps its members itself");
  if (peer < 0 || peer >= s->nshards) return fail(QK_EINVAL, "bad peer shard %d", peer);
  if (peer == s->shard) return QK_OK;
  CUDA_TRY(cudaSetDevice(s->device));
  const unsigned char* in = static_cast<const unsigned char*>(handle128);
  for (int b = 0; b < 2; ++b) {
    bool zero = true;
    for (int i = 0; i < 64; ++i) zero = zero && in[64 * b + i] == 0;
    if (zero) {
      if (b == 1 && s->bufs[1]) return fail(QK_ESIM, "peer shard %d has no second buffer", peer);
      continue;
    }
    if (b == 1 && !s->bufs[1]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, in + 64 * b, sizeof h);
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    (b ? s->peers1 : s->peers)[peer] = (double*)p;
    if (!b) s->peer_flags[peer] = (unsigned long long*)((char*)p + ((size_t)16 << s->nbits));
    s->ipc_mapped = true;
  }
  return QK_OK;
}

int qk_set_overlap(qk_sim* s, int enable) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_set_overlap(m, enable));
  s->overlap = enable ? 1 : 0;
  return QK_OK;
}

int qk_set_barrier(qk_sim* s, qk_barrier_fn fn, void* ctx) {
  if (!s) return fail(QK_EINVAL, "null handle");
  s->barrier = fn;
  s->barrier_ctx = ctx;
  return QK_OK;
}

int qk_mark(qk_sim* s, int slot) {
  if (!s || slot < 0 || slot >= 8) return fail(QK_EINVAL, "bad marker slot");
  QK_GROUP_ALL(qk_mark(m, slot));
  CUDA_TRY(cudaSetDevice(s->device));
  if (!s->marks[slot]) CUDA_TRY(cudaEventCreate(&s->marks[slot]));
  CUDA_TRY(cudaEventRecord(s->marks[slot], s->stream));
  return QK_OK;
}

int qk_mark_elapsed(qk_sim* s, int a, int b, double* ms) {
  if (is_group(s)) {  // the bracket of the slowest device
    double mx = 0.0;
    for (qk_sim* m : s->members) {
      double v = 0.0;
      int rc = qk_mark_elapsed(m, a, b, &v);
      if (rc) return rc;
      mx = std::max(mx, v);
    }
    *ms = mx;
    return QK_OK;
  }
  if (!s || !ms || a < 0 || a >= 8 || b < 0 || b >= 8 || !s->marks[a] || !s->marks[b])
    return fail(QK_EINVAL, "bad marker slots");
  CUDA_TRY(cudaEventSynchronize(s->marks[b]));
  float f = 0;
  CUDA_TRY(cudaEventElapsedTime(&f, s->marks[a], s->marks[b]));
  *ms = f;
  return QK_OK;
}

int qk_sync(qk_sim* s) {
  if (!s) return fail(QK_EINVAL, "null handle");
  QK_GROUP_ALL(qk_sync(m));
  CUDA_TRY(cudaSetDevice(s->device));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return QK_OK;
}

}  // extern "C"
