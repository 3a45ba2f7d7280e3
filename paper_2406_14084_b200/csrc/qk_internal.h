// qk_internal.h — plan structures shared by the host runtime (qk_runtime.cpp)
// and the sm_100a kernels (qk_kernels.cu).
//
// A gate block (circuit.py:166-168, executed by simulator.py:338-357) is
// compiled on the host into one or more PASSES. A pass is one HBM sweep: every
// CTA stages one 2^C-amplitude chunk (the address bits Q of the pass) in
// registers/shared memory, applies the pass's ops, and writes it back. Inside
// a pass the chunk is processed in PHASES: each thread owns 2^M amplitudes
// whose chunk-local indices differ in the M "register qubits" of the phase;
// non-diagonal gates need their target among the register qubits, diagonal
// gates (RZ, RZZ, CP, D<k>) never do — runs of them are fused into one phase
// table per run and applied as a single complex multiply per amplitude.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace qk {

// Function attributes (max dynamic shared memory, ...) are per device: a
// launcher sets them once for every device it runs on (one process may drive
// several GPUs, qk_create_multi). Returns true the first time for the
// current device.
bool first_on_device(unsigned long long* mask);

constexpr int kMaxC = 13;        // 2^13 complex128 = 128 KiB of shared memory per CTA
constexpr int kMaxM = 4;         // register qubits per thread (16 amplitudes)
constexpr int kMaxTM = 5;        // specialised passes only: 5 register qubits (32 amplitudes)
constexpr int kMaxNA = 1 << kMaxTM;
constexpr int kMaxOuter = 48;    // address bits outside the chunk
constexpr int kSqsW = 5;         // SQS tile: runs of 2^5 amplitudes (512 B)

enum OpCode : int32_t {
  OP_H = 0,      // Hadamard butterfly on register slot r0 (1/sqrt2 deferred to the pass scale)
  OP_X = 1,      // register swap on slot r0
  OP_MAT = 2,    // dense 2x2 complex matrix coef[0..7] on slot r0
  OP_CX = 3,     // controlled X: target slot r0; control = slot r1 (ctrl_reg=1) or chunk-local position ctrl
  OP_SWAP = 4,   // swap register slots r0, r1
  OP_DIAG = 5,   // multiply by tables[table + (pt | pr[j])]
  OP_SCALE = 6,  // multiply by the complex coef[0] + i coef[1]
  OP_QUAD = 7,   // diagonal phase exp(i q(x)) with q quadratic in ALL address bits x (tile and chunk
                 // bits); `table` = offset (complex entries) of its QuadLayout data in the table
                 // pool. Specialised kernels only (qk_jit.cpp): the producer warp turns the chunk
                 // bits into per-position factors, each thread multiplies a few of them.
  OP_QLITE = 8,  // OP_QUAD of a run inside the tile (no chunk bits): every factor is chunk-invariant;
                 // data = QuadLayout(C, M, 0) with thr[tid] = (E(tid), e_s(tid)) already holding
                 // the linear angles and the pass scale; pr[0] = slots with e_s != 1, pr[1] = the
                 // register amplitudes j whose pj[j] != 1, pr[2] = 1: constants only (pj[j]
                 // holds the whole factor), 2: E == 1 (specialised kernels only)
};

// Data of one OP_QUAD op (doubles, at tabs + table), for a pass with C chunk
// positions, M register slots, T = C - M thread bits and NO outer bits:
//   thr[2^T][1 + M] complex   per thread: w = scale * exp(i sum of the pairs
//                             among its set thread bits), v_s = exp(i sum over
//                             its set thread bits of beta(bit, slot s))
//   pj[2^M] complex           exp(i sum of the pairs among the slots of j)
//   phi0                      constant angle
//   at[C]                     linear angle of chunk position l
//   ao[NO]                    linear angle of chunk-index bit k
//   bto[C][NO]                pair angle (position l, chunk bit k)
//   boo[NO][NO]               pair angle (chunk bit k, chunk bit k' < k), row k
// Per chunk: b_l = exp(i (at[l] + sum_k bto[l][k] x_k)) and
// b0 = exp(i (phi0 + sum_k x_k (ao[k] + sum_{k'<k} boo[k][k'] x_k'))); a
// thread's amplitude j gets b0 w prod_{thread bits set} b_l prod_{s in j} (b_R(s) v_s) pj[j].
struct QuadLayout {
  int thr, pj, phi0, at, ao, bto, boo, total;  // offsets in doubles
};
inline QuadLayout quad_layout(int C, int M, int nouter) {
  QuadLayout q;
  const int T = C - M;
  q.thr = 0;
  q.pj = q.thr + (1 << T) * (1 + M) * 2;
  q.phi0 = q.pj + (1 << M) * 2;
  q.at = q.phi0 + 2;
  q.ao = q.at + C;
  q.bto = q.ao + nouter;
  q.boo = q.bto + C * nouter;
  q.total = q.boo + nouter * nouter;
  q.total += q.total & 1;
  return q;
}

struct OpDesc {
  int32_t code;
  int32_t r0, r1;
  int32_t ctrl;       // chunk-local control position (OP_CX with ctrl_reg == 0)
  int32_t ctrl_reg;   // 1 if the control is register slot r1
  int32_t coef;       // offset into the coefficient pool (doubles)
  int64_t table;      // offset (complex entries) into the diagonal table pool
  uint16_t tcontrib[16];  // thread bit k -> table index contribution
  uint16_t pr[kMaxNA];    // register amplitude j -> table index contribution
  int32_t nco;            // OP_DIAG over address bits outside the chunk (folded diagonal blocks):
  uint8_t co_k[8];        //   chunk-index bit co_k[i] -> table index contribution co_v[i]
  uint16_t co_v[8];
  uint32_t unit;          // OP_DIAG: register amplitudes j whose entry is exactly 1 for every
                          //   thread and chunk (e.g. CP with a register control at 0)
};

struct PhaseDesc {
  int32_t op_begin, op_end;
  int32_t tbits;          // C - M
  int32_t pad;
  uint8_t tpos[16];       // thread bit k -> chunk-local position
  uint16_t rloc[kMaxNA];  // register amplitude j -> chunk-local index
  uint64_t taddr[16];     // thread bit k -> address offset (amplitudes)
  uint64_t raddr[kMaxNA]; // register amplitude j -> address offset (amplitudes)
};

struct PassDesc {
  int32_t C, M;
  int32_t phase0, nphases;
  int32_t nouter;               // number of outer address bits
  int32_t pad;
  uint64_t ncta;                // 2^nouter (per launch, may be split)
  uint8_t opos[kMaxOuter];      // outer bit k of the CTA index -> address bit
};

// Diagonal table builder: table entry x = prod over gates of entry[sub_g(x)]
struct TableGate {
  int32_t nt;
  int32_t slot[13];       // table-index bit holding targets[j]; targets[0] = entry MSB
  int64_t entries;        // offset (complex) into the entry pool
};
struct TableDesc {
  int64_t out;            // offset (complex) of the table in the table pool
  int32_t bits;           // table has 2^bits entries
  int32_t g0, ng;         // gate range in the TableGate array
  double scale;           // folded pass scale (H normalisation, factored 2x2 gates), real part
  double scale_im;        // imaginary part
};

// SQS / single-device CSQS bit-permutation: new[i] = old[bitswap(i, A, B)]
struct SqsDesc {
  int32_t nv;                 // tile bits (first kSqsW are address bits 0..w-1)
  int32_t w;
  int32_t nouter;
  int32_t nvp;                // in-tile pairs
  int32_t nop;                // outer pairs
  int32_t ident;              // in-tile permutation is the identity
  uint8_t vpos[16];           // tile bit -> address bit (nv <= 10)
  uint8_t opos[kMaxOuter];    // outer bit -> address bit
  uint8_t va[16], vb[16];     // in-tile pairs (tile bit indices)
  uint8_t oa[kMaxOuter], ob[kMaxOuter];  // outer pairs (outer bit indices)
};

// ---- persistent TMA gate-block pass (contiguous chunks, C in [9, 12], M = 4) ----
constexpr int kTMaxPh = 12;
constexpr int kTMaxOps = 64;
constexpr int kTMaxCoef = 256;

// step of a TMA phase program. OP_H/OP_X/OP_MAT never appear as steps:
// consecutive one-qubit gates on distinct register slots are fused into one
// STEP_1Q (slot s gets kind st[s]: 0 none, 1 H butterfly, 2 X, 3 matrix coef[cf[s]]).
constexpr int STEP_1Q = 16;
struct TOp {
  int8_t code, r0, r1, creg;
  int16_t ctrl, coef;
  int32_t table;
  int8_t st[kMaxTM];
  int16_t cf[kMaxTM];
  uint16_t tcontrib[12];
  uint16_t pr[kMaxNA];
  int8_t nco;             // OpDesc::nco / co_k / co_v (specialised kernels only)
  uint8_t co_k[8];
  uint16_t co_v[8];
  uint32_t unit;          // OpDesc::unit (specialised kernels skip those multiplies)
};

struct TPhase {
  int16_t op_begin, op_end;
  uint8_t tpos[12];
  uint16_t rloc[kMaxNA];
};

struct alignas(64) TmaParams {
  CUtensorMap map;              // 2-D view {16 doubles, rows} of the state, SWIZZLE_128B
  const double* tabs;           // diagonal table pool
  double* state;                // buffer read by the TMA loads (and written when not permuted)
  double* out;                  // buffer the last phase writes (== state unless permuted)
  uint64_t nchunks;
  int32_t C, M, nphases, box_rows, ntma, ng, stages;
  int32_t direct_store;         // 1: last phase stores with STG.128, 0: TMA bulk store
  int32_t permuted;             // 1: last phase scatters to the post-SQS positions (out-of-place)
  int32_t nbits;
  int32_t xbits;                // > 0: cluster-exchange store (qk_jit.cpp), 2^xbits CTAs per cluster
  int32_t lazy;                 // 1: strided tile (tbit) loaded through `map` (N-D), stored in place
  int32_t rowbits;              // lazy: contiguous row bits of the tile view (3: 128-B, 2: 64-B rows)
  int32_t needs_jit;            // 1: ops the interpreter cannot run (outer-bit table terms)
  int32_t smax;                 // > 0: at most this many stages (leaves L1 to the diagonal tables)
  int32_t norm;                 // 1: the pass also sums |amp|^2 of what it stores (per group, to p.nrm)
  uint8_t tbit[16];             // lazy: physical address bit of every chunk-local bit (ascending)
  uint8_t xpos[4];              // source address bits of the cluster rank (spectator qubits)
  uint8_t dpos[64];             // destination bit of every source address bit (permuted)
  uint64_t ldst_t[12];          // last phase: thread bit k -> destination offset
  uint64_t ldst_r[kMaxNA];      // last phase: register amplitude j -> destination offset
  TPhase ph[kTMaxPh];
  TOp ops[kTMaxOps];
  double coef[kTMaxCoef];
};

// ---- strided tiles of the lazy in-place layout ------------------------------------
// A tile is 2^C amplitudes at physical address bits T (ascending, always
// containing bits 0..2). The TMA view: dim 0 = bits 0..2 as 16 doubles (128-B
// rows, SWIZZLE_128B), then one dim per maximal run of tile / non-tile bits
// (tile runs split into <= 8-bit dims, box = full extent; non-tile dims box 1).
// When that needs more than 5 dims, everything from the 5th dim up is one
// merged dim with box 1, and the tile bits inside it are iterated by separate
// loads (they are the top chunk-local bits, so each load fills one contiguous
// slice of the stage).
struct TileDims {
  int rank;
  int lo[5], len[5], box[5];
  int inbox;         // chunk-local bits covered by one box
  int nit;           // iterated chunk-local bits (the top ones)
};

// w = row bits: 3 (128-B rows, SWIZZLE_128B) or 2 (64-B rows, SWIZZLE_64B)
inline bool tile_dims(const uint8_t* T, int C, int nbits, TileDims* d, int w = 3) {
  if (C < 3 || C > 16 || nbits > 48 || (w != 2 && w != 3)) return false;
  for (int k = 0; k < w; ++k)
    if (T[k] != k) return false;
  bool in[64] = {false};
  for (int k = 0; k < C; ++k) in[T[k]] = true;
  int lo[64], len[64], box[64];
  bool tile[64];
  int nd = 0;
  lo[0] = 0; len[0] = w; box[0] = 2 << w; tile[0] = true; nd = 1;
  for (int p = w; p < nbits;) {
    int q = p;
    while (q < nbits && in[q] == in[p]) ++q;
    if (in[p]) {
      for (int a = p; a < q; a += 8) {
        const int l = (q - a) < 8 ? (q - a) : 8;
        lo[nd] = a; len[nd] = l; box[nd] = 1 << l; tile[nd] = true; ++nd;
      }
    } else {
      lo[nd] = p; len[nd] = q - p; box[nd] = 1; tile[nd] = false; ++nd;
    }
    p = q;
  }
  d->inbox = 0;
  if (nd <= 5) {
    d->rank = nd;
  } else {
    d->rank = 5;
    lo[4] = lo[4]; len[4] = nbits - lo[4]; box[4] = 1; tile[4] = false;
  }
  for (int j = 0; j < d->rank; ++j) {
    d->lo[j] = lo[j]; d->len[j] = len[j]; d->box[j] = box[j];
    if (tile[j]) d->inbox += len[j];
  }
  d->nit = C - d->inbox;
  return d->nit >= 0 && d->nit <= 6;
}

}  // namespace qk

// ---- kernel launchers (qk_kernels.cu), all asynchronous on `stream` ----
struct CUstream_st;
namespace qk {
int launch_block_pass(double* state, const PassDesc* h_pass, const PassDesc* d_pass,
                      const PhaseDesc* d_phases, const OpDesc* d_ops, const double* d_coef,
                      const double* d_tables, uint64_t first, CUstream_st* stream);
int launch_block_tma(const TmaParams* p, int num_sms, CUstream_st* stream);
int tma_smem_bytes(int C, int M, int* ng, int* stages, int smax = 0);
// load-time specialised passes (qk_jit.cpp)
bool jit_available();
// Per OP_DIAG op of a pass: may its table be applied in the quadratic form?
// The table's phase, restricted to the register slots, has at most pairwise
// terms (every gate touches <= 2 targets, or only one register slot), so
// f_j = f_0 * prod_{s in j} (f_s / f_0) * P_j with P_j the product of the pair
// factors pf[s][s'] = e11 e00 / (e01 e10) of the 2-slot gates: a thread then
// gathers 1 + (#slots) entries per chunk instead of 2^M.
struct QuadOp {
  bool ok = false;
  double pf[16][2] = {};   // pair (s, s') at index s * 4 + s' (s < s'), complex
  double inv2 = 1.0;       // 1 / |table scale|^2 (f_s / f_0 = f_s conj(f_0) inv2)
  // OP_QUAD / OP_QLITE: the 2^M register-amplitude constants pj of the op's
  // data (uniform over threads and chunks), so the kernel takes them as
  // parameters instead of loading them per chunk (0 entries: not known)
  int npj = 0;
  double pj[kMaxNA][2] = {};
};
// variant bits: 1 = no hoisted table, 2 = quadratic table groups
bool jit_source(const TmaParams& tp, std::string* src, std::vector<long long>* toff, std::vector<double>* coef,
                int variant = 0, const std::vector<QuadOp>* quad = nullptr);
void jit_build(const std::vector<std::string>& srcs, std::vector<void*>* handles);
int jit_launch(void* kern, const void* params, int C, int M, uint64_t nchunks, int num_sms, CUstream_st* stream,
               int smax = 0, int extra_smem = 0, int cluster = 1);
// shared-memory bytes of the table slices a specialised pass stages (qk_jit.cpp slice_plan)
int jit_slice_bytes(const TmaParams& tp);
bool jit_pairs(const TmaParams& tp);
bool jit_corder(const TmaParams& tp);  // the specialised kernel walks the table-aware chunk order  // 2-CTA cluster pairs for 128-B-row strided tiles
// cluster-exchange pass: 2^xbits CTAs per cluster, nsuper supertiles
int jit_launch_x(void* kern, const void* params, int C, int M, int xbits, uint64_t nsuper, CUstream_st* stream);
int launch_build_tables(const TableDesc* d_tables, int ntables, const TableGate* d_gates,
                        const double* d_entries, double* d_pool, CUstream_st* stream);
int launch_sqs(double* state, const SqsDesc* h, const SqsDesc* d, CUstream_st* stream);
// out of place into the second buffer (relabeled programs)
int launch_sqs_oop(const double* src, double* dst, const SqsDesc* h, CUstream_st* stream);
int launch_sqs_bulk(double* state, const SqsDesc* h, int num_sms, CUstream_st* stream);
int launch_sqs_range(double* state, uint64_t start, uint64_t stop, const int* p, const int* q,
                     int np, const int* a, const int* b, int k, CUstream_st* stream);
int launch_swap_segments(double* a, double* b, uint64_t n_amps, CUstream_st* stream);
int launch_swap_strided(double* a, double* b, uint64_t n, const int* pos, int npos, CUstream_st* stream);
int preload_exchange_kernels();  // force-load (lazy loading) every kernel an exchange step launches
// device-side barrier of the shards of one exchange (flag arrays in peer memory)
int launch_peer_barrier(unsigned long long* mine, unsigned long long* const* remote, const int* idx,
                        const unsigned long long* epochs, int n, int me, int* err, CUstream_st* stream);
// sum of n partials (fused-norm readback of the last pass)
int launch_sum_final(const double* partial, int n, double* out, CUstream_st* stream);
int launch_sumsq(const double* state, uint64_t n_amps, double* d_partial, double* d_out,
                 CUstream_st* stream);
int launch_gather(const double* state, const uint64_t* d_idx, uint64_t count, double* d_out,
                  CUstream_st* stream);
int launch_gather_logical(const double* state, const int* perm, int n, uint64_t start,
                          uint64_t count, double* d_out, CUstream_st* stream);
int launch_fill_zero_one(double* state, uint64_t n_amps, int set_first, CUstream_st* stream);
// <phi|psi> against a product state: d_tabs = 4 x 1024 conj factor tables, d_work
// overlap_scratch_bytes() bytes; the result (re, im) lands at d_work + 2*148*8
int overlap_scratch_bytes();
int launch_overlap(const double* state, uint64_t n_amps, const double* d_tabs, double* d_work,
                   CUstream_st* stream);
}  // namespace qk
