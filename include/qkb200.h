/*
 * qkb200.h — C ABI of the B200-native all-in-cache (AIC) state-vector simulator.
 *
 * Drop-in boundary for the reference simulation module
 * (/root/reference/pkg/src/quokka/simulator.py). Every entry point takes plain
 * pointers and sizes; no torch or numpy types cross this boundary. The host
 * mirror `paper_2406_14084_b200/simulator.py` binds it with ctypes; the
 * bindings a maintainer would add to the reference are in INTEGRATION.md.
 *
 * State layout: one complex128 vector (re, im interleaved, numpy layout) of
 * 2^n amplitudes per simulated job. Global index bit q = physical qubit q
 * (little endian); the top r bits select the rank partition
 * (circuit.py:157-163, simulator.py:415-419). A handle created
 * with qk_create holds all 2^r partitions on one device, contiguous; a handle
 * created with qk_create_multi splits them over several devices driven by one
 * process; a handle created with qk_create_shard holds the partitions
 * [rank_lo, rank_lo+count) of a multi-process job (one process per GPU) and
 * reaches its peers' state through CUDA IPC mappings over NVLink
 * (qk_ipc_handle / qk_ipc_open). Cross-shard CSQS synchronise on flags in
 * peer memory (device-side barrier), never through the host.
 *
 * Return value of every int function: QK_OK (0) or a negative status; the
 * thread-local message is available from qk_last_error(). The Python mirror
 * maps QK_EINVAL -> ValueError, QK_EPARSE -> ParseError, QK_ESIM/QK_ENOMEM ->
 * SimulationError with the reference's messages (simulator.py:39-40, 64-72,
 * 186-194, 315-320, 494-497, 533-535).
 */
#ifndef QKB200_H
#define QKB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QK_OK 0
#define QK_EINVAL -1   /* bad argument (ValueError in the reference)            */
#define QK_EPARSE -2   /* malformed optimized circuit (circuit.ParseError)       */
#define QK_ESIM -3     /* simulator contract violated (SimulationError)          */
#define QK_ENOMEM -4   /* state does not fit ("cannot allocate state: N bytes") */
#define QK_ECUDA -5    /* CUDA runtime / driver error                            */

/* instruction records of the packed form (qk_load_packed) */
#define QK_INS_BLOCK 0
#define QK_INS_SQS 1
#define QK_INS_CSQS 2

/* gate kinds, circuit.py:34-45 (GateKind) */
#define QK_H 0
#define QK_X 1
#define QK_U 2
#define QK_CX 3
#define QK_CP 4
#define QK_SWAP 5
#define QK_RX 6
#define QK_RY 7
#define QK_RZ 8
#define QK_RZZ 9
#define QK_D 10

typedef struct qk_sim qk_sim;

/* library / device info */
int qk_version(void);
/* 1 when NVRTC is loadable: block passes of states >= 2^20 amplitudes are then
 * specialised per structure at load time (diagonal folding, lazy layout). With
 * 0 they run on the generic interpreter; the runtime warns once on stderr. */
int qk_jit_available(void);
const char* qk_last_error(void);
int qk_device_count(int* count);

/* Simulator(layout) / init_state(layout) — simulator.py:62-74, 430-435.
 * n total qubits, r rank qubits, b exchange-buffer qubits (validated like
 * LayoutParams, circuit.py:143-155; the device exchange needs no buffer).
 * Allocates 2^n complex128 on `device` and sets |0...0>. */
int qk_create(int n, int r, int b, int device, qk_sim** out);

/* Multi-process shard: this process owns ranks [rank_lo, rank_lo + count),
 * count a power of two dividing 2^r, held contiguously on `device`. */
int qk_create_shard(int n, int r, int b, int device, int rank_lo, int count, qk_sim** out);

/* One process, several GPUs (the reference's single-process Simulator for
 * states larger than one device, simulator.py:422-447, cli.py:154-172): the
 * 2^r rank partitions are split over ndev devices (a power of two <= 2^r;
 * devs may repeat an id, which puts several members on one device). Member k
 * holds ranks [k*2^r/ndev, (k+1)*2^r/ndev) on devs[k]; the members reach each
 * other's HBM through peer access (NVLink), and a CSQS whose rank bits cross
 * members is a direct peer-memory exchange between device-side barriers. One
 * host thread drives all devices (a stream per device). Every other entry
 * point accepts the returned handle like a single-device one; qk_kernel_stats
 * reports member 0 (all members run the same passes) and qk_mark_elapsed the
 * slowest device. */
int qk_create_multi(int n, int r, int b, const int* devs, int ndev, qk_sim** out);

int qk_destroy(qk_sim* sim);

/* Simulator.reset — simulator.py:439-442. Writes |0...0>; only the first 2^13
 * amplitudes go to HBM here. The next run's passes then read and write only
 * the address prefix that can hold nonzero amplitudes (zero support); a reader
 * or writer outside a run fills whatever was never written. */
int qk_reset(qk_sim* sim);

/* Layout queries */
int qk_layout(const qk_sim* sim, int* n, int* r, int* b, int* rank_lo, int* count);

/* parse_optimized (circuit.py:347-397) of the `[kind] [targets] [id] [params]`
 * optimized text into the handle's current program. `c` is the chunk width
 * every block target must stay below (circuit.py:391-393); pass c <= 0 to
 * infer it like the Quokka CLI does (cli.py:157-164). On QK_EPARSE the message
 * carries the reference's "line N: ..." text. */
int qk_load_text(qk_sim* sim, const char* text, size_t len, int c, int* n_instr);

/* Standalone parse of the optimized text into the packed form below (no
 * device needed). Two-call protocol: with words/params NULL it only stores the
 * required sizes in *nwords / *nparams; otherwise the buffers must be at least
 * that large. n = total qubits, local = N-R, c = chunk qubits (<= 0: no chunk
 * check). On QK_EPARSE *err_line holds the 1-based line number. */
int qk_parse_text(const char* text, size_t len, int n, int local, int c, int32_t* words,
                  size_t* nwords, double* params, size_t* nparams, int* err_line);

/* Packed program (the Python mirror packs GateBlock/InMemSwap/CrossRankSwap
 * objects, circuit.py:166-193). `words`:
 *   block: QK_INS_BLOCK, ngates, then per gate: kind, nt, t_0..t_{nt-1}, nparam
 *   sqs:   QK_INS_SQS,  k, out_0..out_{k-1}, in_0..in_{k-1}
 *   csqs:  QK_INS_CSQS, k, local_0.., rank_0..
 * `params`: the gates' parameters in order (angles; D<k> as 2^k re,im pairs,
 * i.e. nparam = 2^(k+1) doubles). */
int qk_load_packed(qk_sim* sim, const int32_t* words, size_t nwords,
                   const double* params, size_t nparams);
/* run_gate_by_gate(raw) — simulator.py:557-569: load the raw circuit (packed
 * QK_INS_BLOCK records, gates in order) so that qk_run sweeps the whole state
 * once per gate: no fusion, folding or relabeling. Single rank only (r == 0). */
int qk_load_gate_by_gate(qk_sim* sim, const int32_t* words, size_t nwords,
                         const double* params, size_t nparams);

/* Cross-block pass schedule of a packed program (host only, no device): the
 * schedule qk_load_* uses in the lazy layout (qk_runtime.cpp reblock). The
 * program is rewritten on wires (wire w = start position w, followed through
 * every SQS/CSQS) and cut into passes of at most `cap` wires; out_words holds
 * one QK_INS_BLOCK record per pass (targets = wires, no swaps), p2w[q] the
 * wire at final position q (so the reference's physical bit q is wire
 * p2w[q]). *npass = 0 when the program cannot be rescheduled (a non-quadratic
 * diagonal gate, a gate wider than cap - 3 wires, cap > n). Two-call protocol
 * as qk_parse_text. This replaces no reference interface: it exposes the
 * execution order of simulator.py:529-555's blocks for the parity tests. */
int qk_reblock_packed(const int32_t* words, size_t nwords, const double* params, size_t nparams,
                      int n, int cap, int32_t* out_words, size_t* out_nwords, double* out_params,
                      size_t* out_nparams, int32_t* p2w, int* npass);
/* The same schedule for one shard of a multi-GPU job (simulator.py:179-235):
 * positions >= nlocal are rank bits held by other shards. A CSQS pairing
 * local bits with them is a barrier of the schedule; it comes out as a
 * QK_INS_CSQS record whose a / b are the outgoing / incoming wires. */
int qk_reblock_shard(const int32_t* words, size_t nwords, const double* params, size_t nparams,
                     int n, int nlocal, int cap, int32_t* out_words, size_t* out_nwords,
                     double* out_params, size_t* out_nparams, int32_t* p2w, int* npass);

/* Host-only planning (development and CPU tests; replaces no reference
 * interface): parse `text` for an n-qubit single-rank state and run the
 * planner exactly as qk_load_text would on a B200 (second_buffer: the state
 * has room for the out-of-place buffer, n <= 32 on one B200), without any
 * device. The plan summary goes to stderr; with dump_dir != NULL every pass's
 * specialised kernel source is written there (pass<p>_v<variant>.cu) for
 * offline NVRTC/nvcc builds. *npass = passes planned. */
int qk_plan_dry(const char* text, size_t len, int n, int c, int second_buffer, const char* dump_dir,
                int* npass);

/* Program queries: number of instructions, and the final physical->logical
 * permutation replayed from the swaps (circuit.py:202-210); perm has n ints. */
int qk_program_info(const qk_sim* sim, int* n_instr, int* n_blocks, int* n_sqs,
                    int* n_csqs, int32_t* perm);

/* Simulator.run — simulator.py:529-555. Executes the loaded program against
 * the current state. timings[0..3] = gate, ims, xrs, wall seconds (device
 * event time per instruction class; wall = host time of the whole call).
 * The state is not reset (simulator.py:531). A single-shard handle of at
 * most 2^24 amplitudes (QK_GRAPH_BITS) replays the launches of a run from the
 * same start state (after qk_reset, say) from a CUDA graph captured on the
 * second tuned run from that state (a program loaded for one run stays eager); the class times of a replay are its event time split in the
 * proportions of the last eager run. QK_NO_GRAPH runs every launch eagerly. */
int qk_run(qk_sim* sim, double* timings);

/* Per-kernel-class device time (ms) and launch count since the last reset of
 * the counters: out[0..5] = block_ms, block_launches, sqs_ms, sqs_launches,
 * xrs_ms, xrs_launches. Also algorithmic bytes: out[6] block bytes, out[7]
 * sqs bytes, out[8] xrs bytes. out[9..11] = ms, launches and
 * bytes of the cluster-exchange block passes (block + full chunk swap in one
 * pass), which out[0..1] and out[6] exclude. out[12] = cross-shard exchanges
 * that ran overlapped with their neighbour passes (comm stream; xrs_ms is then
 * the exchange's own span). out[13] = runs replayed from a captured CUDA
 * graph (small single-shard states; qk_run). out must hold 16 doubles. */
int qk_kernel_stats(qk_sim* sim, double* out, int reset);

/* Enable per-launch event timing (1) or per-instruction-class timing only (0). */
int qk_set_profiling(qk_sim* sim, int per_launch);

/* SimResult.norm — simulator.py:393-397 (this handle's partitions only; the
 * multi-process mirror sums squares across ranks). sumsq = sum |a|^2. Right
 * after qk_run it adds the partial sums the program's last pass produced while
 * storing; after any write it reads the whole state. */
int qk_sumsq(qk_sim* sim, double* sumsq);

/* Physical amplitudes of partition `part` (0-based within the handle),
 * offsets in amplitudes; reim holds 2*count doubles. */
int qk_read_physical(qk_sim* sim, int part, uint64_t off, uint64_t count, double* reim);
int qk_write_physical(qk_sim* sim, int part, uint64_t off, uint64_t count, const double* reim);

/* Gather of arbitrary global physical indices (must be owned by the handle). */
int qk_gather(qk_sim* sim, const uint64_t* idx, uint64_t count, double* reim);

/* get_amplitude / logical_state — simulator.py:410-419, oracle.py:149-160:
 * logical index -> physical via perm (pos -> logical qubit), then gather. */
int qk_read_logical(qk_sim* sim, const int32_t* perm, const uint64_t* logical_idx,
                    uint64_t count, double* reim);

/* Logical readback of a contiguous logical range [start, start+count) of a
 * handle holding the whole state (device-side index remap + gather). */
int qk_read_logical_range(qk_sim* sim, const int32_t* perm, uint64_t start, uint64_t count,
                          double* reim);

/* <phi|psi> of this handle's amplitudes with the product state
 * phi = (x)_q (f_q[0] |0> + f_q[1] |1>) over LOGICAL qubits q: factors holds 4n
 * doubles, (f_q[0].re, f_q[0].im, f_q[1].re, f_q[1].im) per logical qubit; perm
 * is the final permutation (pos -> logical qubit, circuit.py:202-210; NULL =
 * identity). Every analytic answer the reference's own tests pin is a product
 * state (QFT|0> and H layers uniform, BV a basis state, test_oracle.py:32-42;
 * U/RZZ layers), so this gives the normalised fidelity
 * |<phi|psi>|^2 / (<phi|phi> <psi|psi>) at sizes the CPU reference cannot run
 * (SURVEY.md §8(c)). One HBM read of the state. out = (re, im). A shard
 * returns its part of the sum (the mirror adds the shards). */
int qk_overlap_product(qk_sim* sim, const int32_t* perm, const double* factors, double* out);

/* Kernel-level entry points (unit parity with the reference functions). */
/* apply_gate_block(partition, block, c, cl, row_start, row_stop) — simulator.py:338-357;
 * block given in packed form (one QK_INS_BLOCK record). rows of 2^c. */
int qk_apply_block(qk_sim* sim, int part, const int32_t* words, size_t nwords,
                   const double* params, size_t nparams, int c,
                   uint64_t row_start, uint64_t row_stop);
/* in_memory_swap(amps, out_set, in_set, cl, start, stop) — simulator.py:159-176:
 * new[i] = old[bitswap(i, out, in)] on partition `part` (bit-exact). start/stop
 * restrict the pair walk to thread indices t in [start, stop) of the
 * reference's bitshift iteration order (cl bits). */
int qk_sqs(qk_sim* sim, int part, const int32_t* out_set, const int32_t* in_set, int k,
           int cl, uint64_t start, uint64_t stop);
/* cross_rank_swap(partitions, local_set, rank_set, layout) — simulator.py:179-235. */
int qk_csqs(qk_sim* sim, const int32_t* local_set, const int32_t* rank_set, int s);
/* apply_gate_full — memory-level single gate on every partition, simulator.py:360-376. */
int qk_apply_gate_full(qk_sim* sim, const int32_t* words, size_t nwords,
                       const double* params, size_t nparams);

/* Multi-process CSQS over NVLink: export this shard's state allocation as a
 * CUDA IPC handle (64 bytes), open the peers' handles, and register a host
 * barrier callback the runtime calls around every cross-rank swap. */
int qk_ipc_handle(qk_sim* sim, void* handle64);
/* Host-only plan of the cross-shard part of a CSQS for shard `shard` of a job
 * with 2^r ranks held `count` per shard (no device needed; used by the
 * exchange and by the multi-process CPU tests). Two-call protocol on *nseg:
 * segs receives 4 uint64 per segment (my offset, peer shard, peer offset,
 * length, in amplitudes of the shard vector); local_pairs receives the
 * in-shard pairs (a_0..a_{m-1}, b_0..b_{m-1}), *nlocal = m. */
int qk_csqs_plan(int n, int r, int count, int shard, const int32_t* local_set,
                 const int32_t* rank_set, int s, uint64_t* segs, size_t* nseg,
                 int32_t* local_pairs, int* nlocal);
int qk_ipc_open(qk_sim* sim, int peer_shard, const void* handle64);
/* Pipeline every cross-shard CSQS with its neighbour passes (1) or not (0):
 * the pass before, the exchange (on a second stream) and the pass after run
 * in parts split on a bit outside both tiles, so the NVLink transfer of one
 * part overlaps the HBM passes of the others. Applies to programs loaded
 * afterwards. Default: on for a qk_create_multi handle whose devices are all
 * distinct, off otherwise (the multi-process mirror enables it when every
 * shard has its own GPU). QK_OVERLAP=1 / QK_NO_OVERLAP=1 override. */
int qk_set_overlap(qk_sim* sim, int enable);
typedef int (*qk_barrier_fn)(void* ctx);
int qk_set_barrier(qk_sim* sim, qk_barrier_fn fn, void* ctx);

/* Device-side markers on the handle's stream (CUDA events, slots 0..7), for
 * timing a bracket of several calls on the launching stream. */
int qk_mark(qk_sim* sim, int slot);
int qk_mark_elapsed(qk_sim* sim, int slot_a, int slot_b, double* ms);

/* Synchronize the handle's streams. */
int qk_sync(qk_sim* sim);

#ifdef __cplusplus
}
#endif
#endif /* QKB200_H */
