/*
 * nucsim_b200.h -- C ABI of the B200-native gate-application path.
 *
 * The reference (arXiv 2310.17739 `nucsim` 0.1.0, /root/reference/pkg) has no
 * FFI: its boundary is the Python API re-exported by nucsim/__init__.py:10-76.
 * Each entry point below replaces one reference function on the hot path
 * (SURVEY.md section 8b); the replaced reference symbol is cited per entry.
 * The Python mirror of that API (paper_2310_17739_b200/) binds these symbols
 * with ctypes; INTEGRATION.md shows the binding a nucsim maintainer would add.
 *
 * Conventions
 *   - Complex numbers are interleaved (re, im) float64 pairs; matrices are
 *     row-major, matrix index = sum_j bit(qubits[j]) << j (slot 0 = LSB),
 *     exactly the reference convention (gates.py:1-17, engine.py:104-107).
 *   - State vectors are little-endian: qubit 0 is the least significant bit
 *     of the basis index (engine.py:1-6).
 *   - Every call returns an int status (NSB_OK = 0).  Calls that can fail
 *     with a reference exception also fill an nsb_status (may be NULL).
 *     No C++ exception, callback or torch type crosses this ABI.
 *   - Calls are synchronous: device work has completed when they return.
 */
#ifndef NUCSIM_B200_H
#define NUCSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSB_ABI_VERSION 1

/* ---- status ------------------------------------------------------------ */
enum {
  NSB_OK = 0,
  NSB_EINVAL = 1,    /* ValueError                     (engine.py:88-89, 96-97, 110-115) */
  NSB_EASSERT = 2,   /* FilterAssertionError(step, prob) (engine.py:187-190, errors.py:27-33) */
  NSB_EPROJECT = 3,  /* ProjectionError                (engine.py:177-178) */
  NSB_ERESOURCE = 4, /* ResourceLimitError / out of device memory */
  NSB_EDEVICE = 5,   /* CUDA / NCCL failure -> RuntimeError */
  NSB_EQASM = 6      /* QasmError(msg, line = step, col = prob)  (errors.py:14-20) */
};

typedef struct nsb_status {
  int32_t code;
  int32_t step; /* NSB_EASSERT: assertion step */
  double prob;  /* NSB_EASSERT / NSB_EPROJECT: offending probability */
  char msg[256];
} nsb_status;

/* ---- packed instruction list (the SoA-free op record) -------------------
 * One record per reference Instruction (circuit.py:20-47).  `tag` is the
 * gate code = position of the tag in the reference's Gate enum
 * (gates.py:30-71); markers use NSB_OP_MEASURE / RESET / BARRIER kinds.    */
enum { NSB_OP_GATE = 0, NSB_OP_MEASURE = 1, NSB_OP_RESET = 2, NSB_OP_BARRIER = 3 };

enum {
  NSB_GATE_U3 = 0, NSB_GATE_U2, NSB_GATE_U1, NSB_GATE_CX, NSB_GATE_ID, NSB_GATE_X,
  NSB_GATE_Y, NSB_GATE_Z, NSB_GATE_H, NSB_GATE_S, NSB_GATE_SDG, NSB_GATE_T,
  NSB_GATE_TDG, NSB_GATE_RX, NSB_GATE_RY, NSB_GATE_RZ, NSB_GATE_CZ, NSB_GATE_CY,
  NSB_GATE_SWAP, NSB_GATE_CH, NSB_GATE_CCX, NSB_GATE_CSWAP, NSB_GATE_CRX,
  NSB_GATE_CRY, NSB_GATE_CRZ, NSB_GATE_CU1, NSB_GATE_CU3, NSB_GATE_RXX,
  NSB_GATE_RZZ, NSB_GATE_RCCX, NSB_GATE_RC3X, NSB_GATE_C3X, NSB_GATE_C3SQRTX,
  NSB_GATE_C4X, NSB_GATE_C1, NSB_GATE_C2, NSB_GATE_MEASURE, NSB_GATE_RESET,
  NSB_GATE_BARRIER, NSB_GATE_COUNT
};

typedef struct nsb_op {
  int32_t kind;    /* NSB_OP_* */
  int32_t tag;     /* NSB_GATE_* */
  int32_t nq;      /* qubits listed in q[] (0 for barrier: see mask) */
  int32_t cbit;    /* measure target bit, else -1 */
  int32_t q[5];    /* qubits in slot order */
  int32_t src;     /* input index this op was copied from unchanged, else -1 */
  int64_t param;   /* offset into the float64 params pool, else -1 */
  int64_t payload; /* offset in COMPLEX elements into the payload pool, else -1 */
  uint64_t mask;   /* qubit set as a bitmask (all kinds, n <= 64) */
} nsb_op;          /* 64 bytes */

/* ---- gate vocabulary --------------------------------------------------- */

/* Dense matrix of a named gate, bit-identical to reference gate_matrix
 * (gates.py:283-291).  out: (2^k)^2 complex.  Replaces gates.gate_matrix. */
int nsb_gate_matrix(int32_t tag, const double* params, int32_t n_params, double* out);

/* ---- OpenQASM 2.0 reader (replaces qasm.parse_qasm, qasm.py:30-347) ------
 * The reference subset: header + qelib1 include, one qreg (<= 64 qubits
 * here), named cregs (also before the qreg), the qelib1 gate names, measure /
 * reset / barrier (indexed or whole register), `//` comments, constant angle
 * expressions folded to doubles in the reference's order.  Output records
 * are ready for nsb_fuse / nsb_plan_create.  Barrier records: nq = 0, mask =
 * the qubit set, param = offset of their operands (first-occurrence order)
 * in barrier_qubits, cbit = their count.  Errors: NSB_EQASM with the
 * reference's message, st->step = line, st->prob = column.                */
typedef struct nsb_qasm {
  int32_t n_qubits;
  int32_t n_cregs;
  nsb_op* ops;              /* library-owned: nsb_qasm_free */
  int64_t n_ops;
  double* params;           /* float64 parameter pool referenced by ops[].param */
  int64_t n_params;
  int32_t* barrier_qubits;
  int64_t n_barrier_qubits;
  char* creg_names;         /* n_cregs NUL-terminated names, declaration order */
  int64_t* creg_sizes;
} nsb_qasm;
int nsb_qasm_parse(const char* text, int64_t len, nsb_qasm* out, nsb_status* st);
void nsb_qasm_free(nsb_qasm* q);

/* ---- fusion (replaces fusion.fuse_pipeline, fusion.py:240-251) --------- */
enum { NSB_PASS_MERGE_1Q = 1, NSB_PASS_ABSORB_1Q = 2, NSB_PASS_NORMALIZE_2Q = 4,
       NSB_PASS_FUSE_2Q = 8, NSB_PASS_ALL = 15 };

/* OpenBLAS zgemm FMA order the reference's `@` reproduces on the host
 * (SURVEY Appendix A.3): CHAIN2 = SkylakeX/SapphireRapids cores (2x2 single
 * chain, 4x4 four accumulators), FOUR = Haswell/Zen (four accumulators). */
enum { NSB_BLAS_CHAIN2 = 1, NSB_BLAS_FOUR = 2 };

typedef struct nsb_fused {
  nsb_op* ops;        /* fused list, library-owned (nsb_fused_free) */
  int64_t n_ops;
  double* payloads;   /* complex payload pool referenced by ops[].payload */
  int64_t n_payload;  /* complex elements */
  int64_t gates_before;
  int64_t pass_before[4]; /* gate counts around each pass (fusion.py:77-79) */
  int64_t pass_after[4];
} nsb_fused;

/* Run the selected passes in the reference order merge_1q -> absorb_1q ->
 * normalize_2q_order -> fuse_2q (fusion.py:101-237).  Unchanged input ops
 * keep `src`; fused C1/C2 payloads live in out->payloads. */
int nsb_fuse(const nsb_op* ops, int64_t n_ops, const double* params,
             const double* payloads, int32_t pass_mask, int32_t blas_variant,
             nsb_fused* out, nsb_status* st);
void nsb_fused_free(nsb_fused* f);

/* ---- native workload generator (projection.build_filter_circuit,
 *      projection.py:191-255) ------------------------------------------- */
/* terms: n_terms Pauli words, letters[t*n_system + q] in {0:I,1:X,2:Y,3:Z};
 * coeffs: real coefficients (already in the reference's sorted_terms order);
 * steps: n_steps (t_i, delta_i) pairs.  Emits the instruction stream of
 * build_filter_circuit(h, schedule, trotter, basis trial `trial_bits`). */
int nsb_generate_filter(int32_t n_system, const uint8_t* letters, const double* coeffs,
                        int64_t n_terms, const double* steps, int32_t n_steps,
                        int64_t trotter, const uint8_t* trial_bits,
                        nsb_fused* out, double** params_out, int64_t* n_params_out,
                        nsb_status* st);
void nsb_free(void* p);

/* ---- device context and state (replaces engine.StateVector,
 *      engine.py:42-84) --------------------------------------------------- */
typedef struct nsb_ctx nsb_ctx;

int nsb_device_count(int32_t* n);
int nsb_ctx_create(int32_t device, nsb_ctx** out, nsb_status* st);
void nsb_ctx_destroy(nsb_ctx* ctx);
/* allocate 2^n amplitudes on the device and set |0...0> */
int nsb_state_init(nsb_ctx* ctx, int32_t n_qubits, nsb_status* st);
int nsb_state_reset(nsb_ctx* ctx, nsb_status* st);                /* StateVector.restart */
int nsb_state_upload(nsb_ctx* ctx, const double* amps, nsb_status* st);
int nsb_state_download(nsb_ctx* ctx, double* amps, nsb_status* st);
int nsb_state_norm2(nsb_ctx* ctx, double* out, nsb_status* st);

/* ---- single-op kernels (apply_1q / apply_2q / apply_dense,
 *      engine.py:92-156) --------------------------------------------------- */
/* k = 1..5 distinct qubits; u is (2^k)^2 complex, slot j = qubits[j]. */
int nsb_apply_matrix(nsb_ctx* ctx, const double* u, const int32_t* qubits, int32_t k,
                     nsb_status* st);

/* ---- measurement (engine.py:159-191) ---------------------------------- */
/* P(qubit q = outcome) = sum |a_i|^2 over that half (_branch_probability) */
int nsb_branch_probability(nsb_ctx* ctx, int32_t q, int32_t outcome, double* p,
                           nsb_status* st);
/* zero the other half and scale by 1/sqrt(prob) (_project) */
int nsb_project(nsb_ctx* ctx, int32_t q, int32_t outcome, double prob, nsb_status* st);
/* |a_i|^2 as re*re + im*im without FMA contraction (sample, engine.py:215) */
int nsb_probabilities(nsb_ctx* ctx, double* out, nsb_status* st);
/* Sampling a sharded state (sample, engine.py:207-222, at scale): sums of
 * |a_i|^2 over consecutive chunks of 2^chunk_log2 local amplitudes
 * (deterministic fixed-order device reduction; out has 2^(n - chunk_log2)
 * entries), and |a_i|^2 of one local index range [offset, offset + count). */
int nsb_prob_chunk_sums(nsb_ctx* ctx, int32_t chunk_log2, double* out, nsb_status* st);
int nsb_probabilities_range(nsb_ctx* ctx, uint64_t offset, uint64_t count, double* out,
                            nsb_status* st);
/* <psi| sum_t c_t P_t |psi> (expectation_pauli, engine.py:225-239).
 * Term t acts as (P_t psi)[j] = (-1)^popcount(j & zmask[t]) psi[j ^ xmask[t]]
 * (xmask: X and Y letters, zmask: Z and Y letters); coeffs are complex
 * (re, im) pairs with the (-i)^#Y phase of the Y letters already folded in. */
int nsb_expectation_pauli(nsb_ctx* ctx, const uint64_t* xmask, const uint64_t* zmask,
                          const double* coeffs, int64_t n_terms, double* out_re,
                          double* out_im, nsb_status* st);

/* ---- compiled plans: the fused gate stream resident on the device
 *      (engine._compile + run, engine.py:295-477) ------------------------ */
typedef struct nsb_plan nsb_plan;

typedef struct nsb_plan_info {
  int64_t n_gates;      /* gate ops in the plan */
  int64_t n_measures;   /* mid-circuit MEASURE ops */
  int64_t n_resets;
  int64_t n_passes;     /* state sweeps (memory passes) the schedule needs */
  int64_t n_segments;   /* gate segments between MEASURE/RESET ops */
  int64_t flops;        /* FP64 flops of all gate ops (8 * nnz * 2^(n-k)) */
  int64_t tile_qubits;  /* qubits per cache-blocked tile */
  int64_t n_items;      /* gate segments + markers (nsb_plan_segment_marker) */
  int64_t n_frame_gates; /* exact CX/SWAP absorbed by the relabeling frame */
  int64_t n_flush_gates; /* physical CX emitted to flush the frame */
  int64_t n_device_gates;/* gate ops executed on the device per run */
  int64_t n_sweeps;      /* shared-memory octet sweeps (gate groups) per run */
  int64_t n_fused_group_ops; /* gate ops merged away by group fusion (whole-octet ops) */
  int64_t n_identity_gates;  /* payloads within rounding of the identity, not executed */
  double identity_error;     /* sum of their ||U - I||_F: bound on the relative L2 change */
} nsb_plan_info;

/* ops: the executable part of the circuit (sampling block already removed,
 * barriers allowed and dropped).  Matrices of named gates come from params
 * (nsb_gate_matrix), C1/C2/k-qubit payloads from `payloads`. */
int nsb_plan_create(nsb_ctx* ctx, const nsb_op* ops, int64_t n_ops, const double* params,
                    const double* payloads, nsb_plan** out, nsb_status* st);
/* nsb_plan_create with flags: NSB_PLAN_EXACT executes every gate, including
 * those within rounding of a scalar identity (for callers that measure the
 * state between nsb_plan_run_segment calls themselves: rejection mode, the
 * sharded schedule). */
enum { NSB_PLAN_EXACT = 1 };
int nsb_plan_create_ex(nsb_ctx* ctx, const nsb_op* ops, int64_t n_ops, const double* params,
                       const double* payloads, int32_t flags, nsb_plan** out, nsb_status* st);
void nsb_plan_destroy(nsb_plan* plan);
/* Host-only dry run of the planner (no device needed): the schedule that
 * nsb_plan_create would upload, summarised.  class_counts (NSB_N_CLASSES
 * entries, may be NULL) receives the gate count per payload class: dense 1q,
 * diagonal 1q, dense 2q, <=2 nnz/row 2q, monomial 2q, diagonal 2q, exact CX
 * (two orientations), two-block 2x2 patterns (three pairings), exact SWAP,
 * read-map-only permutation sweeps. */
#define NSB_N_CLASSES 16
int nsb_plan_analyze(const nsb_op* ops, int64_t n_ops, const double* params,
                     const double* payloads, int32_t n_qubits, nsb_plan_info* info,
                     int64_t* class_counts, nsb_status* st);
int nsb_plan_info_get(const nsb_plan* plan, nsb_plan_info* info);

/* Host-side view of a compiled plan, for tests and tooling: the device
 * program exactly as nsb_plan_create would upload it (PassDesc / GroupDesc / GateOp
 * records of paper_2310_17739_b200/csrc/planner.h, packed matrices).  The
 * library never executes a plan on the host; tests/plan_exec.py does, to
 * verify the planner on machines without a GPU. */
typedef struct nsb_plan_view {
  int32_t n_qubits, tile_qubits, mma_ok, n_measures;
  int32_t pass_desc_bytes, group_desc_bytes, gate_op_bytes;
  int32_t tma_edges;       /* 1: tiles move by TMA -- each pass's first group loads and its
                              last group stores under the 128-byte TMA swizzle */
  int64_t n_passes, n_mma_passes, n_groups, n_gate_ops, n_matrices, n_items;
  const void* passes;      /* plain gate passes (items reference ranges) */
  const void* mma_passes;  /* single-launch MMA program */
  const void* groups;      /* GroupDesc records */
  const void* gate_ops;    /* GateOp records */
  const double* matrices;  /* complex pool */
  const int32_t* items;    /* n_items x 4: kind (0 gates, 1 measure, 2 reset,
                              3 dense), pass_begin | qubit, pass_end | step, k */
  int32_t octets;          /* octets per thread of the kernel layout (1: 256 threads, small
                              states; 2: 128 threads) */
  int32_t thread_bits;     /* log2 threads per CTA */
} nsb_plan_view;
int nsb_host_plan_build(const nsb_op* ops, int64_t n_ops, const double* params,
                        const double* payloads, int32_t n_qubits, int32_t workers, void** out,
                        nsb_status* st);
int nsb_host_plan_view(const void* plan, nsb_plan_view* view);
void nsb_host_plan_free(void* plan);
/* Chunked execution of a gate item (nsb_shard_swap_overlap): the longest
 * prefix of item `item`'s passes whose tiles all leave `want_bits` local
 * qubits other than `avoid_q` untouched (fewer bits if none); *cmask = those
 * qubits (the highest free ones), *n_pass = the prefix length (0: none). */
int nsb_host_plan_chunk_prefix(const void* plan, int64_t item, int32_t avoid_q,
                               int32_t want_bits, int32_t* n_pass, uint64_t* cmask);

/* MMA mode (engine.py:414-423): execute the whole plan from the current
 * state; each MEASURE asserts |0> (p0 < eps -> NSB_EASSERT with step/p0),
 * records p0 into assert_probs[step] and renormalises; RESET is a no-op. */
int nsb_plan_run_mma(nsb_ctx* ctx, nsb_plan* plan, double eps, double* assert_probs,
                     nsb_status* st);
/* Gate segment `seg` only (rejection mode drives MEASURE/RESET from the host,
 * engine.py:439-459).  Segment s ends at marker op index seg_marker[s]. */
int nsb_plan_run_segment(nsb_ctx* ctx, nsb_plan* plan, int64_t seg, nsb_status* st);
int nsb_plan_segment_marker(const nsb_plan* plan, int64_t seg, int32_t* kind, int32_t* qubit,
                            int32_t* step);
/* Gate item `seg`, its chunkable pass prefix (nsb_host_plan_chunk_prefix
 * with avoid_q = -1) run one chunk of 2^chunk_bits at a time, the rest as
 * usual: the same state as nsb_plan_run_segment (the single-GPU check of
 * the chunked launches that nsb_shard_swap_overlap pipelines).
 * *n_chunked = passes run chunk-wise (0: none, the item ran whole). */
int nsb_plan_run_segment_chunked(nsb_ctx* ctx, nsb_plan* plan, int64_t seg, int32_t chunk_bits,
                                 int32_t* n_chunked, nsb_status* st);

/* MMA run with planning streamed behind execution (replaces engine.run(...,
 * "mma")'s gate loop, engine.py:414-423): the op list is cut at its MEASURE /
 * RESET markers, a host thread plans the parts in order and part s runs on
 * the device (one cooperative launch) while part s+1 is planned.  Same
 * outputs and errors as nsb_plan_create + nsb_plan_run_mma (n_measures: the
 * number of assertion probabilities written; device_ms, nullable: device
 * time of the launches).  1q / 2q gates and >= 6 qubits only (else
 * NSB_EINVAL: use the plan calls). */
int nsb_run_mma_streamed(nsb_ctx* ctx, const nsb_op* ops, int64_t n_ops, const double* params,
                         const double* payloads, double eps, double* assert_probs,
                         int64_t* n_measures, double* device_ms, nsb_status* st);

/* Rejection mode (replaces engine.run(..., "rejection"), engine.py:431-474).
 * Plan: built with NSB_PLAN_EXACT.  uniforms: the caller's Philox stream
 * (rng.random() draws, in order; n_uniforms available), consumed in the
 * reference's order -- one per executed MEASURE and RESET, one per accepted
 * shot's sample; *consumed returns how many were used (the caller advances
 * its generator by that many).  Outputs: *accepted, step_rejections
 * [n_measures], sample_index[shots] (basis index of each accepted shot's
 * sample, engine.py:207-222; -1 for a rejected shot), first_state (nullable,
 * 2^n interleaved complex): the first accepted shot's final state (the
 * reference's energy input).  Filter-shaped circuits are replayed from one
 * device pass along the accepted path (a reset draw of 1 falls back to an
 * explicit shot); flags & 1 forces explicit per-shot simulation.
 * NSB_EINVAL if the stream runs out. */
int nsb_plan_run_rejection(nsb_ctx* ctx, nsb_plan* plan, const double* uniforms,
                           int64_t n_uniforms, int64_t shots, int32_t flags, int64_t* consumed,
                           int64_t* accepted, int64_t* step_rejections, int64_t* sample_index,
                           double* first_state, nsb_status* st);

/* Factor between the state's P(|0>) at assertion `step` and the reference's
 * (engine.py:159-161): the product of |s|^2 of the near-scalar gates s I the
 * plan does not execute since the previous assertion (nsb_plan_info
 * n_identity_gates).  nsb_plan_run_mma applies it; callers that measure
 * between nsb_plan_run_segment calls multiply their p0 by it. */
int nsb_plan_p0_scale(const nsb_plan* plan, int32_t step, double* scale);

/* Device time of the last nsb_plan_run_* call in milliseconds (CUDA events
 * on the launching stream), and the number of kernels it launched. */
int nsb_plan_last_timing(const nsb_plan* plan, double* ms, int64_t* launches);

/* Device-side timer on the context's stream (CUDA events): the elapsed
 * device time of everything the context enqueued between the two calls. */
int nsb_timer_start(nsb_ctx* ctx, nsb_status* st);
int nsb_timer_stop(nsb_ctx* ctx, double* ms, nsb_status* st);

/* ---- Sharded state (one process per GPU, NCCL over NVLink) -------------
 * A state of n qubits is split on its top g = log2(nranks) qubits: rank r
 * keeps the 2^(n-g) amplitudes whose top bits equal r, as the ordinary
 * (n-g)-qubit state of its context.  Gates on the local qubits run through
 * the single-GPU calls above; paper_2310_17739_b200/sharded.py schedules the
 * qubit swaps that bring a global qubit into the local range (SURVEY.md
 * 8(e); the reference has no multi-device path -- it replaces engine.py's
 * full-state loops for states larger than one GPU).
 *
 * nsb_comm_unique_id: 128-byte NCCL id, made on one rank and shared with the
 * others through any host channel.  nsb_comm_init: bind the context to rank
 * `rank` of `nranks` (a power of two).
 * nsb_shard_swap: global qubit `global_bit` (rank bit) and local qubit
 * `local_q` trade places.  The half of the shard whose bit local_q differs
 * from this rank's bit is exchanged element for element with the partner
 * rank (rank ^ 1 << global_bit), in chunks of chunk_amps (<= 0: 2^26).
 * Collective: both partners must call it.
 * nsb_shard_reset: the shard of |0...0> (rank 0: amplitude 1 at index 0;
 * other ranks: zeros), on the device.
 * nsb_shard_allgather: every rank contributes `count` doubles; `out`
 * receives nranks * count values in rank order (deterministic sums).
 * nsb_shard_ipc_handle: 64-byte CUDA IPC handle of this rank's shard;
 * nsb_shard_open_peers: map every other rank's shard (handles: nranks x 64
 * bytes in rank order, own entry ignored) into this context.
 * nsb_shard_swap_p2p: nsb_shard_swap through peer memory over NVLink: the
 * element pairs are split in chunks, this rank swaps the chunks of its
 * parity with one kernel that reads and writes both shards directly (no
 * staging copies, no pack / unpack), between two stream-ordered barriers.
 * Collective: both partners must call it (after nsb_shard_open_peers).
 * Opening checks that every rank's shard has this rank's size and re-maps
 * shards that were already mapped.  nsb_shard_close_peers (collective):
 * unmap them and rendezvous, so no rank frees or reallocates its exported
 * shard while a partner still maps it; nsb_state_init refuses to resize a
 * shard while peers are mapped. */
int nsb_comm_unique_id(uint8_t* id, nsb_status* st);
int nsb_comm_init(nsb_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank,
                  nsb_status* st);
int nsb_shard_swap(nsb_ctx* ctx, int32_t global_bit, int32_t local_q, int64_t chunk_amps,
                   nsb_status* st);
int nsb_shard_reset(nsb_ctx* ctx, nsb_status* st);
int nsb_shard_allgather(nsb_ctx* ctx, const double* in, int32_t count, double* out,
                        nsb_status* st);
int nsb_shard_ipc_handle(nsb_ctx* ctx, uint8_t* handle, nsb_status* st);
int nsb_shard_open_peers(nsb_ctx* ctx, const uint8_t* handles, nsb_status* st);
int nsb_shard_swap_p2p(nsb_ctx* ctx, int32_t global_bit, int32_t local_q, nsb_status* st);
int nsb_shard_close_peers(nsb_ctx* ctx, nsb_status* st);
/* A qubit swap overlapped with the gate item that follows it (north_star:
 * "qubit-remap ... overlapped with local-gate blocks"; the reference has no
 * counterpart -- its state is one host array, engine.py:51, 68-71).  The
 * item's chunkable pass prefix (nsb_host_plan_chunk_prefix, avoid_q =
 * local_q) runs chunk by chunk on the context stream while the peer-memory
 * swap (nsb_shard_swap_p2p's exchange) moves the next chunk on a second
 * stream with `swap_ctas` CTAs (0: default 32); chunk c's passes start once
 * both partners' halves of chunk c have landed (per-chunk flags written over
 * NVLink).  The rest of the item then runs on all tiles.  Falls back to
 * swap-then-item when no pass prefix is chunkable.  Collective: both
 * partners call it with the same arguments (their plans are the same
 * schedule step).  *n_chunked = passes overlapped (0: none). */
int nsb_shard_swap_overlap(nsb_ctx* ctx, int32_t global_bit, int32_t local_q, nsb_plan* plan,
                           int64_t seg, int32_t chunk_bits, int32_t swap_ctas,
                           int32_t* n_chunked, nsb_status* st);
/* The same overlap with the exchange on the COPY ENGINES (no SMs): per block
 * of a chunk, each partner pulls the other's half into a staging slot of its
 * own (a 2-D peer cudaMemcpy over NVLink), tells the partner so (a stream
 * memory write into the partner's flag word), waits for the partner's word,
 * and copies the slot into its own half (a local copy-engine copy); chunk c's
 * passes run at the full grid once its blocks are in.  stage_bytes bounds a
 * staging slot (two slots; 0: 4 GiB).  Same semantics and collective
 * contract as nsb_shard_swap_overlap. */
int nsb_shard_swap_overlap_ce(nsb_ctx* ctx, int32_t global_bit, int32_t local_q,
                              nsb_plan* plan, int64_t seg, int32_t chunk_bits,
                              int64_t stage_bytes, int32_t* n_chunked, nsb_status* st);

#ifdef __cplusplus
}
#endif
#endif /* NUCSIM_B200_H */
