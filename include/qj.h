/*
 * qj.h -- C ABI of the B200 state-vector gate-application library (libqj.so).
 *
 * What it computes: Schroedinger state-vector gate application, Eq. 1 of
 * "Quantum simulation with just-in-time compilation" (PAPER.md:79-86,
 * \label{eq:gateapplication}):
 *
 *     psi'(sigma_1..tau..sigma_n) = sum_{tau'} G(tau, tau') psi(sigma_1..tau'..sigma_n)
 *
 * applied IN PLACE ("custom operators perform in-place
 * updates"), with the sparsity of Pauli / controlled gates exploited
 * and specialised X / Z / SWAP operators,
 * plus fSim / diagonal entry points and circuit execution named by the
 * BASELINE.json north star, and Born-rule probabilities.
 *
 * Conventions (DESIGN.md readings):
 *   R1  qubit q is bit (n-1-q) of the basis index (qubit 0 = most significant).
 *   R3  gate matrices are row-major 2^k x 2^k; the first-listed target is the
 *       most significant bit of the row/column index.  Targets may be listed in
 *       any order.
 *   R4  controls: the gate acts only where every control qubit is 1.
 *   Data: amplitudes are interleaved (re, im); complex64 = 2 x float,
 *       complex128 = 2 x double.  Host-side matrices / diagonals / fSim
 *       parameters are interleaved complex values IN THE STATE'S DTYPE.
 *
 * Ownership: the caller owns the amplitude buffer (e.g. a torch tensor:
 * contiguous, 16-byte aligned, >= 2^n_local elements, alive while the handle
 * lives).  The library owns its scratch (reduction bins, staged gate programs)
 * and frees it in qj_state_free.  Every host array passed in (targets,
 * controls, matrices, gate lists) is copied or consumed before the call
 * returns; the caller may free it immediately.
 *
 * Execution: all device work is enqueued on the handle's CUDA stream and is
 * asynchronous w.r.t. the host; qj_sync blocks.  A handle is not thread-safe:
 * one thread mutates it at a time.
 *
 * Errors: every entry point returns a qj_status.  Argument errors are detected
 * synchronously, before anything is enqueued, and leave the state untouched.
 * Asynchronous CUDA failures surface as QJ_ERR_CUDA on a later call or on
 * qj_sync.  qj_last_error() returns a thread-local message for the last failure.
 * No C++ exception crosses this ABI.  Matrices are not checked for unitarity
 * and the state is never renormalised.
 */
#ifndef QJ_H
#define QJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QJ_OK = 0,
    QJ_ERR_INVALID_ARG = 1,        /* NULL pointer, nt < 1, n != state's n, bad flag */
    QJ_ERR_INDEX_OUT_OF_RANGE = 2, /* qubit >= n, basis_index >= 2^n */
    QJ_ERR_OVERLAPPING_QUBITS = 3, /* duplicate qubit, or targets and controls intersect */
    QJ_ERR_TOO_MANY_TARGETS = 4,   /* nt > QJ_MAX_TARGETS or nc > QJ_MAX_CONTROLS */
    QJ_ERR_CAPACITY = 5,           /* n outside [1, QJ_MAX_QUBITS] or shard too large */
    QJ_ERR_DTYPE = 6,              /* unknown dtype */
    QJ_ERR_CUDA = 7,               /* a CUDA runtime error (launch or asynchronous) */
    QJ_ERR_NCCL = 8,               /* a NCCL error in the multi-GPU layer */
    QJ_ERR_UNSUPPORTED = 9,        /* valid request this build does not implement */
    QJ_ERR_ZERO_PROBABILITY = 10   /* collapse / sampling on an outcome set of probability ~0 */
} qj_status;

typedef enum { QJ_C64 = 0, QJ_C128 = 1 } qj_dtype;

typedef struct qj_state_s* qj_state;

#define QJ_KEEP UINT64_MAX   /* qj_state_init: leave the buffer's contents as they are */
#define QJ_MAX_TARGETS 8
#define QJ_MAX_CONTROLS 16
#define QJ_MAX_QUBITS 40     /* total qubits; a shard must also fit one GPU */

/* ---- state handle ---------------------------------------------------------
 * qj_state_init: wrap the caller's device buffer `amps_dev` (2^n amplitudes of
 * dtype `dt` on the current device) and, unless basis_index == QJ_KEEP, write
 * the basis state |basis_index> into it (|0..0> for 0).
 * `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 * `nccl_comm` = NULL for a single-GPU state; otherwise an ncclComm_t of P
 * ranks (one process per GPU, P a power of two): the state is then rank
 * r's shard of an n-qubit state sharded on its top log2(P) qubits, amps_dev
 * holds 2^(n - log2 P) amplitudes, and gates on global qubits run through
 * local<->global exchanges (grouped ncclSend/ncclRecv through a bounded
 * staging ring; NCCL is dlopen'ed on first use).  Every rank must make the
 * same sequence of calls.  (qj_state_init_sharded: P virtual shards in one
 * process.)
 * Errors: INVALID_ARG (out or amps_dev NULL), CAPACITY (n < 1 or n > 40),
 * DTYPE, INDEX_OUT_OF_RANGE (basis_index >= 2^n), CUDA. */
qj_status qj_state_init(qj_state* out, void* amps_dev, int n, qj_dtype dt,
                        uint64_t basis_index, void* cuda_stream, void* nccl_comm);

/* Sharded state on the top g = log2(nshards) "global" qubits (
 * the paper's multi-device scheme is PAPER.md:469-489).  Shard r holds the
 * 2^(n-g) amplitudes whose global bits equal r, while the qubit map is
 * canonical.  `shards` = nshards device pointers, all owned by this process
 * on this device (virtual ranks; nshards a power of two >= 1).  Gates on
 * global qubits are applied through local<->global qubit swaps executed as
 * device-to-device exchanges; qubit labels stay logical at this ABI. */
qj_status qj_state_init_sharded(qj_state* out, void* const* shards, int nshards, int n,
                                qj_dtype dt, uint64_t basis_index, void* cuda_stream);

/* Host-staged state ("the full state vector is stored in
 * the host memory ... only slices of it are transferred to the GPUs for
 * calculation", with "a single GPU that is re-used for multiple state
 * slices").  `amps_host` is caller-owned HOST memory of 2^n amplitudes
 * (16-byte aligned; pin it -- cudaHostRegister / cudaMallocHost -- or copies
 * cannot overlap), split into `nslices` (power of two) slices on the top
 * log2(nslices) qubits.  The planner is the sharded one; each run of per-slice
 * passes between global-qubit exchanges streams every slice through the GPU
 * once (three slice buffers of 2^(n - log2 nslices) amplitudes in HBM, H2D /
 * compute / D2H overlapped on separate streams).  A slice is held as two
 * half-slices through a pointer table: a global-qubit exchange with the top
 * local bit swaps table entries (no bytes move); one with a lower local bit L
 * adds SWAP(L, top) passes to the neighbouring sweeps.  Results are bit
 * identical to qj_state_init_sharded with the same slice count.  After
 * exchanges the caller's buffer holds the half-slices in permuted order (like
 * the permuted bit order of device states); qj_state_canonicalize restores
 * the canonical layout (host block moves) and returns after the data is in
 * place; otherwise the buffer is valid after qj_sync.  Plans are not cached.
 * qj_probabilities' out_dev, qj_sample and qj_collapse work as for device
 * states.  Errors: as qj_state_init_sharded; CUDA errors if the slice buffers
 * do not fit the device. */
qj_status qj_state_init_host(qj_state* out, void* amps_host, int n, qj_dtype dt, int nslices,
                             uint64_t basis_index, void* cuda_stream);

/* Re-initialise an existing handle to |basis_index> (QJ_KEEP: no-op). */
qj_status qj_state_reset(qj_state s, uint64_t basis_index);

/* Release the handle and library scratch.  The amplitude buffer is the caller's. */
qj_status qj_state_free(qj_state s);

/* ---- gate application (Eq. 1) ----------------------------------------------
 * qj_apply_gate: apply the 2^nt x 2^nt matrix `matrix` (host, row-major,
 * state dtype) to `targets` (nt qubits, listed order = matrix bit order R3),
 * controlled on `controls` (nc qubits, may be NULL when nc == 0).  `n` must
 * equal the state's qubit count (S:124 ShapeMismatch -> INVALID_ARG). */
qj_status qj_apply_gate(qj_state s, int n, const int* targets, int nt,
                        const int* controls, int nc, const void* matrix);

/* Specialised operators: amplitude permutations / sign
 * flips with no arithmetic; results are exact (IEEE ==) vs Eq. 1. */
qj_status qj_apply_x(qj_state s, int target, const int* controls, int nc);
qj_status qj_apply_z(qj_state s, int target, const int* controls, int nc);
qj_status qj_apply_swap(qj_state s, int t0, int t1, const int* controls, int nc);

/* fSim: [[1,0,0,0],[0,u00,u01,0],[0,u10,u11,0],[0,0,0,phase11]] on (t0, t1)
 * (t0 = MSB).  u2x2: 4 complex (row-major), phase11: 1 complex (e^{-i phi}). */
qj_status qj_apply_fsim(qj_state s, int t0, int t1, const void* u2x2, const void* phase11,
                        const int* controls, int nc);

/* Diagonal gate: psi_i <- diag[row(i)] psi_i, row(i) = target bits of i in
 * listed order (first = MSB); `diag` = 2^nt complex values. */
qj_status qj_apply_diagonal(qj_state s, const int* targets, int nt, const void* diag,
                            const int* controls, int nc);

/* ---- circuits --------------------------------------------------------------- */
typedef enum {
    QJ_GATE_DENSE = 0,   /* data: 4^nt complex (row-major matrix)       */
    QJ_GATE_X = 1,       /* data: unused                                */
    QJ_GATE_Z = 2,       /* data: unused                                */
    QJ_GATE_SWAP = 3,    /* data: unused (nt == 2)                      */
    QJ_GATE_FSIM = 4,    /* data: 5 complex: u00,u01,u10,u11,phase11    */
    QJ_GATE_DIAG = 5     /* data: 2^nt complex                          */
} qj_gate_kind;

typedef struct {
    int kind;
    int nt;
    int nc;
    int targets[QJ_MAX_TARGETS];
    int controls[QJ_MAX_CONTROLS];
    const void* data;    /* host pointer, state dtype, read before return */
} qj_gate;

#define QJ_FUSE 1u       /* plan runs of gates into fused window tile passes */
#define QJ_FUSE_GATES 2u /* first apply the paper's greedy fusion into <= 2-qubit
                            dense gates; combinable with QJ_FUSE */
/* QJ_FUSE_GATES with a fusion width k in 1..5 (bits 4-7; 0 = 2, the paper's):
 * "fusing gates up to about five [qubits] may provide additional advantage"
 * (PAPER.md:574-575).  complex64 dense fused gates of 4-5 qubits run as
 * tensor-core contractions (3xTF32 tcgen05.mma). */
#define QJ_FUSE_GATES_K(k) (QJ_FUSE_GATES | (((uint32_t)(k) & 15u) << 4))

/* Apply `ngates` gates in order.  Without QJ_FUSE every gate is one pass as
 * if issued through the single-gate entry points.  With QJ_FUSE the planner
 * groups runs of consecutive gates into window passes (one HBM round trip per
 * run, PAPER.md:539-550 fusion, done B200-style); results agree with the
 * unfused path within floating-point tolerance.  All gates are validated
 * before anything is enqueued. */
qj_status qj_apply_circuit(qj_state s, const qj_gate* gates, int ngates, uint32_t flags);

/* One simulation step in a single call: the same result as
 *     qj_state_reset(s, basis); qj_apply_circuit(s, gates, ngates, flags);
 *     qj_probabilities(s, qubits, nq, out_dev)   (skipped when nq == 0)
 * with the state left in the buffer (possibly in a permuted bit order, as
 * after qj_apply_circuit).  With QJ_FUSE on a single-device state (nq <= 10,
 * JIT available) the library fuses the step's ends into its tile passes:
 * the first pass synthesises |basis> in registers instead of reading an
 * initialised buffer, and the last pass accumulates the fp64 marginal while
 * it stores -- two fewer sweeps over the state.  Marginal sums are
 * accumulated in a different order than qj_probabilities (agreement to fp64
 * rounding).  Otherwise it runs the three calls.  Plans (and, from the
 * second call on a non-default stream, a CUDA graph of the whole step) are
 * cached per (circuit, flags, basis, qubits); out_dev is patched per call.  Errors: as the three
 * calls. */
qj_status qj_simulate(qj_state s, uint64_t basis, const qj_gate* gates, int ngates, uint32_t flags,
                      const int* qubits, int nq, void* out_dev);

/* Physical layout.  Qubit labels at this ABI are always logical: the handle
 * tracks a logical->physical bit map.  Fused circuits apply uncontrolled SWAP
 * gates as relabellings of that map and sharded states remap global qubits,
 * so after qj_apply_circuit(QJ_FUSE) or on sharded states the amplitude
 * buffer may hold the state in a permuted bit order (qj_probabilities is
 * canonical regardless).  qj_state_canonicalize moves the data back to the
 * canonical order (R1) with SWAP passes / exchanges (two global bits trade
 * places by three exchanges through the top local bit) and resets the map. */
qj_status qj_state_canonicalize(qj_state s);

/* The current logical->physical map: phys[q] (n ints, caller-owned host
 * memory) receives the bit of the global index (local bits first, then the
 * global / shard bits) that holds qubit q; canonical = n-1-q.  Host-only
 * read, no synchronisation.  Errors: INVALID_ARG (NULL). */
qj_status qj_state_layout(qj_state s, int* phys);

/* ---- readout -----------------------------------------------------------------
 * Born-rule probabilities.  qubits == NULL and nq == -1:
 * the full vector |psi_i|^2 in canonical index order (2^n values).  Otherwise
 * the marginal over the listed qubits, first listed = most significant bit of
 * the output index (2^nq values, accumulated in fp64).  `out_dev` is caller
 * owned DEVICE memory of the state's real type (float for C64, double for
 * C128).  Virtual-rank sharded states: out_dev must hold the full output.
 * NCCL-sharded states: the full vector is distributed -- rank r's out_dev
 * receives the canonical slice [r 2^n_local, (r+1) 2^n_local); if global
 * qubits were remapped the state is first canonicalised in place
 * (qj_state_canonicalize: exchanges, collective over the ranks); marginals
 * are all-reduced and replicated on every rank. */
qj_status qj_probabilities(qj_state s, const int* qubits, int nq, void* out_dev);

/* ---- measurement ("a custom operator for collapsing and
 * re-normalizing states and a method for sampling shot frequencies based on
 * Metropolis algorithm"; R26-R28) ---------------------------------
 *
 * Outcomes are integers over the listed qubits, first listed = most
 * significant bit (the qj_probabilities convention).
 *
 * qj_collapse: P = sum |psi_i|^2 over the basis states consistent with
 * `outcome` (fp64, fixed reduction order: deterministic); if P <= 1e-14 the
 * call fails with QJ_ERR_ZERO_PROBABILITY and the state is untouched;
 * otherwise consistent amplitudes are divided by sqrt(P) and all others set to
 * 0, in place.  `prob_out` (host, may be NULL) receives P.
 * Synchronises the handle's stream once (P is checked on the host).  Works on
 * remapped, virtual-sharded and NCCL-sharded states (P is all-reduced).
 * Errors: INVALID_ARG (NULL, nq < 1, outcome >= 2^nq), INDEX_OUT_OF_RANGE,
 * OVERLAPPING_QUBITS, ZERO_PROBABILITY. */
qj_status qj_collapse(qj_state s, const int* qubits, int nq, uint64_t outcome, double* prob_out);

typedef enum {
    QJ_SAMPLE_DIRECT = 0,          /* exact inverse CDF (2^-60 fixed point, R27)      */
    QJ_SAMPLE_METROPOLIS = 1,      /* Metropolis chains, uniform proposal (R28)       */
    QJ_SAMPLE_METROPOLIS_FLIP = 2  /* Metropolis chains, single-bit-flip proposal     */
} qj_sample_method;

#define QJ_AUTO UINT64_MAX

typedef struct {
    int method;        /* qj_sample_method                                         */
    uint32_t nchains;  /* Metropolis: independent chains; 0 = min(nshots, 4096)   */
    uint64_t burnin;   /* Metropolis: steps per chain before recording; QJ_AUTO =
                          max(100, ceil(ceil(nshots / nchains) / 10))              */
} qj_sample_opts;

/* Draw `nshots` outcomes from the distribution `probs_dev` (DEVICE, 2^nbits
 * fp64 weights, need not be normalised; negative / NaN entries count as 0;
 * the direct method needs their sum < 15.5 -- its CDF is 2^-60 fixed point --
 * and returns INVALID_ARG otherwise, e.g. for raw histogram counts) with the counter-based generator Philox4x32-10 keyed by `seed`:
 * shot i of the direct method uses counter (i mod 2^32, i >> 32, 0, 0) (R27), chain c
 * step t of Metropolis uses counter (t, c, 1, 0) (R28), so results depend only
 * on (probs, nshots, seed, opts), never on the device or launch shape.
 * Outputs (DEVICE, each may be NULL, not both): samples_dev[nshots] int64
 * outcomes (Metropolis: chain c's shots contiguous at offset
 * c*floor(nshots/C) + min(c, nshots mod C)); counts_dev[2^nbits] uint64
 * frequencies, ADDED to (zero it first).  opts NULL = direct.  Work is
 * enqueued on `stream` (cudaStream_t, NULL = legacy default).  The direct
 * method synchronises once to check the total (ZERO_PROBABILITY if 0) and
 * allocates its CDF scratch (8 (2^nbits + 2^nbits/4096 + 1) bytes) stream-
 * ordered.  Errors: INVALID_ARG (nshots == 0, NULL outputs, bad opts),
 * CAPACITY (nbits > 34, Metropolis burnin + shots per chain >= 2^32 - 1),
 * ZERO_PROBABILITY. */
qj_status qj_sample_distribution(const double* probs_dev, int nbits, uint64_t nshots, uint64_t seed,
                                 const qj_sample_opts* opts, int64_t* samples_dev, uint64_t* counts_dev,
                                 void* stream);

/* Shots over the marginal of the listed qubits of the state (the fp64 bins
 * of qj_probabilities, all-reduced across NCCL ranks; nq <= 30), then
 * qj_sample_distribution on the handle's stream with the handle's scratch.
 * The state is not modified.  Bins come from fp64 atomics, so their last
 * bit may differ between runs; a draw can change only when that moves a
 * decision boundary (probability ~1e-16 per draw). */
qj_status qj_sample(qj_state s, const int* qubits, int nq, uint64_t nshots, uint64_t seed,
                    const qj_sample_opts* opts, int64_t* samples_dev, uint64_t* counts_dev);

/* One projective measurement of the listed qubits: draw one outcome with the
 * direct method (shot 0 of `seed`), then qj_collapse onto it.  `outcome_out`
 * (host) receives it, `prob_out` (host, may be NULL) its probability. */
qj_status qj_measure(qj_state s, const int* qubits, int nq, uint64_t seed, uint64_t* outcome_out,
                     double* prob_out);

/* Block until all work enqueued on the handle has finished; reports
 * asynchronous CUDA errors. */
qj_status qj_sync(qj_state s);

/* ---- introspection -------------------------------------------------------- */
typedef struct {
    uint64_t launches;       /* kernels launched by the library                  */
    uint64_t passes;         /* state passes (gate or fused window passes)       */
    uint64_t exchanges;      /* global<->local qubit swaps (sharded states)      */
    double alg_bytes;        /* algorithmic HBM bytes of all passes (C15)        */
    double exchange_bytes;   /* bytes moved by exchanges                          */
} qj_counters;

qj_status qj_get_counters(qj_state s, qj_counters* out, int reset);

/* Per-kernel-kind timing: with profiling on, the library records a pair of
 * CUDA events on the handle's stream around every pass it enqueues.
 * qj_get_profile synchronises the stream and returns, per pass kind
 * ("gate_dense", "gate_x", "gate_swap", "diag_table", "diag_phase",
 * "diag_neg", "tile", "exchange"), the number of launches, their summed
 * device time and their summed algorithmic bytes.  `count` receives the
 * number of entries written (<= max_entries).  `reset` bit 0: clear the
 * records afterwards; bit 1: return one entry per recorded launch instead,
 * in enqueue order (launches = 1). */
typedef struct {
    char name[32];
    uint64_t launches;
    double total_ms;
    double alg_bytes;
} qj_profile_entry;

qj_status qj_set_profiling(qj_state s, int on);
qj_status qj_get_profile(qj_state s, qj_profile_entry* out, int max_entries, int* count, int reset);

/* n, local qubits, dtype, number of shards of the handle. */
qj_status qj_state_info(qj_state s, int* n, int* n_local, int* dtype, int* nshards);

/* Thread-local message describing the last failure ("" if none). */
const char* qj_last_error(void);

/* Library version string. */
const char* qj_version(void);

/* ---- host-side planning (no GPU needed; exported for CPU tests) -------------
 * qj_plan_circuit runs the same planner qj_apply_circuit uses on a state of
 * n qubits split in `nshards` shards (a power of two; global qubits = top
 * log2(nshards) bits) and returns its steps: per-shard passes on physical
 * local bit positions, and EXCHANGE steps (global bit `gbit` <-> local bit
 * `lbit`).  Gate data are read as complex128.  `phys` (n ints, may be NULL)
 * receives the final logical->physical bit map.  Fused (TILE) steps are
 * reported with type 2 and no payload; with QJ_FUSE on one shard of n <= 13 (c128) / 14 (c64) qubits, runs of gates are reported as type 3 (one whole-state shared-memory program, no payload).  Errors: INVALID_ARG / INDEX / OVERLAP
 * as qj_apply_circuit, CAPACITY if more than max_steps steps, UNSUPPORTED for
 * dense payloads larger than 4 targets. */
typedef struct {
    int type;                   /* 0 = pass, 1 = exchange, 2 = tile, 3 = small */
    int shard;                  /* global shard index the pass runs on            */
    int kind;                   /* 0 dense, 1 x, 2 swap, 3 diag, 4 phase, 5 neg    */
    int k;                      /* number of targets                              */
    int tpos[QJ_MAX_TARGETS];   /* target bit positions, matrix order (MSB first) */
    int nfix;                   /* fixed bits: controls / phase pattern           */
    int fpos[64];
    int fval[64];
    uint32_t touch;             /* dense: touched-member mask (listed order)      */
    int nm;                     /* complex values in m                            */
    double m[2 * 256];          /* dense 4^k / diag 2^k / phase 1 (interleaved)   */
    int gbit, lbit;             /* exchange                                       */
    double alg_bytes;
} qj_plan_step;

qj_status qj_plan_circuit(int n, int nshards, int amp_bytes, const qj_gate* gates, int ngates,
                          uint32_t flags, qj_plan_step* out, int max_steps, int* nsteps, int* phys);

/* The steps qj_state_canonicalize runs on a state of n qubits in `nshards`
 * shards whose logical->physical map is phys_in (n ints, a permutation):
 * SWAP passes for local pairs (one per shard index), exchanges for
 * local/global and global/global pairs; afterwards qubit q is at bit n-1-q.
 * Host only.  Errors: INVALID_ARG (NULL, nshards not a power of two, phys_in
 * not a permutation), CAPACITY (too many shards for n, > max_steps steps). */
qj_status qj_plan_canonicalize(int n, int nshards, const int* phys_in, qj_plan_step* out, int max_steps,
                               int* nsteps);

/* Tooling (host only, no GPU): plan the circuit with QJ_FUSE on one shard of
 * n qubits (amp_bytes 16 = complex128, 8 = complex64), emit the source of
 * every tile-pass kernel the JIT would compile (written as dir/qj_tile_K.cu
 * when dir != NULL) and, with compile != 0, compile each with NVRTC for
 * sm_100a.  *nkernels receives the number of tile passes.  Errors: as
 * qj_plan_circuit; UNSUPPORTED with the NVRTC log on a compile failure. */
qj_status qj_debug_tile_sources(int n, int amp_bytes, const qj_gate* gates, int ngates, uint32_t flags,
                                const char* dir, int compile, int* nkernels);

/* Tooling: run the NCCL exchange machinery (pipelined grouped send / recv
 * through the staging ring, pack / unpack kernels, two streams) with this
 * rank as its own partner on the half of its shard whose `local_bit` is 1.
 * The state must come back unchanged; used to exercise the multi-GPU data
 * path on one GPU.  Errors: INVALID_ARG (not an NCCL state), INDEX, NCCL, CUDA. */
qj_status qj_debug_nccl_self_exchange(qj_state s, int local_bit);

/* The paper's gate fusion (Table 2 Gates* / Depth*), host
 * only: greedily combine the circuit into gates of at most `max_qubits` (1 to
 * 5; the paper's fusion is 2) qubits.  Fused groups come back as
 * QJ_GATE_DENSE gates whose matrices (complex128, row-major, first target =
 * MSB) are written to `mats` (caller buffer of 2 * 4^max_qubits doubles per
 * output gate: 32 for the paper's 2) and pointed to by `data`; gates on more
 * qubits are copied unchanged (their `data` still points at the caller's
 * input).  Gate data are read as complex128.  Errors: as qj_apply_circuit,
 * CAPACITY if more than max_out gates. */
qj_status qj_fuse_circuit(int n, const qj_gate* in, int nin, int max_qubits, qj_gate* out, double* mats,
                          int max_out, int* nout, int* src /* max_out, may be NULL: input index or -1 */);

/* The exchange rule of the multi-GPU layer: for a swap of global bit `gbit`,
 * rank `rank` trades with `*peer` the amplitudes of its shard whose swapped
 * local bit equals `*half_bit`. */
void qj_exchange_peer(int rank, int gbit, int* peer, int* half_bit);

/* Host-side index math used by every pass (exported for exhaustive CPU
 * tests): insert a 0 bit at each of the `npos` ascending bit positions
 * `sorted_pos` into g (PAPER.md:221-227 listing, i1 = ((g>>m)<<(m+1)) + (g & (k-1))). */
uint64_t qj_insert_zero_bits(uint64_t g, const int* sorted_pos, int npos);

#ifdef __cplusplus
}
#endif

#endif /* QJ_H */
