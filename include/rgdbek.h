/*
 * rgdbek.h — C ABI of the B200-native RGDBEK hot path (arXiv 2509.19267).
 *
 * The operation: solve A x = b, A in R^{m x n}, b in R^m (PAPER.md P:38-41,
 * eq:Ax=b) with the randomized greedy double-block extended Kaczmarz sweep of
 * Algorithm 1, in the pseudoinverse-free form BASELINE.json's
 * north_star prescribes (reading R1):
 *
 *   x_0 = 0, z_0 = b
 *   for k = 0, 1, ...
 *     s = A^T z_k;  eps^z_j = s_j^2 / ||A_(j)||^2
 *     U_k = the k_c indices with the smallest Philox exponential keys
 *           -ln(u_j)/eps^z_j  (sampling "n eta columns using P(j_k)")
 *     zeta = s on U_k;  w = A zeta;  z_{k+1} = z_k - (||zeta||^2/||w||^2) w
 *     r = b - z_{k+1} - A x_k;  eps^x_i = r_i^2 / ||A^(i)||^2
 *     J_k = the k_r smallest row keys ("m eta rows using P(i_k)")
 *     xi = r on J_k;  v = A^T xi;  x_{k+1} = x_k + (||xi||^2/||v||^2) v
 *   stop on RSE = ||A x - b||^2/||b||^2 <= tol, or on
 *   ||x - x*||/||x*|| <= tol (BASELINE.json metric), or on the iteration cap.
 *
 * with k_c = max(1, floor(eta n + 1/2)) and k_r = max(1, floor(eta m + 1/2))
 * clamped to the number of positive scores, and the Philox4x32-10 stream
 * u(seed, k, step, index) defined in DESIGN.md §2 (readings R2-R6).
 *
 * Conventions
 *  - All floating point is IEEE binary64 (double); indices are int32 (column
 *    and row indices) and int64 (CSR row offsets, sizes, iteration counts).
 *  - Pointers passed IN may be host or device (CUDA unified addressing; torch
 *    CUDA tensors pass data_ptr()).  create() deep-copies A and b into device
 *    memory owned by the handle; the library never keeps a caller pointer.
 *    get_*() write into caller buffers (host or device).
 *  - Every call returns an rgdbek_status; negative = error.  The message of
 *    the last error is rgdbek_last_error(handle) (or (NULL) for create
 *    failures, thread-local).  CUDA / NCCL errors are sticky: once one is
 *    seen every later call on that handle returns the same code.
 *  - A handle is not thread-safe; distinct handles are independent.  All work
 *    runs on options.stream (or a library stream); calls that return results
 *    synchronise that stream before returning.
 *  - Multi-GPU: each rank creates its handle with the GLOBAL m, n, its own
 *    contiguous global row range [row_begin, row_end) and its local rows of A
 *    and b (column indices global), plus either an ncclComm_t in
 *    options.nccl_comm (the NCCL graph engine: x replicated) or no communicator
 *    (the peer-memory sharded engine, see rgdbek_peer_connect / rgdbek_group_create).
 *    z (local rows) is sharded.  Results are identical on every rank.
 *  - No CPU fallback exists: without a usable sm_100 GPU create() fails with
 *    RGDBEK_E_CUDA.
 */
#ifndef RGDBEK_H_
#define RGDBEK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGDBEK_ABI_VERSION 1

typedef struct rgdbek_ctx* rgdbek_handle;
typedef struct rgdbek_group_s* rgdbek_group;    /* emulated ranks on one GPU (peer-sharded) */
#define RGDBEK_PEER_HANDLE_BYTES 64             /* cudaIpcMemHandle_t */
#define RGDBEK_MAX_PEER_RANKS 8

typedef enum {
  RGDBEK_OK = 0,
  RGDBEK_E_ARG = -1,        /* NULL pointer, eta not in (0,1), tol <= 0, n_iter < 0, ...      */
  RGDBEK_E_DIM = -2,        /* m, n < 1, row range outside [0, m), inconsistent lengths         */
  RGDBEK_E_CSR = -3,        /* row_ptr[0] != 0, non-monotone, row_ptr[m] != nnz, col >= n or
                               < 0, columns not strictly increasing within a row               */
  RGDBEK_E_ZERO_RHS = -4,   /* ||b|| == 0: RSE undefined                            */
  RGDBEK_E_NONFINITE = -5,  /* NaN / Inf in A or b                                              */
  RGDBEK_E_STATE = -6,      /* e.g. STOP_REL_ERR without rgdbek_set_reference                   */
  RGDBEK_E_CUDA = -7,       /* CUDA runtime error or no sm_100 device (sticky)                  */
  RGDBEK_E_NCCL = -8,       /* NCCL error (sticky)                                              */
  RGDBEK_E_OOM = -9,        /* device allocation failed                                         */
  RGDBEK_E_INTERNAL = -10   /* a device self-check failed (e.g. block size mismatch)            */
} rgdbek_status;

typedef enum {              /* rgdbek_result.outcome (SPEC exit codes 0/2/3)                    */
  RGDBEK_CONVERGED = 0,
  RGDBEK_MAX_ITER = 2,
  RGDBEK_STALLED = 3        /* both blocks empty (no positive score mass) before the stop test */
} rgdbek_outcome;

typedef enum {
  RGDBEK_STOP_RSE = 0,      /* ||A x - b||^2 / ||b||^2 <= tol (the paper's RSE)      */
  RGDBEK_STOP_REL_ERR = 1,  /* ||x - x*|| / ||x*|| <= tol, x* from rgdbek_set_reference          */
  RGDBEK_STOP_NONE = 2      /* iterate to the cap                                               */
} rgdbek_stop;

typedef struct {
  double  eta;              /* block fraction, in (0,1); default 0.5                    */
  int32_t stop;             /* rgdbek_stop used by rgdbek_solve; default RGDBEK_STOP_RSE        */
  int32_t device;           /* CUDA ordinal; default 0                                          */
  void*   stream;           /* cudaStream_t to run on (must outlive the handle); NULL = a
                               library-owned stream                                            */
  void*   nccl_comm;        /* ncclComm_t; NULL = single GPU                                    */
  int64_t row_begin;        /* this rank's first global row; -1 (default) = 0                   */
  int64_t row_end;          /* one past this rank's last global row; -1 (default) = m          */
  int32_t symmetric;        /* 1 = caller asserts A == A^T (square CSR); the CSR then also
                               serves as the transposed copy.  Verified at create.             */
  int32_t trace_capacity;   /* per-iteration records kept on device (ring); default 4096       */
} rgdbek_options;

typedef struct {
  int32_t outcome;          /* rgdbek_outcome                                                   */
  int32_t pad_;
  int64_t iters;            /* total iterations k of the returned iterate x_k                   */
  double  rse;              /* RSE(x_k) = ||A x_k - b||^2 / ||b||^2                              */
  double  rel_err;          /* ||x_k - x*|| / ||x*|| (NaN without a reference)                  */
  double  seconds;          /* device time of the call (CUDA events on the handle's stream)    */
} rgdbek_result;

typedef struct {            /* what iteration k produced (trace ring, rgdbek_get_trace)         */
  int64_t  k;
  int64_t  kp;              /* |U_k|                                                            */
  uint64_t hash_u;          /* sum of splitmix64(j) over j in U_k, mod 2^64                     */
  double   Z;               /* ||zeta||^2                                                       */
  double   W;               /* ||A zeta||^2                                                     */
  int64_t  kpp;             /* |J_k|                                                            */
  uint64_t hash_j;          /* sum of splitmix64(i) over GLOBAL rows i in J_k                   */
  double   X;               /* ||xi||^2                                                         */
  double   V;               /* ||A^T xi||^2                                                     */
  double   rse;             /* RSE(x_{k+1})                                                     */
} rgdbek_trace_record;

int32_t       rgdbek_abi_version(void);
void          rgdbek_options_default(rgdbek_options* opts);

/* Create from CSR rows [row_begin, row_end) of A (m_local = row_end - row_begin rows):
 * row_ptr_local[m_local+1] (int64, row_ptr_local[0] == 0), col_idx[nnz_local] (int32, global
 * column ids, strictly increasing within each row), val[nnz_local], b_local[m_local]. */
rgdbek_status rgdbek_create_csr(rgdbek_handle* out, int64_t m, int64_t n, int64_t nnz_local,
                                const int64_t* row_ptr_local, const int32_t* col_idx,
                                const double* val, const double* b_local,
                                const rgdbek_options* opts);

/* Create from a dense row-major block of rows: A_local[i*lda + j], lda >= n. */
rgdbek_status rgdbek_create_dense(rgdbek_handle* out, int64_t m, int64_t n,
                                  const double* A_local, int64_t lda, const double* b_local,
                                  const rgdbek_options* opts);

/* x = 0, z = b, k = 0, sampler seed = seed. */
rgdbek_status rgdbek_reset(rgdbek_handle h, uint64_t seed);

/* Exactly n_iter more iterations from the current state, no stop test.
 * result->rse is RSE of the final iterate. */
rgdbek_status rgdbek_step(rgdbek_handle h, int64_t n_iter, rgdbek_result* result);

/* reset(seed), then iterate until the stop test (options.stop / rgdbek_set_stop) holds
 * after an iteration, both blocks are empty (STALLED), or max_iter iterations ran. */
rgdbek_status rgdbek_solve(rgdbek_handle h, double tol, int64_t max_iter, uint64_t seed,
                           rgdbek_result* result);

rgdbek_status rgdbek_set_stop(rgdbek_handle h, int32_t stop);

/* Update mode.  mode 0 (default): the pseudoinverse-free block updates
 * of BASELINE.json's north_star.  mode 1: Algorithm 1's exact projections
 *   z_{k+1} = z_k - A_U A_U^+ z_k,  x_{k+1} = x_k + (A^J)^+ (b^J - z^J - A^J x_k),
 * realised by inner CGLS iterations (minimum-norm, from 0) on the masked operators
 * — the Krylov solvers equivalent to the paper's LSQR — each stopped when its
 * residual has dropped by inner_tol (relative) or after inner_max iterations.  mode 1 needs the
 * single-GPU persistent engine (RGDBEK_E_STATE otherwise). */
rgdbek_status rgdbek_set_mode(rgdbek_handle h, int32_t mode, double inner_tol, int32_t inner_max);

/* Block selection rule.  0 (default): RGDBEK's randomized sampling of
 * eta*n columns / eta*m rows with P(j) proportional to the residual scores (P:93-100,
 * Alg. 1 lines 4-7 and 9-12).  1: GDBEK's greedy threshold sets
 *   U = {j : eps^z_j >= eta * max eps^z},  J = {i : eps^x_i >= eta * max eps^x}
 * (no sampling; block sizes vary).  Combine with rgdbek_set_mode(1) for GDBEK's
 * pseudoinverse updates (eq:updateGDBEK).  Needs the single-GPU persistent engine. */
rgdbek_status rgdbek_set_selection(rgdbek_handle h, int32_t selection);

/* The paper's parallel Algorithm 2 (alg:rgdbek_bsas) on ONE
 * GPU with `processes` logical processes P in [1, 8]: the rows are split into P
 * contiguous blocks [floor(m p/P), floor(m (p+1)/P)); every iteration samples one global
 * column set U from A^T z, lets each process take its own first-Krylov
 * z-step on its rows and sample round(eta d_p) of its own rows,
 * and applies the lazily averaged x-update x += (1/P) sum_p (X_p/V_p) (A^(p))^T xi_p
 * — the pseudoinverse-free reading R28 of DESIGN.md.  P = 1 is Algorithm 1.
 * processes = 0 returns to Algorithm 1.  Needs a dense A on the single-GPU persistent
 * engine, the pseudoinverse-free update and random selection (RGDBEK_E_STATE otherwise),
 * and at most 32768 rows per process (RGDBEK_E_ARG).  The persistent grid is rounded
 * down to a multiple of P (each process is a run of G/P CTAs).  Traces report the sums
 * over processes of Z_p, W_p, X_p, V_p and |J| = sum_p |J_p|. */
rgdbek_status rgdbek_set_lazy(rgdbek_handle h, int32_t processes);
rgdbek_status rgdbek_set_reference(rgdbek_handle h, const double* xstar /* n values */);

rgdbek_status rgdbek_get_x(rgdbek_handle h, double* out_n);
rgdbek_status rgdbek_get_z(rgdbek_handle h, double* out_local_m);

/* Blocks of the last completed iteration (k-1): sizes and order-free hashes from the trace.
 * U / J may be NULL.  Non-NULL U / J (host or device int32 buffers of n and m_local entries)
 * receive the sorted indices (U: columns, n_u values; J: GLOBAL rows of this rank, n_j
 * values) and need rgdbek_set_capture(h, 1) before the iterations ran (RGDBEK_E_STATE
 * otherwise).  Sharded: n_j is this rank's share of J when J is requested. */
rgdbek_status rgdbek_get_blocks(rgdbek_handle h, int64_t* n_u, uint64_t* hash_u, int32_t* U,
                                int64_t* n_j, uint64_t* hash_j, int32_t* J);

/* Copies up to max_records trace records of iterations [max(0, k - cap), k) in order. */
rgdbek_status rgdbek_get_trace(rgdbek_handle h, rgdbek_trace_record* out, int64_t max_records,
                               int64_t* n_out);

/* Resume from a saved state: x (n), z_local, iteration k (the seed stays). */
rgdbek_status rgdbek_set_state(rgdbek_handle h, const double* x, const double* z_local, int64_t k);

/* Timing hook for the bench: enqueue `reps` launches of one hot kernel on the handle's stream
 * (kernel 0 = pass T [A^T z, A^T xi], 1 = pass N [A zeta, A x]).  Clobbers the iteration
 * state: call rgdbek_reset afterwards.  bytes_per_launch receives the algorithmic bytes. */
rgdbek_status rgdbek_launch_kernel(rgdbek_handle h, int32_t kernel, int32_t reps,
                                   double* bytes_per_launch);

/* Kernels launched per iteration body of the graph engine (for the bench's gpu_launches
 * count); 0 for the persistent engine, which is one launch per rgdbek_step/solve call. */
rgdbek_status rgdbek_launches_per_iteration(rgdbek_handle h, int64_t* out);

/* Diagnostics.  rgdbek_phase_times: accumulated device time (ns, %globaltimer read by CTA 0
 * after each grid barrier) of the persistent engine's phases, when the handle was
 * created with RGDBEK_PHASE_TIMING=1 in the environment; *n_out = 0 otherwise.  Up to 24
 * entries: ids 0..15 are times, 16..17 event counts.
 * Phase ids: 1 pass T, 2 s/v + column keys, 3-4 column selection levels, 5 mask + x update,
 * 6 pass N, 7 stop test + z update + row keys, 8-9 row selection levels, 10 row mask,
 * 0 bookkeeping, 11-12 dense column sums / flush, 13-14 local column selection (level 1,
 * levels 2-3 + rank), 15 local row selection; 16 / 17 = number of local column / row
 * selections that overflowed the shared-memory candidate list.  rgdbek_engine_info: engine 0 = persistent kernel (ctas = its grid),
 * 1 = multi-kernel CUDA graph (RGDBEK_ENGINE=graph). */
rgdbek_status rgdbek_phase_times(rgdbek_handle h, double* out_ns, int32_t max_phases,
                                 int32_t* n_out);
rgdbek_status rgdbek_engine_info(rgdbek_handle h, int32_t* engine, int32_t* ctas);
/* Full passes over A executed by the persistent engine since the last reset (2 per
 * iteration in mode 0; 2 + 2 per inner iteration in mode 1). */
rgdbek_status rgdbek_get_counters(rgdbek_handle h, int64_t* passes);
/* Exact mode (mode 1): algorithmic bytes of A read since the last reset — full passes
 * count all of A, the dense x-solve's row-masked passes only the |J| rows of A^J. */
rgdbek_status rgdbek_get_a_bytes(rgdbek_handle h, double* bytes);

/* Block capture (test / diagnostics; SURVEY §8(c) parity protocol "full lists"): with
 * enable = 1 every later iteration also writes one byte per column and per local row
 * marking U_k and J_k (2 x (n + m_local) bytes of device memory, allocated on first use),
 * so rgdbek_get_blocks can return the index lists.  enable = 0 stops the writes. */
rgdbek_status rgdbek_set_capture(rgdbek_handle h, int32_t enable);

/* Selection path counters since create, out4[4]: [0] CTA-local selections whose level-1
 * bucket overflowed the shared-memory candidate list (fallback: rescans of all keys),
 * [1] selections finished by the persistent engine's exact slow path (candidate or
 * survivor overflow), [2] selections finished by the graph engine's k_select_slow,
 * [3] reserved (0). */
rgdbek_status rgdbek_selection_stats(rgdbek_handle h, int64_t* out4);

/* Compile-time geometry of this build (no device needed).  out[i] for i <
 * min(max_entries, RGDBEK_BUILD_INFO_COUNT): 0 TILE_NNZ (nonzeros per sparse tile),
 * 1 TILE_ROWS, 2 LOCAL_SEL_MAX (selections over <= this many keys run CTA-locally),
 * 3 LCAND_CAP, 4 CAND_CAP, 5 FINAL_CAP (selection candidate capacities), 6 threads per
 * persistent CTA, 7 threads per tile worker group.  Returns the number written
 * (RGDBEK_BUILD_INFO_COUNT when out == NULL). */
#define RGDBEK_BUILD_INFO_COUNT 8
int32_t       rgdbek_build_info(int32_t* out, int32_t max_entries);

/* The cudaStream_t the handle runs on (for events / synchronisation). */
void*         rgdbek_stream(rgdbek_handle h);

/* ---------------------------------------------------------------------------------------
 * Peer-memory sharded engine: Algorithm 1 row-sharded over R
 * ranks as ONE persistent kernel per rank, ranks exchanging through peer memory (NVLink P2P
 * loads / stores and release/acquire flag words), no NCCL calls.  A rank is a handle created
 * with a partial row range [row_begin, row_end) and NO options.nccl_comm; global m, n, GLOBAL
 * column ids.  Rank r's rows touch the column window W_r (min .. max column of its rows; all
 * columns for dense A); every column is owned by one rank (rgdbek_plan_ownership), whose
 * copy of s = A^T z (summed over the ranks whose window holds the column), keys, zeta and x
 * is authoritative; the non-owned window columns of zeta and x (the halo) are read from
 * their owners each iteration.  Trajectories do not depend on R (global Philox indices).
 * Supported: the pseudoinverse-free update, random selection (RGDBEK_E_STATE otherwise).
 * Sharded get_x gathers the owned parts of every rank; get_z is the rank's rows; get_blocks
 * index lists are the rank's OWNED columns of U and its rows of J.
 * ------------------------------------------------------------------------------------- */

/* Owned-column boundaries for R ranks whose windows are windows[2r], windows[2r+1]
 * (half-open): owned_bounds[0..R], owned_bounds[0] = 0, owned_bounds[R] = n.  Window
 * starts and ends strictly increasing in r (banded A): each boundary splits the overlap of
 * neighbouring windows at its midpoint (the halo exchange is then the overlap); otherwise
 * (e.g. dense A, every window [0, n)) equal column slices.
 * Host-only (no device needed). */
rgdbek_status rgdbek_plan_ownership(int32_t nranks, const int64_t* windows, int64_t n,
                                    int64_t* owned_bounds);

/* out4 = {window begin, window end, first global row, one past the last row} of a rank. */
rgdbek_status rgdbek_peer_window(rgdbek_handle h, int64_t* out4);

/* R ranks on ONE GPU (emulated multi-GPU, e.g. for P-invariance tests): handles[r] are the
 * ranks in row order (contiguous ranges covering [0, m), same device, m, n, storage).  The
 * group runs ONE cooperative launch of R x G CTAs (G = SMs / R), so ranks that wait on one
 * another are co-resident.  While grouped, rgdbek_step / rgdbek_solve on a member return
 * RGDBEK_E_STATE; the per-rank getters work as documented above. */
rgdbek_status rgdbek_group_create(rgdbek_group* out, const rgdbek_handle* handles, int32_t nranks);
rgdbek_status rgdbek_group_reset(rgdbek_group g, uint64_t seed);
rgdbek_status rgdbek_group_step(rgdbek_group g, int64_t n_iter, rgdbek_result* result);
rgdbek_status rgdbek_group_solve(rgdbek_group g, double tol, int64_t max_iter, uint64_t seed,
                                 rgdbek_result* result);
void          rgdbek_group_destroy(rgdbek_group g);

/* R real GPUs, one process per GPU: every rank exports its exchange block
 * (RGDBEK_PEER_HANDLE_BYTES, a CUDA IPC handle), the caller allgathers the handles and the
 * windows (rgdbek_peer_window) over its process group, and every rank calls
 * rgdbek_peer_connect with them (handles: nranks x RGDBEK_PEER_HANDLE_BYTES, windows:
 * 2 x nranks).  Afterwards rgdbek_step / rgdbek_solve are collectives: every rank must make
 * the same call (its kernel waits on the others' flag words). */
rgdbek_status rgdbek_peer_export(rgdbek_handle h, void* out_handle);
rgdbek_status rgdbek_peer_connect(rgdbek_handle h, int32_t nranks, int32_t rank,
                                  const void* handles, const int64_t* windows);

/* ---------------------------------------------------------------------------------------
 * Several right-hand sides sharing A (the paper's 3-channel deblurring
 * solves A x_i = b_i with one blur operator).  nrhs <= 4 independent Algorithm-1
 * solves (reading R29): right-hand side q has its own z, x, blocks and Philox
 * stream with seed + q, so it follows exactly the single-RHS solve of (A, b_q, seed + q);
 * every pass over A serves all of them.  b_all holds nrhs vectors of m values, RHS-major
 * (b_all[q * m + i]).  Sparse A, one GPU, all rows; pseudoinverse-free update and random
 * selection (RGDBEK_E_STATE otherwise).  rgdbek_step / rgdbek_solve run all right-hand
 * sides together; solve stops when every right-hand side meets the stop test (or stalls),
 * or at max_iter.  The rgdbek_result and the plain getters describe right-hand side 0;
 * the *_rhs calls address right-hand side `rhs` (RGDBEK_E_ARG outside [0, nrhs)).
 * STOP_REL_ERR needs rgdbek_set_reference_rhs for every right-hand side. */
rgdbek_status rgdbek_create_csr_multi(rgdbek_handle* out, int64_t m, int64_t n, int64_t nnz,
                                      const int64_t* row_ptr, const int32_t* col_idx,
                                      const double* val, const double* b_all, int32_t nrhs,
                                      const rgdbek_options* opts);
int32_t       rgdbek_rhs_count(rgdbek_handle h);
rgdbek_status rgdbek_get_x_rhs(rgdbek_handle h, int32_t rhs, double* out_n);
rgdbek_status rgdbek_get_z_rhs(rgdbek_handle h, int32_t rhs, double* out_m);
rgdbek_status rgdbek_set_reference_rhs(rgdbek_handle h, int32_t rhs, const double* xstar);
rgdbek_status rgdbek_get_trace_rhs(rgdbek_handle h, int32_t rhs, rgdbek_trace_record* out,
                                   int64_t max_records, int64_t* n_out);

/* NCCL bootstrap helpers (rank 0 makes the id; it is broadcast by the caller). */
rgdbek_status rgdbek_nccl_unique_id(void* out_128_bytes);
rgdbek_status rgdbek_nccl_comm_init(void** comm_out, int32_t nranks, int32_t rank,
                                    const void* id_128_bytes, int32_t device);
rgdbek_status rgdbek_nccl_comm_destroy(void* comm);

const char*   rgdbek_last_error(rgdbek_handle h);
/* Frees the handle.  Its device memory goes back to the device's stream-ordered memory pool
 * (cudaFreeAsync on the handle's stream, which is synchronised; a caller-supplied
 * options.stream must therefore still be valid here), where the next create of the process
 * reuses it; NULL is a no-op. */
void          rgdbek_destroy(rgdbek_handle h);

#ifdef __cplusplus
}
#endif
#endif /* RGDBEK_H_ */
