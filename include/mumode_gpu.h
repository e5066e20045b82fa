/* mumode_gpu.h -- C-ABI of the B200 (sm_100a) mu-mode product / Tucker engine.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * (arXiv 2112.11238's mu-mode BLAS, /root/reference/proj). The reference is
 * header-only C++ whose only compiled seam is la::gemm_raw
 * (proj/include/mumode/gemm.hpp:15-18, proj/src/gemm.cpp:53-66); replacing
 * that seam alone would keep the host permutes, so this ABI sits one level up,
 * at the operators themselves. Each entry point names the reference interface
 * it replaces.
 *
 * Conventions (identical to the reference, proj/include/mumode/shape.hpp:68-77,
 * matrix.hpp:14):
 *   - tensors are column-major, first index fastest; extents are int64
 *     (the reference's int32 GEMM casts, src/gemm.cpp:55-57, do not apply);
 *   - modes are 1-based (shape.hpp:91-95);
 *   - a factor matrix L_mu is column-major with ld = rows. Forward products
 *     use L_mu as n_mu x m_mu; adjoint (cttucker) products use L_mu^H, so the
 *     stored L_mu is m_mu x n_mu (tucker.hpp:73);
 *   - complex128 data is interleaved (re, im) doubles (std::complex<double>).
 *
 * Device entry points take caller-owned DEVICE pointers, run stream-ordered on
 * the handle's stream and do not allocate after the first call with a given
 * shape (the handle owns workspace and TMA descriptors). Host entry points
 * (mumode_host_*) take HOST pointers and include the host<->device copies; they
 * are what the reference-shaped C++ API (include/mumode_b200/mumode.hpp) calls.
 *
 * Errors: every call returns a status; the message is mumode_last_error()
 * (thread-local). MUMODE_ERR_SIZE carries the reference's SizeError text,
 * naming the offending mode ("... mode 2 ..."), MUMODE_ERR_ARGUMENT the
 * ArgumentError text (errors.hpp:8-26).
 */
#ifndef MUMODE_GPU_H
#define MUMODE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mumode_status {
  MUMODE_OK = 0,
  MUMODE_ERR_SIZE = 1,      /* reference SizeError      (errors.hpp:8-11)  */
  MUMODE_ERR_ARGUMENT = 2,  /* reference ArgumentError  (errors.hpp:13-16) */
  MUMODE_ERR_CUDA = 3,
  MUMODE_ERR_NCCL = 4,
  MUMODE_ERR_OOM = 5,
  MUMODE_ERR_CONTRACT = 6,  /* reference ContractError  (errors.hpp:23-26) */
  MUMODE_ERR_NUMERICAL = 7  /* reference NumericalError (errors.hpp:18-21) */
};

typedef struct mumode_handle_s* mumode_handle_t;

/* ---- handle ---------------------------------------------------------- */
int mumode_handle_create(mumode_handle_t* h, int device);
int mumode_handle_destroy(mumode_handle_t h);
/* cudaStream_t passed as void*, used as given (NULL = the legacy default
 * stream). A new handle starts on its own non-blocking stream. */
int mumode_set_stream(mumode_handle_t h, void* stream);
void* mumode_get_stream(mumode_handle_t h);
const char* mumode_last_error(void);
const char* mumode_version(void);
/* Number of mumode kernels launched on this handle since creation (the bench
 * reports it as gpu_launches). */
int64_t mumode_launch_count(mumode_handle_t h);
/* Kernel path selection for tests/benchmarks: 0 = auto (default),
 * 1 = force the generic SIMT kernel, 2 = force the TMA/DMMA kernel where the
 * shape allows it (tile shape by cost model), 3..6 = TMA/DMMA kernel with tile
 * configuration 0..3 forced, 7 = auto including the fused two-mode passes,
 * 8 = force the LDG-staged DMMA kernel for real products, 9 = auto with the
 * 32-wide strided-pair (tail) pass forced wherever the shape allows it,
 * 10 = auto with the tail pass disabled, 11 = auto with whole Tucker chains
 * run as one persistent launch where the tile configs allow (tma_chain.cuh),
 * 12 = auto with the fused passes' non-warp-specialised kernels
 * (fused_pair_kernel / tail_pair_kernel instead of fused_ws / tail_ws),
 * 13 = auto without the small-extent (skinny) mode-product kernel,
 * 14 = auto without the small-extent fused two-mode passes (spair.cuh),
 * 15 = auto with the small-extent fused passes wherever eligible,
 * 16 = auto with the in-place block passes (block.cuh) wherever eligible,
 * 17 = auto without the in-place block passes,
 * 18 / 19 = the 48-wide TMA tile configurations forced for real products
 *      (T-side 128 x 48 / L-side 48 x 128), 20 / 21 = the 56-wide ones,
 * 23 = itucker's real modes through the left-looking sweep kernel (22 is
 *      unused; auto takes the right-looking lu_solve_rl_kernel for n <= 408),
 * 24 = auto without that kernel's 96-fibre tiles, 25 = auto with its factor
 *      panels copied by cp.async also where bulk copies would be used,
 * 26 = kronsumv without the fused pass over its first two terms (kron12.cuh).
 * Not a fallback switch: all are CUDA kernels. */
int mumode_set_kernel_policy(mumode_handle_t h, int policy);

/* ---- device-resident operators --------------------------------------- */

/* Replaces core::mode_product (proj/include/mumode/mode_product.hpp:64-77):
 * S = T x_mu L, T with d extents m[0..d-1], L n_mu x m[mu-1]; S has m with
 * m[mu-1] replaced by n_mu. No permutation is materialised. */
int mumode_mode_product_f64(mumode_handle_t h, int d, const int64_t* m, int mu, int64_t n_mu,
                            const double* T, const double* L, double* S);
int mumode_mode_product_c128(mumode_handle_t h, int d, const int64_t* m, int mu, int64_t n_mu,
                             const double* T, const double* L, double* S);

/* Replaces ops::tucker (adjoint = 0, tucker.hpp:129-132) and ops::cttucker
 * (adjoint = 1, tucker.hpp:149-151): S = T x_1 op(L_1) ... x_d op(L_d),
 * modes applied in order 1..d. n[mu] = output extent of mode mu, i.e. rows of
 * L_mu (forward) or columns of L_mu (adjoint). */
int mumode_tucker_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                      const double* T, const double* const* L, double* S, int adjoint);
int mumode_tucker_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                       const double* T, const double* const* L, double* S, int adjoint);
/* Real tensor against a complex stack (tucker.hpp:142-144, :153-155):
 * T real, L and S complex. */
int mumode_tucker_promote(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                          const double* T, const double* const* L, double* S, int adjoint);

/* Modes mu_lo..mu_hi (1-based, inclusive) of the Tucker chain only; extents
 * of the other modes pass through. The local step of the slab-partitioned
 * Tucker (modes 1..d-1 on each rank's slab). */
int mumode_tucker_range_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int mu_lo,
                            int mu_hi);

/* Modes mu_lo..mu_hi of the Tucker chain with the LAST one's result (viewed
 * as rows x cols: rows = every extent up to mode mu_hi, cols = the extents
 * after it) scattered by row blocks: rows a_off[q]..a_off[q+1] go to
 * dst[q], a column-major (a_off[q+1]-a_off[q]) x (col0 + cols ...) matrix,
 * at column col0 + c. The TMA kernel's epilogue stores straight to dst[q]
 * (the fused exchange of mumode_dist_tucker_* with peer pointers); other
 * paths compute then copy. Forward chains. */
int mumode_tucker_range_scatter_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                    const double* T, const double* const* L, int mu_lo, int mu_hi,
                                    int P, const int64_t* a_off, int64_t col0, double* const* dst);
/* complex128: offsets and rows count complex elements; dst interleaved. */
int mumode_tucker_range_scatter_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                     const double* T, const double* const* L, int mu_lo, int mu_hi,
                                     int P, const int64_t* a_off, int64_t col0, double* const* dst);
/* Slab-transpose pack for the all-to-all: Y is A x C column-major; for each
 * destination rank q the row block Y[a_off[q]:a_off[q+1], :] is written as a
 * contiguous column-major block, blocks in rank order (a_off has P+1
 * entries, a_off[0] = 0, a_off[P] = A, P <= 64). */
int mumode_slab_pack_f64(mumode_handle_t h, int64_t A, int64_t C, int P, const int64_t* a_off,
                         const double* Y, double* send);
/* Inverse of mumode_slab_pack_f64 (send layout -> Y); the receive side of the
 * integrator's return exchange. */
int mumode_slab_unpack_f64(mumode_handle_t h, int64_t A, int64_t C, int P, const int64_t* a_off,
                           const double* send, double* Y);

/* ---- multi-GPU: slab-partitioned Tucker (SURVEY 8b "mumode_dist_tucker_f64(h,
 * comm, ...)", 8e) ---------------------------------------------------------
 * A communicator wraps an NCCL communicator (NCCL is loaded at run time,
 * libnccl.so.2) plus an exchange stream and the exchange buffers. */
typedef struct mumode_comm_s* mumode_comm_t;
/* 128-byte NCCL unique id: rank 0 creates it, the caller broadcasts it. */
int mumode_comm_unique_id(void* id_out);
int mumode_comm_create(mumode_comm_t* c, int device, const void* id, int nranks, int rank);
/* Wrap a caller-owned ncclComm_t (not destroyed by mumode_comm_destroy);
 * nccl_comm may be NULL when nranks == 1. */
int mumode_comm_wrap(mumode_comm_t* c, int device, void* nccl_comm, int nranks, int rank);
int mumode_comm_destroy(mumode_comm_t c);
/* Exchange used by mumode_dist_tucker_f64: 0 = NCCL grouped send/recv
 * (default), 1 = peer stores: the last local mode's epilogue writes every row
 * straight into the owning rank's matrix through CUDA-IPC peer pointers
 * (NVLink), then a system-scope flag handshake (csrc/slab_dist.cuh). The
 * first call per shape maps the peers (collective). */
int mumode_comm_set_exchange(mumode_comm_t c, int mode);
/* SMs the persistent compute kernels leave free while sub-slabs overlap the
 * NCCL exchange (default 16; NCCL's kernels need SMs to run beside them). */
int mumode_comm_set_overlap_sms(mumode_comm_t c, int sms);
/* A communicator WITHOUT NCCL for the peer-store exchange (mode 1 only):
 * the caller moves the CUDA-IPC handles between ranks itself --
 * mumode_comm_ipc_export writes this rank's handles for a shape
 * (mumode_comm_ipc_handle_bytes() bytes: Z[0], Z[1], flags), the caller
 * all-gathers them (any transport) and passes the P x that many bytes, in rank
 * order, to mumode_comm_ipc_import. Used to exercise the IPC mappings and the
 * epoch handshake across processes. */
int mumode_comm_create_local(mumode_comm_t* c, int device, int nranks, int rank);
int mumode_comm_ipc_handle_bytes(void);
int mumode_comm_ipc_export(mumode_comm_t c, int d, const int64_t* m, const int64_t* n, int cplx, void* handles);
int mumode_comm_ipc_import(mumode_comm_t c, int d, const int64_t* m, const int64_t* n, int cplx,
                           const void* all_handles);
/* Wait for the handle's and the comm's queued work with failure detection:
 * polls both streams and ncclCommGetAsyncError every 50 us; an NCCL error or
 * timeout_ms without completion (<= 0: no limit) aborts an owned
 * communicator (ncclCommAbort) and returns MUMODE_ERR_NCCL instead of
 * hanging on a lost peer. */
int mumode_comm_poll(mumode_handle_t h, mumode_comm_t c, int64_t timeout_ms);
/* The partition (host only): c_off[P+1] = last-mode slab offsets (rank r
 * holds T[..., c_off[r]:c_off[r+1]]), a_off[P+1] = output row blocks over
 * A = n_1...n_{d-1} (rank r returns rows a_off[r]:a_off[r+1] of the result
 * flattened to A x n_d). Even splits; MUMODE_ERR_SIZE if m_d < P. */
int mumode_slab_plan(int nranks, int d, const int64_t* m, const int64_t* n, int64_t* c_off,
                     int64_t* a_off);
/* The schedule mumode_dist_tucker_* executes on rank `rank` (host only):
 * chunk_tab rows (col0, width, send_offset) per sub-slab, op_tab rows
 * (chunk, kind, peer, send_offset, z_offset, count) with kind 0 = NCCL send,
 * 1 = NCCL receive, 2 = own block (written in place by the last local
 * mode's scatter epilogue, like the packed send blocks -- no pack pass);
 * offsets/counts in doubles.
 * Lets the multi-rank logic be checked without GPUs. Tables too small ->
 * MUMODE_ERR_ARGUMENT with the needed sizes in n_chunks / n_ops. */
int mumode_dist_plan(int nranks, int rank, int d, const int64_t* m, const int64_t* n, int chunks,
                     int cplx, int64_t* chunk_tab, int max_chunks, int* n_chunks, int64_t* op_tab,
                     int max_ops, int* n_ops);
/* One slab-partitioned Tucker application (replaces ops::tucker across
 * ranks, tucker.hpp:129-144). m, n: GLOBAL extents. T: this rank's slab
 * (m_1 x ... x m_{d-1} x c_r, column-major); S: this rank's (A_r x n_d)
 * column-major output rows. The slab is processed in `chunks` sub-slabs whose
 * NCCL exchange overlaps the next sub-slab's contraction (0 = auto: split only
 * while each sub-slab keeps >= 4M elements, at most 4). All ranks call it
 * with the same extents and chunks. Stream-ordered on the handle's stream. */
int mumode_dist_tucker_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m,
                           const int64_t* n, const double* T, const double* const* L, double* S,
                           int chunks);
int mumode_dist_tucker_c128(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m,
                            const int64_t* n, const double* T, const double* const* L, double* S,
                            int chunks);
/* The peer-store application in phases (exchange mode 1, one sub-slab):
 * phase 0 = the whole application; 1 = local modes + peer stores + signal;
 * 2 = wait for every rank's signal of this epoch + mode d. Running phase 2
 * only after all ranks finished phase 1 (a host barrier) means no kernel ever
 * waits on another process. */
int mumode_dist_tucker_phase_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m,
                                 const int64_t* n, const double* T, const double* const* L, double* S,
                                 int phase);
int mumode_dist_tucker_phase_c128(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m,
                                  const int64_t* n, const double* T, const double* const* L, double* S,
                                  int phase);
/* The local half of one NCCL-path application on rank `rank` of `nranks`
 * without a communicator: every sub-slab's modes 1..d-1, its last local mode
 * storing the packed send blocks into `send` and the own row block into its
 * final columns of Z (A_r x m_d) -- exactly what mumode_dist_tucker_f64 does
 * before its NCCL group. Lets tests emulate the exchange between simulated
 * ranks on one GPU and check the send layout bitwise. */
int mumode_dist_local_f64(mumode_handle_t h, int nranks, int rank, int d, const int64_t* m, const int64_t* n,
                          const double* T, const double* const* L, double* send, double* Z, int chunks);
/* Return exchange after an application with output extents n (host only):
 * rank r's output rows (A_r x n_d) -> the last-mode slabs of the output for
 * the next application. op_tab rows as in mumode_dist_plan (send_offset into
 * the rows, z_offset into a [s][A_s x c_r] staging buffer). */
int mumode_dist_return_plan(int nranks, int rank, int d, const int64_t* n, int64_t* op_tab,
                            int max_ops, int* n_ops);
/* `steps` exponential-integrator steps u <- tucker(u, {E_1..E_d}) across ranks
 * (apps::linear_evolution_exact, src/evolution.cpp:70-82): each step is a
 * slab-partitioned Tucker, a return exchange and an unpack, in the
 * reference's mode order. u0, u: this rank's last-mode slabs (E square). */
int mumode_dist_expint_f64(mumode_handle_t h, mumode_comm_t c, int d, const int64_t* m,
                           const double* const* E, const double* u0, double* u, int steps);

/* Replaces ops::kronsumv (tucker.hpp:209-232): W = sum_mu V x_mu A_mu with
 * square A_mu of size m[mu], accumulated in the reference's order
 * (((t_1 + t_2) + t_3) + ...). */
int mumode_kronsumv_f64(mumode_handle_t h, int d, const int64_t* m, const double* V,
                        const double* const* A, double* W);
int mumode_kronsumv_c128(mumode_handle_t h, int d, const int64_t* m, const double* V,
                         const double* const* A, double* W);

/* Direct solve with the Kronecker sum of d symmetric factors
 * M_mu = Q_mu diag(evals_mu) Q_mu^T: x = tucker(tucker(b, Q^T) ./ Lambda, Q),
 * Lambda(j) = evals_1[j_1] + ... + evals_d[j_d] -- the IMEX direct backend's
 * solve (apps DirectSolver::solve, src/imex.cpp:67-86). Q, Qt (= Q^T) are
 * device m_mu x m_mu matrices; evals are HOST arrays (small). A zero
 * denominator returns MUMODE_ERR_NUMERICAL like the reference. */
int mumode_kronsum_solve_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* Q,
                             const double* const* Qt, const double* const* evals, const double* b,
                             double* x);

/* Exponential-integrator march (apps::linear_evolution_exact applied
 * repeatedly, src/evolution.cpp:70-82): u <- tucker(u; E_1..E_d) `steps`
 * times with square E_mu; u0 and u_out may alias. Captured in a CUDA graph
 * after the first call with a given shape. */
int mumode_expint_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* E,
                      const double* u0, double* u_out, int steps);

/* ---- host-buffer drop-in (copies included) ---------------------------- */
int mumode_host_mode_product_f64(mumode_handle_t h, int d, const int64_t* m, int mu,
                                 int64_t n_mu, const double* T, const double* L, double* S);
int mumode_host_mode_product_c128(mumode_handle_t h, int d, const int64_t* m, int mu,
                                  int64_t n_mu, const double* T, const double* L, double* S);
int mumode_host_tucker_f64(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                           const double* T, const double* const* L, double* S, int adjoint);
/* Enqueue-only variant of mumode_host_tucker_f64 (forward, real): returns
 * after queuing the upload, the chain and the download. Consecutive calls
 * alternate two device staging slots, so one call's download overlaps the
 * next call's upload (PCIe full duplex). T, L and S must stay valid (and S
 * unread) until mumode_host_wait; T and S in pinned memory make it fully
 * asynchronous (pageable buffers still work, with host-blocking copies). */
int mumode_host_tucker_f64_async(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                                 const double* T, const double* const* L, double* S);
/* Wait for every queued host-buffer call on the handle. */
int mumode_host_wait(mumode_handle_t h);
int mumode_host_tucker_c128(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                            const double* T, const double* const* L, double* S, int adjoint);
int mumode_host_tucker_promote(mumode_handle_t h, int d, const int64_t* m, const int64_t* n,
                               const double* T, const double* const* L, double* S, int adjoint);
int mumode_host_kronsumv_f64(mumode_handle_t h, int d, const int64_t* m, const double* V,
                             const double* const* A, double* W);
int mumode_host_kronsumv_c128(mumode_handle_t h, int d, const int64_t* m, const double* V,
                              const double* const* A, double* W);
int mumode_host_expint_f64(mumode_handle_t h, int d, const int64_t* m, const double* const* E,
                           const double* u0, double* u_out, int steps);

/* ---- diagnostics ------------------------------------------------------ */
/* FP64 tensor-pipe (DMMA) peak of this GPU at its current clocks, TFLOP/s:
 * the roofline denominator bench.py reports against. */
int mumode_probe_fp64_peak(mumode_handle_t h, double* tflops);

/* ---- host preprocessing ---------------------------------------------- */
/* Matrix exponential, scaling-and-squaring with the degree-13 Pade
 * approximant (Higham 2005), host fp64. Role of la::expm
 * (proj/src/expm.cpp:97-151) for the exponential integrator's E_mu.
 * Bitwise equal to la::expm linked against OpenBLAS 0.3.15's SkylakeX kernels
 * for n <= 384 (its products and triangular solves restate that build's
 * k-ordered FMA chains and 16-row trsm blocks; probed to n = 400); with another
 * BLAS build, or larger n, the two agree to ~1e-15 relative. */
int mumode_expm_f64(int64_t n, const double* A, double* E);

/* Inverse of a square matrix (LU with partial pivoting, host fp64). Kept for
 * callers that want P^-1 itself; ops::itucker runs on mumode_lu_factor_* +
 * mumode_itucker_* (per-mode solves, no inverse formed). Returns
 * MUMODE_ERR_NUMERICAL on a zero pivot (lu.hpp:33). */
int mumode_inverse_f64(int64_t n, const double* P, double* Pinv);

/* la::lu_factor (proj/include/mumode/lu.hpp:23-47), host: P = perm * L * U
 * with partial pivoting; lu (n x n, column-major) holds the unit-lower L
 * below the diagonal and U on/above it, piv[k] = the row swapped into row k
 * at step k. Bitwise the reference's factors (the FactorizedStack role,
 * tucker.hpp:34-51). MUMODE_ERR_NUMERICAL "lu_factor: singular pivot". */
int mumode_lu_factor_f64(int64_t n, const double* P, double* lu, int64_t* piv);
int mumode_lu_factor_c128(int64_t n, const double* P, double* lu, int64_t* piv);

/* Replaces ops::itucker (tucker.hpp:187-204): S = T x_1 P_1^-1 ... x_d P_d^-1
 * by per-mode triangular solves with DEVICE factors LU[k] (m_k x m_k, as
 * mumode_lu_factor_*) and DEVICE pivots piv[k] (m_k int64); lu_solve's
 * arithmetic (lu.hpp:52-69 on OpenBLAS's trsm kernels). S may alias T.
 * Bitwise equal to the reference linked against OpenBLAS 0.3.15 (SkylakeX)
 * for real extents up to 384; beyond, that build splits each trsm update at
 * GEMM_Q = 384 columns (two chains per row) and the two agree to ~1e-16
 * relative (tests: 391..409 within 1e-13). Complex: bitwise for extents
 * that are multiples of 4. */
int mumode_itucker_f64(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                       const int64_t* const* piv, double* S);
int mumode_itucker_c128(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                        const int64_t* const* piv, double* S);
/* The same with HOST buffers (copies included). */
int mumode_host_itucker_f64(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                            const int64_t* const* piv, double* S);
int mumode_host_itucker_c128(mumode_handle_t h, int d, const int64_t* m, const double* T, const double* const* LU,
                             const int64_t* const* piv, double* S);

/* The IMEX direct backend's factor preprocessing (apps DirectSolver,
 * src/imex.cpp:56-65), host: extract_tridiag (src/imex.cpp:28-48) returns the
 * symmetric tridiagonal part of M (n x n) or MUMODE_ERR_ARGUMENT with the
 * reference's "factor is not tridiagonal" / "not symmetric" text;
 * symtridiag_eig (src/tridiag.cpp:12-90, EigMode::FullVectors) returns the
 * ascending eigenvalues and the m x m eigenvector matrix (columns), bitwise
 * the reference's implicit-shift QL. */
int mumode_extract_tridiag_f64(int64_t n, const double* M, double* diag, double* offdiag);
int mumode_symtridiag_eig_f64(int64_t m, const double* diag, const double* offdiag, double* values,
                              double* vectors);

/* Seeded input generator reproducing the reference's draws bit-for-bit:
 * std::mt19937_64(seed) and a FRESH std::normal_distribution<double> per
 * filled object (tools/mumode_cli.cpp:94-121). Complex draws re then im. */
typedef struct mumode_rng_s* mumode_rng_t;
int mumode_rng_create(mumode_rng_t* r, uint64_t seed);
int mumode_rng_destroy(mumode_rng_t r);
/* Fill n doubles (or n complex = 2n doubles if complex_ != 0). */
int mumode_rng_normal(mumode_rng_t r, double* out, int64_t n, int complex_);
/* Raw 64-bit draws (the reference's `g() % k` shape draws). */
int mumode_rng_u64(mumode_rng_t r, uint64_t* out, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* MUMODE_GPU_H */
