/*
 * blocksolve_b200.h — C ABI of the B200 (sm_100a) block-Jacobi / Krylov
 * 7-point stencil engine (libbsgpu.so).
 *
 * The reference package `blocksolve` is pure Python and has no FFI; its seam
 * is the Python solver API.  Each entry point below replaces the numerical
 * core of one reference function (cited file:line into
 * /root/reference/pkg/src/blocksolve).  The Python host layer
 * (paper_2009_12638_b200/) binds these through ctypes and keeps the
 * reference's signatures and error behaviour.
 *
 * Conventions
 *  - All vectors are fp64, x-fastest (index = i + nx*(j + ny*k),
 *    problems.py:110-111), laid out over each block's *padded box*: the owned
 *    box dilated by `overlap` and clipped to the grid (the bounding box of the
 *    block's extended region, problems.py:330-340).
 *  - Pointers are device pointers; `stream` is a cudaStream_t (NULL = legacy).
 *  - Every call returns 0 on success, a negative BS_E* code on failure;
 *    bs_last_error() returns a thread-local message for the last failure.
 *  - Calls are asynchronous on `stream` unless documented as blocking.
 */
#ifndef BLOCKSOLVE_B200_H
#define BLOCKSOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 2

#define BS_OK 0
#define BS_EINVAL -1   /* bad argument  -> ValueError / ConfigurationError */
#define BS_ECUDA -2    /* CUDA runtime failure -> RuntimeError              */
#define BS_ESTATE -3   /* call out of protocol order -> ProtocolError       */

/* inner-solver stop reasons (inner_solvers.py:64) */
#define BS_STOP_NONE 0
#define BS_STOP_TOLERANCE_MET 1
#define BS_STOP_MAX_ITERATIONS 2
#define BS_STOP_BREAKDOWN 3

/* tolerance basis: "rhs" is the reference (inner_solvers.py:70-72,108-113);
 * "initial" measures against ||b - A x0|| (SURVEY §8(c) wrapper). */
#define BS_BASIS_RHS 0
#define BS_BASIS_INITIAL 1

#define BS_KIND_CG 0
#define BS_KIND_GMRES 1

/* Direction order = ascending global column order of the stencil
 * (problems.py:142-167): 0 z-1, 1 y-1, 2 x-1, 3 x+1, 4 y+1, 5 z+1. */
#define BS_NDIR 6

typedef struct bs_block_desc {
    int32_t global_dims[3];  /* nx, ny, nz of the interior grid (Grid3D)    */
    int32_t owned_lo[3];     /* owned box, half-open, (x,y,z) (problems.py:193-213) */
    int32_t owned_hi[3];
    int32_t overlap;         /* L1 dilation radius o (problems.py:178-190)  */
    double *x;               /* iterate over the padded box (holds halo values at
                                non-region cells when overlap > 0)          */
    double *r;               /* residual scratch                            */
    double *p0, *p1;         /* ping-pong search directions                 */
    const double *b;         /* global rhs restricted to the padded box     */
    double *ghost[BS_NDIR];  /* halo planes just outside the padded box (NULL
                                where the face lies on the global boundary) */
    double *history;         /* device residual history, history_cap entries */
    int32_t history_cap;
    int32_t remote;          /* 1: phantom of a block another process owns —
                                geometry + r (its snapshot, peer-mapped) only;
                                read by the overlap merge, never solved
                                (multi-process overlap > 0, config 5) */
} bs_block_desc;

/* Per-block solver report, host side (InnerSolveReport, inner_solvers.py:60-67,
 * plus the squared sums the outer sweep needs, multisplit.py:372-406). */
typedef struct bs_block_report {
    int32_t phase;
    int32_t stop_reason;
    int32_t iterations_used;
    int32_t pending_flush;
    double final_relative_residual;
    double rhs_sq;       /* ||rhs||^2 of the last residual sweep            */
    double r_sq;         /* ||rhs - A x||^2 over the region                 */
    double r_owned_sq;   /* same restricted to owned rows (local residual)  */
    double rglob_owned_sq; /* ||b - A_global x||^2 over owned rows (true mode) */
    double scale;
    int32_t last_iterations;   /* the solve before the last bs_*_begin (its count / */
    int32_t last_stop_reason;  /* stop), so the outer sweep reads them with the residual */
} bs_block_report;

typedef struct bs_ctx bs_ctx;

int bs_abi_version(void);
const char *bs_last_error(void);

/* Create an engine over `nblocks` blocks resident on `device`.  Sweeps tile
 * each block into 32 x 8 columns; z_chunk = 0 streams full-depth columns
 * unless the block has too few columns to fill the GPU (then z is split into
 * chunks of >= 32 planes); z_chunk > 0 forces the chunk depth.  The tiling is
 * a function of the block alone, so reductions do not depend on which blocks
 * share a GPU.  The descriptor table is copied; the buffers stay owned by the
 * caller.  bs_run drives CG solves with one persistent cooperative launch
 * when every tile fits co-resident (environment BS_PERSIST=0 forces the
 * CUDA-graph path; both give bitwise-identical results). */
int bs_ctx_create(int device, int nblocks, const bs_block_desc *blocks, int z_chunk,
                  bs_ctx **out);
int bs_ctx_destroy(bs_ctx *ctx);
int bs_ctx_num_ctas(const bs_ctx *ctx);
/* How the last bs_run drove its solves: 0 CUDA graph of sweep launches,
 * 1 persistent cooperative kernel (one tile per CTA), 2 streaming persistent
 * kernel (k_cg_stream), 3 launch mode (per-kernel timing), 4 point-Jacobi
 * graph, -1 none yet. */
int bs_ctx_run_path(const bs_ctx *ctx);

/* Row pitch (in doubles) of block `block`'s padded-box vectors: the x extent
 * rounded up to 4 (TMA needs 16-byte row strides).  Index of padded-box cell
 * (i, j, k) = i + pitch * (j + ny_pad * k).  Returns < 0 on error. */
int bs_block_pitch(const bs_ctx *ctx, int block);

/* a1: y = A_ii x on block `block`'s region (x, y in the block's pitched layout) — the principal-submatrix SpMV
 * (linalg.py:178-194 on problems.py:362-406's A_ii), bit-identical to the
 * reference's reduceat association.  Values of y outside the region are 0. */
int bs_stencil_apply(bs_ctx *ctx, int block, const double *x, double *y, void *stream);

/* a2: arm an inner CG solve on every block with active[b] != 0
 * (inner_solvers.py:102-146, dispatched from multisplit.py:562-563).
 * active == NULL arms all blocks.  The right-hand side is assembled on the
 * device as b - C*ghost (multisplit.py:333-338); x is the warm start. */
int bs_cg_begin(bs_ctx *ctx, int max_iterations, double tolerance, int basis,
                const int32_t *active, void *stream);

/* a2': arm point-Jacobi sweeps x <- D^-1 (b - (A - D) x) on the active blocks
 * (inner_solvers.py:75-99; same rhs assembly and warm start as bs_cg_begin).
 * One fused sweep per iteration k reads x_k once (haloed), reports
 * ||rhs - A x_k|| / ||rhs|| and writes x_{k+1}; stops at the first x_k that
 * meets the tolerance (k = iterations used), on a non-finite residual
 * (breakdown) or at k = max_iterations.  bs_run drives the solve; the iterate
 * is home in x after bs_flush (halo packs and residual sweeps read it where it
 * is without a flush). */
int bs_jacobi_begin(bs_ctx *ctx, int max_iterations, double tolerance, int basis,
                    const int32_t *active, void *stream);

/* a3: restarted GMRES(m) workspace.  Per block: V = m Krylov vectors in the
 * block's pitched layout, V[j] = V + j*vstride; W = the Arnoldi work vector.
 * m <= 64.  (inner_solvers.py:149-251; V is fp64[(m+1) x n] there.) */
typedef struct bs_gmres_desc {
    double *V;
    int64_t vstride;  /* elements between consecutive Krylov vectors */
    double *W;
} bs_gmres_desc;

int bs_gmres_setup(bs_ctx *ctx, int m, const bs_gmres_desc *per_block);

/* Arm restarted GMRES(m) on the active blocks (same rhs assembly and warm
 * start as bs_cg_begin; stop rules of inner_solvers.py:153-243: happy
 * breakdown, recurrence claim verified against the true residual, restart,
 * stagnation -> breakdown). */
int bs_gmres_begin(bs_ctx *ctx, int max_iterations, double tolerance, int basis,
                   const int32_t *active, void *stream);

/* Run armed GMRES solves: per restart cycle the host enqueues every Arnoldi
 * step (v_j = w/||w||, w = A v_j fused with h_0j, j modified Gram-Schmidt
 * passes, ||w|| + Givens), x += V y and the true residual, then polls one
 * counter.  Finished blocks skip the remaining launches.  Blocking. */
int bs_gmres_run(bs_ctx *ctx, int max_cycles, void *stream, int64_t *kernels_out);

/* The same for block `block` alone: every launch covers only that block's
 * CTAs and only its solve is polled.  Blocks solved one after another this
 * way may share one V/W workspace (bs_gmres_setup with equal pointers),
 * which is what lets eight 514^3 blocks of a 1024^3 grid with GMRES(30)
 * fit one GPU (one basis: 34 GB instead of 270 GB).  Same results, bit
 * for bit, as the all-block run (multisplit.py:562-580: the sweep-k inner
 * solves are independent). */
int bs_gmres_run_block(bs_ctx *ctx, int block, int max_cycles, void *stream, int64_t *kernels_out);

/* Run armed solves to completion with device-side stopping.  Default: one
 * CUDA-graph launch whose WHILE node iterates {CG sweep 1, CG sweep 2,
 * IF(any block verifying) residual sweep} until no block is active — no host
 * round trip per iteration (after bs_jacobi_begin: WHILE { Jacobi sweep }).  With timing enabled (bs_timing) the same kernels
 * are launched from the host in batches of `batch` cycles with CUDA events
 * around each.  max_launches > 0 bounds the sweeps (runaway guard; exceeding
 * it stops the solves and returns BS_ESTATE).  Blocking.  *sweeps_out
 * receives the number of sweep kernels that ran. */
int bs_run(bs_ctx *ctx, int batch, int max_launches, void *stream, int64_t *sweeps_out);

/* Run only the residual sweep of armed solves (the INIT step: rhs assembly
 * + r0 = rhs - A x0 + the local/true residual sums of the current iterate,
 * multisplit.py:333-338 and 372-406).  Lets the outer driver read the
 * sweep-k residual and decide termination (multisplit.py:409-426) before
 * any CG iteration of sweep k+1 runs. */
int bs_sweep_resid(bs_ctx *ctx, void *stream);

/* Disarm the active blocks (phase -> done) without touching their iterate. */
int bs_cancel(bs_ctx *ctx, const int32_t *active, void *stream);

/* One residual sweep on the active blocks without starting a solve:
 * r = (b - C*ghost) - A_ii x and the report's squared sums (multisplit.py:
 * 372-396 local residual, 404-406 true residual on owned rows).  Blocking
 * only through bs_read_reports. */
int bs_residual(bs_ctx *ctx, const int32_t *active, void *stream);

/* Apply the deferred x += alpha*p update of every block that has one. */
int bs_flush(bs_ctx *ctx, void *stream);

/* a8 (sync halo, overlap 0): for each plan entry (dst_block, dir, src_block)
 * write src's current boundary values (x + pending alpha*p) into dst's
 * ghost[dir] plane (comm.py:332-365 + multisplit.py:341-369 with m=1). */
int bs_halo_pack(bs_ctx *ctx, int nplan, const int32_t *plan, void *stream);

/* a6 (overlap > 0): equal-weight merge of overlapping values
 * (multisplit.py:341-369).  Requires every block's x to be final (bs_flush).
 * Snapshots x into r (the post-solve payloads), then writes the 1/m average
 * over covering blocks — own value first, neighbours in ascending id — into
 * x at shared points, and the average over covering blocks into the halo
 * cells (x cells outside the region, face planes). */
int bs_overlap_merge(bs_ctx *ctx, void *stream);

/* The two halves of bs_overlap_merge, for blocks spread over processes: every
 * process snapshots its blocks, a host barrier orders the snapshots before
 * any read, then the combine step reads the neighbours' snapshots — through
 * the peer-mapped pointers of their phantom descriptors (remote = 1, r = the
 * owner's snapshot opened with bs_ipc_open) — over NVLink, in the same
 * order and with the same arithmetic as the single-process merge. */
int bs_overlap_snapshot(bs_ctx *ctx, void *stream);
int bs_overlap_combine(bs_ctx *ctx, void *stream);

/* a7 (overlap > 0): local residual with owner-canonical values
 * (multisplit.py:372-396) = b - A x_gathered on each block's owned rows,
 * read from the snapshots of bs_overlap_merge; reported in r_owned_sq and
 * rglob_owned_sq. */
int bs_owner_residual(bs_ctx *ctx, void *stream);

/* a9 async halo, sender side (comm.py:367-400): retire slot seq % R
 * (seqs[slot] = 0), store block `block`'s own boundary plane facing `dir`
 * (x + pending alpha p) into it (plane layout = the receiver's ghost plane),
 * then publish seqs[slot] = seq + 1 with a system-scope release.  `ring` and
 * `seqs` may be local or peer-mapped (NVLink) memory.  Never blocks. */
int bs_async_post(bs_ctx *ctx, int block, int dir, double *ring, uint64_t *seqs, int R, uint64_t seq,
                  void *stream);

/* a9 async halo, receiver side (comm.py:401-416): take the freshest published
 * slot newer than *applied (stale payloads are never applied), copy it via
 * `stage`, re-validate its seq (seqlock) and install it in ghost[ghost_dir];
 * *applied becomes that seq + 1.  A slot the sender lapped while it was read
 * is rejected (counted in *torn) and the old halo is kept, exactly like
 * "nothing newer delivered".  Never blocks. */
int bs_async_receive(bs_ctx *ctx, int block, int ghost_dir, const double *ring, const uint64_t *seqs, int R,
                     uint64_t *applied, double *stage, int *torn, void *stream);

/* Injected-latency variants (DelayModel, comm.py:51-81 and 376-416; SURVEY
 * §8(f) item 4).  The sender picks the ring slot itself (its host keeps the
 * reference's R-slot in-flight accounting: reclaim once the receiver reached
 * the delivery iteration, skip the send when no slot is free) and stamps
 * deliver[slot] = deliver_at (sender iteration + drawn delay) before the seq
 * release.  The receiver only considers slots with deliver[slot] <=
 * receiver_k, the outer iteration it has reached.  deliver == NULL gives the
 * plain calls above. */
int bs_async_post_slot(bs_ctx *ctx, int block, int dir, double *ring, uint64_t *seqs, int64_t *deliver, int slot,
                       uint64_t seq, int64_t deliver_at, void *stream);
int bs_async_receive_at(bs_ctx *ctx, int block, int ghost_dir, const double *ring, const uint64_t *seqs,
                        const int64_t *deliver, int R, int64_t receiver_k, uint64_t *applied, double *stage,
                        int *torn, void *stream);

/* Peer memory for one-sided halo puts across processes (one process per GPU,
 * NVLink): export a device pointer as a 64-byte CUDA IPC handle of its
 * allocation plus the offset inside it; open it in another process (peer
 * access enabled lazily) to get a pointer that bs_async_post / the halo puts
 * can store into directly.  bs_ipc_close takes the base returned by
 * bs_ipc_open minus the offset. */
int bs_ipc_export(const void *ptr, unsigned char *handle_out /* 64 bytes */, uint64_t *offset_out);
int bs_ipc_open(const unsigned char *handle /* 64 bytes */, uint64_t offset, void **ptr_out);
int bs_ipc_close(void *base);

/* the seeded rhs generated on the device, bit-identical
 * to numpy's default_rng(seed).uniform(low, high, n) — PCG64 state/increment
 * as numpy reports them after seeding (bit_generator.state). */
int bs_uniform_pcg64(double *out, int64_t n, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, double low, double high, void *stream);

/* Power-iteration vector helpers (linalg.py:243-276).
 * bs_vec_nrm2: work[0] = ||x||_2 (device memory, work >= BS_VEC_WORK doubles),
 * fixed reduction order — bitwise repeatable.  bs_vec_scale: y = x / denom
 * elementwise (y may alias x). */
#define BS_VEC_WORK 512
int bs_vec_nrm2(const double *x, int64_t n, double *work, void *stream);
int bs_vec_scale(const double *x, int64_t n, double denom, double *y, void *stream);

/* Number of kernels this library has launched (process lifetime). */
unsigned long long bs_launch_count(void);

/* CUDA-event timing of the sweep kernels issued by bs_run, per kind
 * [0] residual sweep, [1] CG sweep 1, [2] CG sweep 2: total milliseconds and
 * launch counts since the last reset.  enable: 1 on, 0 off, -1 read only
 * (1 and 0 also reset the totals). */
int bs_timing(bs_ctx *ctx, int enable, double *ms_out, long long *n_out);

/* Copy every block's report to host memory (blocking). */
int bs_read_reports(bs_ctx *ctx, bs_block_report *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKSOLVE_B200_H */
