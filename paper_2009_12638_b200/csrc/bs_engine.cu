// bs_engine.cu — sm_100a engine for the block-Jacobi / CG 7-point stencil path.
//
// One translation unit: the TMA-fed stencil sweep kernels, the fused CG phase
// machine with device-side stopping (CUDA-graph WHILE loop), halo packing and
// the C ABI declared in include/blocksolve_b200.h.
//
// Reference algorithm (file:line into /root/reference/pkg/src/blocksolve):
//   SpMV            linalg.py:178-194 on the block system of problems.py:362-406
//   CG              inner_solvers.py:102-146 (scale = ||rhs||, 70-72)
//   rhs assembly    multisplit.py:333-338
//   local residual  multisplit.py:372-396, true residual 404-406
//   sync halo       comm.py:332-365 + merge multisplit.py:341-369 (overlap 0)
//
// Design:
//   * Every vector lives over the block's padded box, x-fastest with a row
//     pitch rounded up to 4 doubles (TMA needs 16-byte global strides).
//   * A CTA owns a TX x TY column tile and marches CZ planes in z.  One
//     thread issues cp.async.bulk.tensor (TMA) loads of whole planes — the
//     tile plus a one-cell x/y halo for the stencil inputs, the bare tile for
//     epilogue operands — into an 8..12-deep shared-memory ring completed on
//     mbarriers (a dedicated producer warp; consumers release stages through
//     `empty` mbarriers, so there is no CTA-wide barrier per plane).  Cells
//     outside the padded box are zero-filled by TMA (= absent neighbours).
//   * The stencil input u is formed from the staged operands: u = r + beta*p
//     in CG sweep 1 (p written once, never re-read), u = p in sweep 2,
//     u = x + alpha*p in residual sweeps (x += alpha p is deferred).  One CG
//     iteration therefore moves 64 B/point of compulsory HBM traffic.
//   * Reductions are fixed-order (thread z order, xor-butterfly warps,
//     sequential warps, strided+tree across the block's tiles).  The last CTA
//     of each block reduces that block and runs its scalar recurrence; the
//     last CTA of the launch sets the graph's loop conditions.  Results are
//     deterministic and independent of which other blocks share the GPU.
//   * All arithmetic is explicit round-to-nearest without FMA contraction
//     (__dadd_rn/__dmul_rn and -fmad=false): the SpMV is bit-identical to the
//     reference's numpy reduceat.

#include "blocksolve_b200.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define BS_CU(call)                                                                  \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess)                                                       \
            return fail(BS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#ifndef BS_TX
#define BS_TX 32
#endif
#ifndef BS_RY
#define BS_RY 1
#endif
constexpr int TX = BS_TX;              // tile width (x, contiguous)
constexpr int RY = BS_RY;              // rows per consumer thread
#ifndef BS_NT
#define BS_NT 256
#endif
constexpr int NT = BS_NT;              // sweep consumer threads: TX columns x NT/TX thread rows
constexpr int NPT = 256;               // threads of the pointwise (GMRES) passes
constexpr int TY = (NT / TX) * RY;     // tile height
constexpr int NCW = NT / 32;           // consumer warps
constexpr int NTHR = NT + 32;          // + one TMA producer warp
constexpr int HY = TY + 2;
// TMA boxes must start on a 16-byte boundary in the innermost dimension, so
// the staged haloed box spans x in [x0-2, x0+TX+2): 2 cells left, 2 right.
constexpr int SX = TX + 4;
constexpr int SC = SX * HY;            // staged haloed-box cells
constexpr int NQ = 4;                  // partial sums per CTA
#ifndef BS_NSTAGE_AB
#define BS_NSTAGE_AB (BS_RY == 1 ? 8 : 6)  // ring depth of sweeps staging two haloed operands
#endif
#ifndef BS_NSTAGE_A
#define BS_NSTAGE_A (BS_RY == 1 ? 12 : 10)  // ring depth of sweeps staging one haloed operand
#endif
constexpr int PITCH_ALIGN = 4;         // doubles
#ifndef BS_MINBLOCKS
#define BS_MINBLOCKS (BS_RY == 1 ? 3 : 2)  // resident CTAs per SM the sweep kernels are compiled for
#endif
// The residual and point-Jacobi sweeps (four sums, face couplings, two
// reduceat chains) spill at the 72 registers of 3 CTAs per SM: ncu showed
// long-scoreboard stalls on the spill reloads as the top stall of a serving
// residual sweep (profiles/r02_ncu_resid_summary.md).  They are compiled for
// 2 CTAs per SM (112 registers) instead.
#ifndef BS_MINBLOCKS_HEAVY
#define BS_MINBLOCKS_HEAVY 2
#endif

constexpr int SEG_H = ((SC * 8 + 127) / 128) * 128;  // staged haloed box, 128B aligned
constexpr int SEG_O = TX * TY * 8;                    // bare tile

enum Phase : int {
    PH_IDLE = 0,
    PH_INIT = 1,    // residual sweep that starts a CG solve
    PH_S1 = 2,      // p = r + beta p_old ; x += alpha_pend p_old ; p.Ap
    PH_S2 = 3,      // r -= alpha A p ; r.r
    PH_VERIFY = 4,  // true-residual check on claimed convergence
    PH_DONE = 5,
    PH_RESID = 6,   // standalone residual sweep (outer residual / checks)
    // restarted GMRES(m) (inner_solvers.py:149-243), one Arnoldi step j =
    // NORM(j) -> SPMV(j) -> MGS(j, 1..j) -> FINAL(j); a cycle ends FORM -> G_RESID
    PH_G_NORM = 7,    // v_j = w / ||w||   (v_0 = r / beta)
    PH_G_SPMV = 8,    // w = A v_j ; h_0j = v_0 . w
    PH_G_MGS = 9,     // w -= h_{i-1,j} v_{i-1} ; h_ij = v_i . w
    PH_G_FINAL = 10,  // w -= h_jj v_j ; ||w|| ; Givens ; stop tests
    PH_G_FORM = 11,   // x += V y
    PH_G_RESID = 12,  // true residual of the formed iterate ; restart or stop
    PH_OWNRES = 13,   // residual of the gathered (owner) iterate on owned rows
    PH_JAC = 14,      // point-Jacobi sweep: rel of x_k and x_{k+1} = (rhs - offd x_k) / 6
};

enum Kind : int { KIND_CG = 0, KIND_GMRES = 1, KIND_JACOBI = 2 };

enum Op : int { OP_RESID = 0, OP_S1 = 1, OP_S2 = 2, OP_APPLY = 3, OP_GSPMV = 4, OP_JAC = 5 };

// pointwise (non-stencil) GMRES passes
enum Pk : int { PK_NORM = 0, PK_MGS = 1, PK_FINAL = 2, PK_FORM = 3, PK_OWNRES = 4 };

constexpr int MAXM = 64;    // largest supported GMRES restart length
constexpr int MAXNBR = 32;  // neighbour list capacity per block (overlapping merge)
#ifndef BS_PCHUNK
#define BS_PCHUNK 16384
#endif
constexpr int PCHUNK = BS_PCHUNK;  // doubles per CTA in pointwise passes
enum GFlag : int { GF_NONE = 0, GF_HAPPY = 1, GF_CHECK = 2, GF_CYCLE = 3 };

// Stage layout per op: [A haloed][B haloed, if the op has one][C bare tile].
// Fewer bytes per stage buys a deeper ring in about the same shared memory,
// so every op keeps ~60 KB of loads in flight per CTA.
__host__ __device__ constexpr bool op_has_b(int op) { return op == OP_RESID || op == OP_S1; }
#ifndef BS_EASY
#define BS_EASY 1  // interior planes of dilated regions take the box logic (sweep_tile)
#endif
#ifndef BS_REV_PASSES
#define BS_REV_PASSES 1
#endif
// Cache policy of the GMRES pointwise passes.  1: the streams the next pass
// re-reads (w, v_i, the fresh v_{j+1}) are loaded/stored with the default L2
// policy and the one it does not (v_{i-1}, v_j in FINAL, NORM's source) is
// marked evict-first, so with BS_REV_PASSES the next pass starts on L2 hits.
// 2 (default): as 1, but in a launch over one block, MGS/FINAL CTAs among
// the last BS_MGS_KEEP of the launch (the chunks the next, reversed pass reads first; 256 chunks = 64 MB
// of w + v_i) access w and v_i with an L2 evict_last policy and every other
// MGS/FINAL access is evict_first (profiles/r01_ab_mgs_cache_hint.log).
// 0: every w access streaming (evict-first), V through the read-only path.
#ifndef BS_MGS_HINT
#define BS_MGS_HINT 2
#endif
#ifndef BS_MGS_KEEP
#define BS_MGS_KEEP 256  // BS_MGS_HINT 2: trailing chunks per pass kept evict_last
#endif
#ifndef BS_REV_S2
#define BS_REV_S2 1
#endif
__host__ __device__ constexpr bool op_rev(int op) { return BS_REV_S2 && op == OP_S2; }
// Planes per ring stage: CG sweep 2 stages its planes in pairs (one TMA box of
// depth 2 per operand): half the TMA issues and mbarrier round trips per byte
// of the lightest sweep.
#ifndef BS_ZP_S2
#define BS_ZP_S2 2
#endif
#ifndef BS_ZP_S1
#define BS_ZP_S1 1
#endif
#ifndef BS_ZP_LIGHT
#define BS_ZP_LIGHT 2  // SpMV, point-Jacobi and GMRES-SpMV sweeps (one haloed operand)
#endif
#ifndef BS_ZP_RESID
#define BS_ZP_RESID 2
#endif
__host__ __device__ constexpr int op_zp(int op) {
    return op == OP_S2      ? BS_ZP_S2
           : op == OP_S1    ? BS_ZP_S1
           : op == OP_RESID ? BS_ZP_RESID
           : (op == OP_APPLY || op == OP_JAC || op == OP_GSPMV) ? BS_ZP_LIGHT
                                                                : 1;
}
#ifndef BS_NSTAGE_APPLY
#define BS_NSTAGE_APPLY 20  // ring depth (planes) of the standalone SpMV: nothing but the stencil per plane
#endif
// The residual and point-Jacobi sweeps run 2 CTAs per SM (BS_MINBLOCKS_HEAVY),
// so each can afford a deeper ring than the 3-per-SM CG sweeps: the residual
// sweep at 256^3 takes 90.5 / 83.1 / 80.1 us with 8 / 10 / 12 planes in flight
// (16 and 20 planes slow the Jacobi sweep down: 83.3 / 93.7 us against 79.3;
// profiles/r02_ab_lean.log).
#ifndef BS_NSTAGE_RESID
#define BS_NSTAGE_RESID 12
#endif
#ifndef BS_NSTAGE_JAC
#define BS_NSTAGE_JAC BS_NSTAGE_A
#endif
__host__ __device__ constexpr int op_planes(int op) {
    return op == OP_RESID   ? BS_NSTAGE_RESID
           : op == OP_JAC   ? BS_NSTAGE_JAC
           : op_has_b(op)   ? BS_NSTAGE_AB
           : op == OP_APPLY ? BS_NSTAGE_APPLY
                            : BS_NSTAGE_A;
}
__host__ __device__ constexpr int op_stages(int op) { return (op_planes(op) + op_zp(op) - 1) / op_zp(op); }
// stage layout: [A: zp haloed planes][B: zp haloed planes, if any][C: zp bare planes]
__host__ __device__ constexpr int op_sega(int op) { return ((op_zp(op) * SC * 8 + 127) / 128) * 128; }
__host__ __device__ constexpr int op_coff(int op) { return op_has_b(op) ? 2 * op_sega(op) : op_sega(op); }
__host__ __device__ constexpr int op_stage_bytes(int op) { return op_coff(op) + op_zp(op) * SEG_O; }
__host__ __device__ constexpr int op_smem(int op) { return op_stages(op) * (op_stage_bytes(op) + 16); }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int SMEM_MAX = cmax(cmax(cmax(op_smem(OP_RESID), op_smem(OP_S1)), cmax(op_smem(OP_S2), op_smem(OP_APPLY))),
                              cmax(op_smem(OP_GSPMV), op_smem(OP_JAC)));

// Tensor maps per block, one set per sweep op: each op's boxes are op_zp(op)
// planes deep (H: haloed (TX+4) x (TY+2) box, O: bare TX x TY tile).
enum Tm : int {
    TM_RH_S1 = 0, TM_P0H_S1, TM_P1H_S1, TM_XO_S1,  // CG sweep 1
    TM_P0H_S2, TM_P1H_S2, TM_RO_S2,                // CG sweep 2
    TM_XH_J, TM_P0H_J, TM_BO_J,                    // point-Jacobi sweeps
    TM_XH_R, TM_P0H_R, TM_P1H_R, TM_BO_R,          // residual sweeps
    NTM
};

constexpr int STOP_STALLED = 4;

struct DBlock {
    int gn[3];
    int lo[3], hi[3];        // owned box
    int plo[3], pdim[3];     // padded box
    int pitch;               // row pitch (doubles) >= pdim[0]
    int overlap;
    int cta_begin, cta_end;  // CTA range in sweep launches
    int tiles_x, tiles_y, tiles_z, cz;  // tile grid (cz planes per z-chunk)
    int pcta_begin, pcta_end;  // CTA range in pointwise (GMRES) launches: fixed
                               // PCHUNK-element chunks of the pitched box
    double *x, *r, *p[2];
    const double *b;
    double *ghost[BS_NDIR];
    double *hist;
    int hist_cap;
    double *V;          // GMRES basis: V[j] = V + j * vstride (pitched padded box)
    long long vstride;
    double *W;          // GMRES work vector w
    int remote;         // phantom of a block owned by another process: only its
                        // snapshot (r, peer-mapped) is read, by the merge kernels
    int nnbr;           // neighbours, ascending ids (problems.py:343-349)
    int nbr[MAXNBR];
};

struct alignas(16) DState {
    // head (64 bytes): everything a sweep's CTAs need at its start
    int phase, first, pend, pcur;
    int xin;  // where the block's iterate lives: 0 = x, 1 = p[0] (Jacobi ping-pong)
    int gj, gi, kind;
    double alpha, beta, alpha_pend, rr;
    // rest: recurrence bookkeeping, touched only by transitions and reports
    int stop, it, max_its, basis, gflag, gm;
    int last_it, last_stop;  // the previous solve's count / stop, kept by k_arm(PH_INIT)
    double tol, tol_eff, scale, rel;
    double q[NQ];
    double cycle_start, gnrm;
};
constexpr int DSTATE_HEAD = 64;
static_assert(sizeof(DState) % 16 == 0, "DState is copied in 16-byte words");

// Small dense GMRES state of one block (inner_solvers.py:167-171).
struct GState {
    double H[(MAXM + 1) * MAXM];  // H[row * MAXM + col]
    double cs[MAXM], sn[MAXM];
    double g[MAXM + 1];
    double y[MAXM + 1];
};

struct Control {
    int cycles;      // WHILE-body iterations (S1 + S2 launches each)
    int max_cycles;  // runaway guard (0 = unlimited)
    int stalled;
    int resid_runs;  // residual-sweep launches inside the graph
    // persistent CG kernel: software grid barrier + loop conditions
    unsigned bar_count, bar_gen;
    int active, verify;
};

struct KParams {
    const DBlock *blocks;
    DState *states;
    const CUtensorMap *tmaps;
    const int *cta_block;
    int nblocks;
    int nctas;
    const int *pcta_block;  // pointwise-launch CTA table
    int npctas;
    double *partials;
    unsigned *blk_counter;
    unsigned *launch_counter;
    int *n_active;
    Control *ctl;
    cudaGraphConditionalHandle h_loop;
    cudaGraphConditionalHandle h_verify;
    int use_graph;
    GState *gstates;
    const CUtensorMap *gmaps;  // per block: V[0..MAXM-1] haloed, [MAXM] = V[0] bare
    int launch_j, launch_i;    // GMRES step served by this launch
    int cta_base, pcta_base;   // first CTA-table entry of this launch (one-block launches)
    int ntiles;                // tiles of this sweep launch (CTA-table entries from cta_base)
    unsigned *tile_counter;    // next tile of a sweep launch (rewound by its last CTA)
    int part_stride;           // doubles per quantity of one parity buffer of `partials`
};

// ------------------------------------------------------------------ geometry

__device__ __forceinline__ long long sidx(const DBlock &B, int i, int j, int k) {
    return (long long)(i - B.plo[0]) +
           (long long)B.pitch * ((long long)(j - B.plo[1]) + (long long)B.pdim[1] * (long long)(k - B.plo[2]));
}

__device__ __forceinline__ bool in_grid(const DBlock &B, int i, int j, int k) {
    return i >= 0 && j >= 0 && k >= 0 && i < B.gn[0] && j < B.gn[1] && k < B.gn[2];
}

__device__ __forceinline__ int box_dist1(const DBlock &B, int i, int j, int k) {
    int dx = max(0, max(B.lo[0] - i, i - (B.hi[0] - 1)));
    int dy = max(0, max(B.lo[1] - j, j - (B.hi[1] - 1)));
    int dz = max(0, max(B.lo[2] - k, k - (B.hi[2] - 1)));
    return dx + dy + dz;
}

// Extended region = L1 ball of radius `overlap` around the owned box, clipped
// to the grid (problems.py:330-340 dilation of a box under the 7-pt stencil).
__device__ __forceinline__ bool in_region(const DBlock &B, int i, int j, int k) {
    return in_grid(B, i, j, k) && box_dist1(B, i, j, k) <= B.overlap;
}

__device__ __forceinline__ bool in_owned(const DBlock &B, int i, int j, int k) {
    return i >= B.lo[0] && i < B.hi[0] && j >= B.lo[1] && j < B.hi[1] && k >= B.lo[2] && k < B.hi[2];
}

__device__ __forceinline__ bool in_pad(const DBlock &B, int i, int j, int k) {
    return i >= B.plo[0] && j >= B.plo[1] && k >= B.plo[2] && i < B.plo[0] + B.pdim[0] &&
           j < B.plo[1] + B.pdim[1] && k < B.plo[2] + B.pdim[2];
}

// Halo value of a coupled column (a grid point outside the region): stored in
// x itself when it lies inside the padded box (overlap > 0), otherwise in the
// face plane of direction `dir`.
__device__ __forceinline__ double ghost_at(const DBlock &B, int i, int j, int k, int dir) {
    if (in_pad(B, i, j, k)) return B.x[sidx(B, i, j, k)];
    long long idx;
    if (dir == 0 || dir == 5)
        idx = (long long)(i - B.plo[0]) + (long long)B.pdim[0] * (j - B.plo[1]);
    else if (dir == 1 || dir == 4)
        idx = (long long)(i - B.plo[0]) + (long long)B.pdim[0] * (k - B.plo[2]);
    else
        idx = (long long)(j - B.plo[1]) + (long long)B.pdim[1] * (k - B.plo[2]);
    return B.ghost[dir][idx];
}

// ------------------------------------------------------------------ arithmetic

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

template <int V>
struct IntC {
    static constexpr int value = V;
};

// L2 cache-policy loads/stores (BS_MGS_HINT 2): evict_last for the data the
// next GMRES pass re-reads first, evict_first for the rest.
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t pol;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ld_pol(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_pol(double2 *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// x / 6 correctly rounded (= __ddiv_rn(x, 6.0), the reference's division by
// the diagonal, inner_solvers.py:88) without the reciprocal refinement the
// compiler repeats per division: with z = RN(1/6) (relative error 2^-54),
// q = RN(x z) is within one ulp of x / 6, the residual e = x - 6 q is exact in
// one FMA, and RN(q + e z) is the correctly rounded quotient (Markstein's
// correction step; 6's significand is not all ones).  Zeros, subnormal-range
// and huge operands take the generic division.
__device__ __noinline__ double div6_generic(double x) { return __ddiv_rn(x, 6.0); }
__device__ __forceinline__ double div6(double x) {
    const unsigned ex = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
    if (ex - 200u > 1600u) return div6_generic(x);
    const double z = 0x1.5555555555555p-3;
    const double q = __dmul_rn(x, z);
    const double e = __fma_rn(-6.0, q, x);
    return __fma_rn(e, z, q);
}

// One CSR row of the 7-point operator as numpy's reduceat evaluates it
// (linalg.py:188-193): present terms in ascending column order
// t = [-zm, -ym, -xm, 6c, -xp, -yp, -zp], y = t_first + (((t_a + t_b) + ...)).
// Absent neighbours carry exact zeros inside the left-to-right chain (which
// leaves every partial sum unchanged), so only the choice of the first term
// depends on presence; the centre is always present.
__device__ __forceinline__ double stencil7(double zm, double ym, double xm, double c, double xp,
                                           double yp, double zp, bool pz, bool py, bool px) {
    const double t3 = mul(6.0, c);
    if (pz) return add(-zm, add(add(add(add(add(-ym, -xm), t3), -xp), -yp), -zp));
    if (py) return add(-ym, add(add(add(add(-xm, t3), -xp), -yp), -zp));
    if (px) return add(-xm, add(add(add(t3, -xp), -yp), -zp));
    return add(t3, add(add(-xp, -yp), -zp));
}

// One row of the operator without its diagonal (linalg.py:144-159) under the
// same reduceat rule: present terms [-zm, -ym, -xm, -xp, -yp, -zp], the first
// present one plus the left-to-right sum of those after it (absent ones are
// exact zeros there).  Without any lower neighbour the upper flags decide
// which term leads; a row with no neighbour at all is an empty segment (0).
__device__ __forceinline__ double offdiag6(double zm, double ym, double xm, double xp, double yp, double zp, bool pz,
                                           bool py, bool px, bool qx, bool qy, bool qz) {
    if (pz) return add(-zm, add(add(add(add(-ym, -xm), -xp), -yp), -zp));
    if (py) return add(-ym, add(add(add(-xm, -xp), -yp), -zp));
    if (px) return add(-xm, add(add(-xp, -yp), -zp));
    if (qx) return add(-xp, add(-yp, -zp));
    if (qy) return add(-yp, -zp);
    if (qz) return -zp;
    return 0.0;
}

// Rows on a region face: rhs = b - C*halo with the coupling row summed by the
// reduceat rule (entries of -1 in ascending column order, first + seq(rest);
// multisplit.py:333-338), and (want_global) the global operator row on the
// gathered iterate for the true residual (residual_norms).  Out of line: only
// face rows call it.
__device__ __noinline__ void face_coupling(const DBlock &B, int gi, int gj, int gk, double bv, double zm, double ym,
                                           double xm, double c, double xp, double yp, double zp, bool want_global,
                                           double &rhs, double &rg_au) {
    const int ni[6] = {gi, gi, gi - 1, gi + 1, gi, gi};
    const int nj[6] = {gj, gj - 1, gj, gj, gj + 1, gj};
    const int nk[6] = {gk - 1, gk, gk, gk, gk, gk + 1};
    double firstc = 0.0, rest = 0.0;
    int cnt = 0;
    double v[6] = {zm, ym, xm, xp, yp, zp};
    bool pg[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        pg[d] = in_grid(B, ni[d], nj[d], nk[d]);
        if (pg[d] && !in_region(B, ni[d], nj[d], nk[d])) {
            const double h = ghost_at(B, ni[d], nj[d], nk[d], d);
            v[d] = h;  // the global operator sees the coupled value
            if (cnt == 0) firstc = -h;
            else if (cnt == 1) rest = -h;
            else rest = add(rest, -h);
            ++cnt;
        }
    }
    if (cnt) rhs = sub(bv, cnt == 1 ? firstc : add(firstc, rest));
    if (want_global) rg_au = stencil7(v[0], v[1], v[2], c, v[3], v[4], v[5], pg[0], pg[1], pg[2]);
}

// Box blocks (overlap 0): the same on local coordinates — a neighbour across
// a block face is coupled iff that face is not a grid face, and its value is
// the face plane's entry; no region tests, no local arrays.
__device__ __forceinline__ void face_coupling_box(const DBlock &B, int lx, int ly, int lz, double bv, double zm,
                                                  double ym, double xm, double c, double xp, double yp, double zp,
                                                  bool want_global, double &rhs, double &rg_au) {
    const int pdx = B.pdim[0], pdy = B.pdim[1], pdz = B.pdim[2];
    // coupled (in the grid, outside the block) and in-block presence per direction
    const bool cz0 = lz == 0 && B.plo[2] > 0, cy0 = ly == 0 && B.plo[1] > 0, cx0 = lx == 0 && B.plo[0] > 0;
    const bool cx1 = lx == pdx - 1 && B.plo[0] + pdx < B.gn[0];
    const bool cy1 = ly == pdy - 1 && B.plo[1] + pdy < B.gn[1];
    const bool cz1 = lz == pdz - 1 && B.plo[2] + pdz < B.gn[2];
    if (!(cz0 | cy0 | cx0 | cx1 | cy1 | cz1)) {  // only grid faces: no coupling
        if (want_global) rg_au = stencil7(zm, ym, xm, c, xp, yp, zp, lz > 0, ly > 0, lx > 0);
        return;
    }
    double h[6];
    h[0] = cz0 ? B.ghost[0][lx + pdx * ly] : 0.0;
    h[1] = cy0 ? B.ghost[1][lx + pdx * lz] : 0.0;
    h[2] = cx0 ? B.ghost[2][ly + pdy * lz] : 0.0;
    h[3] = cx1 ? B.ghost[3][ly + pdy * lz] : 0.0;
    h[4] = cy1 ? B.ghost[4][lx + pdx * lz] : 0.0;
    h[5] = cz1 ? B.ghost[5][lx + pdx * ly] : 0.0;
    const bool cp[6] = {cz0, cy0, cx0, cx1, cy1, cz1};
    double firstc = 0.0, rest = 0.0;
    int cnt = 0;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        if (!cp[d]) continue;
        if (cnt == 0) firstc = -h[d];
        else if (cnt == 1) rest = -h[d];
        else rest = add(rest, -h[d]);
        ++cnt;
    }
    rhs = sub(bv, cnt == 1 ? firstc : add(firstc, rest));
    if (want_global)
        rg_au = stencil7(cz0 ? h[0] : zm, cy0 ? h[1] : ym, cx0 ? h[2] : xm, c, cx1 ? h[3] : xp, cy1 ? h[4] : yp,
                         cz1 ? h[5] : zp, lz > 0 || cz0, ly > 0 || cy0, lx > 0 || cx0);
}

// ------------------------------------------------------------------ TMA / mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Wait for a TMA stage.  A transfer that never completes (a bug, never a
// legal state) traps after ~4 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const unsigned long long t0 = global_ns();
    for (unsigned n = 1;; ++n) {
        if (mbar_try(bar, parity)) return;
        if ((n & 1023u) == 0 && global_ns() - t0 > 4000000000ull) asm volatile("trap;");
    }
}

__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                          uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------ reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic CTA reduction of NQ values over all NTH threads; result
// valid in thread 0.  `red` holds NQ x (NTH/32) doubles of shared memory.
template <int NTH>
__device__ __forceinline__ void cta_sum(double (&acc)[NQ], double *red) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NTH / 32;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double v = warp_sum(acc[q]);
        if (lane == 0) red[q * NW + warp] = v;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double s = red[q * NW];
            for (int w = 1; w < NW; ++w) s = add(s, red[q * NW + w]);
            acc[q] = s;
        }
    }
}

// Sum of partials[begin:end) in a fixed order: 256 virtual lanes, lane l
// sums part[begin + l + 256 k] (k ascending), then a binary tree pairing
// l with l + w for w = 128, 64, ..., 1.  The lane sums are spread over the
// CTA (all loads in flight at once); warp 0 then folds the tree levels
// 128 / 64 / 32 in registers (lane t holds virtual lanes t + 32 m) and the
// last five with shuffles — the same tree, so the same bits, as a
// shared-memory tree over 256 threads, with three CTA barriers instead of
// ten.  All NTH threads call it and get the sum (scratch: 256 doubles).
// Consumer-warps-only CTA barrier (named barrier 1): in multi-tile sweeps the
// producer warp is already streaming the next tile meanwhile.
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

template <int NTH, bool CONSUMERS = false>
__device__ double range_sum(const double *part, int begin, int end, double *scratch) {
    static_assert(NTH >= 32, "range_sum needs a full warp");
    static_assert(!CONSUMERS || NTH == NT, "the consumer-only form runs on the NT consumer threads");
    auto sync = [] {
        if (CONSUMERS) consumer_sync();
        else __syncthreads();
    };
    const int tid = threadIdx.x;
    for (int l = tid; l < 256; l += NTH) {
        double s = 0.0;
        for (int c = begin + l; c < end; c += 256) s = add(s, __ldcg(part + c));
        scratch[l] = s;
    }
    sync();
    if (tid < 32) {
        double v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = scratch[tid + 32 * m];
#pragma unroll
        for (int m = 0; m < 4; ++m) v[m] = add(v[m], v[m + 4]);  // w = 128
        v[0] = add(v[0], v[2]);                                    // w = 64
        v[1] = add(v[1], v[3]);
        double t = add(v[0], v[1]);                                // w = 32
#pragma unroll
        for (int w = 16; w > 0; w >>= 1) t = add(t, __shfl_down_sync(0xffffffffu, t, w));
        if (tid == 0) scratch[0] = t;
    }
    sync();
    const double out = scratch[0];
    sync();
    return out;
}

// ------------------------------------------------------------------ tracing (BS_TRACE builds)
// Per-CTA globaltimer stamps of the last traced launch: [0] entry, [1] first
// stage landed, [2] last plane done, [3] epilogue done.
#ifdef BS_TRACE
constexpr int TRACE_CTAS = 4096;
__device__ unsigned long long g_trace[5][TRACE_CTAS];  // [4] = SM id
// persistent kernel: [sweep][stamp][cta] for the first PT_SWEEPS sweeps:
// 0 sweep start, 1 tiles done, 2 partials written, 3 barrier released,
// 4 = SM clock at stamp 0 (low 48 bits) | SM id << 48
constexpr int PT_SWEEPS = 2048, PT_CTAS = 448;
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ unsigned long long g_ptrace[PT_SWEEPS][5][PT_CTAS];  // [4]: SM clock at stamp 0
#define BS_PSTAMP(sw, i)                                                             \
    do {                                                                             \
        if (threadIdx.x == 0 && blockIdx.x < PT_CTAS) {                              \
            g_ptrace[(sw) % PT_SWEEPS][(i)][blockIdx.x] = global_ns();               \
            if ((i) == 0) g_ptrace[(sw) % PT_SWEEPS][4][blockIdx.x] = (clock64() & 0xFFFFFFFFFFFFull) | ((unsigned long long)smid() << 48); \
        }                                                                            \
    } while (0)
// streaming kernel: [sweep][stamp][cta], stamps 0..6 (see k_cg_stream), [7] SM clock at stamp 0
__device__ unsigned long long g_strace[PT_SWEEPS][8][PT_CTAS];
#define BS_SSTAMP(sw, i)                                                             \
    do {                                                                             \
        if (threadIdx.x == 0 && blockIdx.x < PT_CTAS) {                              \
            g_strace[(sw) % PT_SWEEPS][(i)][blockIdx.x] = global_ns();               \
            if ((i) == 0) g_strace[(sw) % PT_SWEEPS][7][blockIdx.x] = (clock64() & 0xFFFFFFFFFFFFull) | ((unsigned long long)smid() << 48); \
        }                                                                            \
    } while (0)
#define BS_STAMP(i)                                                                  \
    do {                                                                             \
        if ((threadIdx.x == 0 || threadIdx.x == NT) && blockIdx.x < TRACE_CTAS)       \
            g_trace[i][blockIdx.x] = global_ns();                                   \
    } while (0)
#else
#define BS_STAMP(i) \
    do {            \
    } while (0)
#define BS_PSTAMP(sw, i) \
    do {                 \
    } while (0)
#define BS_SSTAMP(sw, i) \
    do {                 \
    } while (0)
#endif

// ------------------------------------------------------------------ sweep

struct SweepCtx {
    const DBlock *B;
    bool pend, first, want_global;
    double alpha_pend, beta, alpha;
    const CUtensorMap *map_a;  // stencil operand (haloed)
    const CUtensorMap *map_b;  // second stencil operand (haloed) or null
    const CUtensorMap *map_c;  // epilogue operand (bare tile) or null
    double *pout;              // S1: p[1-pcur]
    double *yout;              // APPLY output
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Process one tile (TX x TY cells, planes [lz0, lz1) of the padded box).
//
// Warp roles: warps 0..NCW-1 consume (thread = one column, RY rows), warp NCW
// produces: its lane 0 streams plane q = 0..nplanes-1 (lz = lz0-1+q) into
// stage q % NS with TMA, after every consumer warp released that stage's
// previous plane (empty mbarrier, count NCW).  Consumers never block on each
// other — only on `full` — so there is no CTA-wide barrier per plane.  All
// tiles of a launch stream z in lockstep, so neighbouring tiles read the same
// DRAM rows at about the same time.
//
// BOX (overlap 0, region == padded box): TMA zero-fill supplies the absent
// neighbours, presence tests are local-coordinate compares and couplings only
// exist on the box faces.  !BOX evaluates the L1-dilated region analytically.
//
// Direction: S2 walks its planes top-down (op_rev).  A CG iteration is S1
// then S2, so consecutive sweeps always run in opposite z order and the
// planes one sweep touched last (still in the 126 MB L2) are the first the
// next one reads.  Per point the arithmetic is the same in both directions
// (the stencil chain is fixed by column order, not by traversal); only the
// order of a thread's partial sums moves, deterministically per op.
// g0 < 0: the tile owns the ring (initialised here, one tile per ring).
// g0 >= 0: the ring is shared by a sequence of tiles (multi-tile CTAs):
// initialised once, and this tile's stages are ring-global stages g0, g0+1,
// ... — tiles follow each other with no gap in the ring, so the producer
// streams the next tile's first planes while the consumers finish this one.
// The consumers' plane loop stays aligned to ring rounds of NS stages (the
// compile-time stage schedule below): a tile starting at stage g0 % NS = o
// enters its first round at plane -o*ZP, whose planes < 1 belong to the
// previous tile and are skipped.  Returns the stages the tile used (0 for g0 < 0).
template <int OP, bool BOX>
__device__ int sweep_tile(const SweepCtx &C, int tile, unsigned char *smem, double (&acc)[NQ], int g0 = -1) {
    const DBlock &B = *C.B;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int pdx = B.pdim[0], pdy = B.pdim[1], pdz = B.pdim[2];
    const int tiles_x = B.tiles_x, tiles_y = B.tiles_y, cz = B.cz;
    int t = tile;
    const int ix = t % tiles_x;
    t /= tiles_x;
    const int iy = t % tiles_y;
    const int iz = t / tiles_y;
    const int lx0 = ix * TX, ly0 = iy * TY;  // tile origin, padded-box coordinates
    const int lz0 = iz * cz;
    const int lz1 = min(lz0 + cz, pdz);
    const int nplanes = lz1 - lz0 + 2;       // q = 0..nplanes-1 <-> lz = lz0-1+q (lz1-q reversed)
    constexpr bool REV = op_rev(OP);
    constexpr int DZ = REV ? -1 : 1;
    const int lzq0 = REV ? lz1 : lz0 - 1;    // plane of q = 0; plane q is lzq0 + DZ*q

    constexpr int NS = op_stages(OP);
    constexpr int STB = op_stage_bytes(OP);
    constexpr int COFF = op_coff(OP);
    constexpr int ZP = op_zp(OP);     // planes per stage
    constexpr int BOFF = op_sega(OP); // B operand of a plane, from its A plane
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STB);
    uint64_t *empty = full + NS;
    const bool use_b = C.map_b != nullptr;
    const bool use_c = C.map_c != nullptr;
    // slot of plane q inside its stage's box (boxes run upwards in z)
    auto slot = [](int qq) { return REV ? ZP - 1 - qq % ZP : qq % ZP; };

    const bool shared_ring = g0 >= 0;
    const int nst = (nplanes + ZP - 1) / ZP;   // stages with data
    const int k0 = shared_ring ? g0 : 0;       // ring-global index of the tile's stage 0
    const int o = k0 % NS;                     // ring stage of the tile's stage 0
    if (!shared_ring) {
        if (tid == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], NCW);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
    }

    if (warp == NCW) {  // ---------------- TMA producer warp
        if (lane == 0) {
            for (int k = 0; k < nst; ++k) {  // stage k holds planes ZP*k .. ZP*k+ZP-1
                const int kg = k0 + k;
                const int s = kg % NS;
                if (kg >= NS) mbar_wait(&empty[s], (uint32_t)((kg / NS - 1) & 1));
                const int lz = REV ? lzq0 - ZP * k - (ZP - 1) : lzq0 + ZP * k;  // lowest plane of the box
                // ZP == 1: the bare operand only for computed planes; ZP > 1: always
                const bool epi = use_c && (ZP > 1 || (k >= 1 && k <= nplanes - 2));
                unsigned char *st = smem + s * STB;
                const uint32_t bytes =
                    (uint32_t)(ZP * SC * 8) * (use_b ? 2u : 1u) + (epi ? (uint32_t)(ZP * SEG_O) : 0u);
                mbar_expect_tx(&full[s], bytes);
                tma_load3(st, C.map_a, lx0 - 2, ly0 - 1, lz, &full[s]);
                if (use_b) tma_load3(st + BOFF, C.map_b, lx0 - 2, ly0 - 1, lz, &full[s]);
                if (epi) tma_load3(st + COFF, C.map_c, lx0, ly0, lz, &full[s]);
            }
        }
        __syncwarp();
        return shared_ring ? nst : 0;
    }

    // ---------------- consumers: thread (tx, ty) owns column x = lx0 + tx of
    // rows ly0 + ty*RY + r, r < RY; z-neighbours live in registers, the
    // thread's own y-neighbours too, x-neighbours and the rows above/below
    // come from the staged haloed plane.
    const int tx = tid % TX, ty = tid / TX;
    const int lx = lx0 + tx, ly_0 = ly0 + ty * RY;
    const int gi = B.plo[0] + lx;
    const long long plane = (long long)B.pitch * pdy;
    long long sx = (long long)lx + (long long)B.pitch * ((long long)ly_0 + (long long)pdy * (lzq0 + DZ));
    const double beta = C.beta, alpha = C.alpha, alpha_pend = C.alpha_pend;
    const bool pend = C.pend, first = C.first;
    const long long pitch = B.pitch;

    // pd: the residual sweep's `pend` flag — the run-time one, or a constant in
    // the lean rounds below (compiled once per value)
    auto val_p = [&](const unsigned char *st, int cell, bool pd) -> double {
        const double a = reinterpret_cast<const double *>(st)[cell];
        if (OP == OP_RESID) return pd ? add(a, mul(alpha_pend, reinterpret_cast<const double *>(st + BOFF)[cell])) : a;
        if (OP == OP_S1) return first ? a : add(a, mul(beta, reinterpret_cast<const double *>(st + BOFF)[cell]));
        return a;
    };
    // !BOX: a plane is `easy` for a warp when every point it computes lies at
    // L1 distance <= overlap-1 from the owned box.  Every in-grid neighbour of
    // such a point is then in the region (distance grows by at most 1 per
    // step), none sits on the padded box's edge unless the grid ends there,
    // and no coupling exists: the BOX logic (unmasked values, local-coordinate
    // presence, no face terms) is exact for it.  Only the outer shell of the
    // region (about 1% of a 514^3 block) takes the analytic path.
    bool easy = BOX;
    // u at (row gj_, x + dx) of plane lz (local z), masked to the region for !BOX
    auto uval_p = [&](const unsigned char *st, int cell, int dx, int gj_, int lz, bool pd) -> double {
        const double v = val_p(st, cell, pd);
        if (BOX || easy) return v;
        return in_region(B, gi + dx, gj_, B.plo[2] + lz) ? v : 0.0;
    };
    auto uval = [&](const unsigned char *st, int cell, int dx, int gj_, int lz) -> double {
        return uval_p(st, cell, dx, gj_, lz, pend);
    };
    int own[RY], gjr[RY];
    bool row_in[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
        own[r] = (ty * RY + r + 1) * SX + (tx + 2);
        gjr[r] = B.plo[1] + ly_0 + r;
        row_in[r] = lx < pdx && ly_0 + r < pdy;
    }

    const uint32_t par0 = (uint32_t)((k0 / NS) & 1);  // completion parity of the tile's first round
    double u_prev[RY], u_cur[RY];
    mbar_wait(&full[o], par0);
    if (tid == 0) BS_STAMP(1);
#pragma unroll
    for (int r = 0; r < RY; ++r) u_prev[r] = uval(smem + o * STB + slot(0) * (SC * 8), own[r], 0, gjr[r], lzq0);
    const int s1 = ZP == 1 ? (k0 + 1) % NS : o;
    if (ZP == 1) mbar_wait(&full[s1], (uint32_t)(((k0 + 1) / NS) & 1));
    const unsigned char *st1 = smem + s1 * STB + slot(1) * (SC * 8);
#pragma unroll
    for (int r = 0; r < RY; ++r) u_cur[r] = uval(st1, own[r], 0, gjr[r], lzq0 + DZ);
    if (ZP == 1) {  // plane 0 is never computed: its stage is free (ZP > 1: plane 1 shares it)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[o]);
    }

    const bool px_box = lx > 0;
    // output pointers hoisted into registers: stores through them cannot alias
    // the block descriptor, so the compiler need not re-load it every plane
    double *__restrict__ out_r = B.r;
    double *__restrict__ out_x = B.x;
    double *__restrict__ out_w = B.W;
    double *__restrict__ out_p = C.pout;
    double *__restrict__ out_y = C.yout;
    // Plane q sits in stage q % NS and completes phase (q / NS) & 1.  The
    // loop below is unrolled by NS so both are compile-time per step: `s`
    // (this plane's stage), `sn` (the next plane's) and `par_n` (the next
    // plane's parity) are constants or one loop-carried bit.
    // u_prev / u_next are the planes behind / ahead in traversal order: the
    // z-1 / z+1 neighbours forward, z+1 / z-1 reversed.
    // plane q: stage s, slot sl; the next plane: stage sn, slot sln, waited
    // for only when it opens a new stage; the stage is released after its
    // last plane.
    // FC = std::true_type: a fast round — box region, full tile, and no plane
    // of the round without its z-1 neighbour — so no presence, row or region
    // test is evaluated per plane (only the uniform plane-range guard).
    // PC: the residual sweep's pend flag as a constant (0 / 1) or -1 = run time.
    // A fast round of the residual / Jacobi sweeps is *lean*: the round
    // selection below guarantees that none of its rows has a coupling, so
    // rhs = b and the global-row residual equals the local one — no face code
    // at all in the unrolled copy.
    auto single_step = [&](auto FC, auto PC, int q, int s, int sl, int sn, int sln, bool wait_next, uint32_t par_n,
                           bool release) {
        constexpr bool FR = decltype(FC)::value;
        constexpr int PK = decltype(PC)::value;
        const bool pd = PK < 0 ? pend : PK != 0;
        const int lz = lzq0 + DZ * q;
        const unsigned char *st = smem + s * STB + sl * (SC * 8);
        const double *cst = reinterpret_cast<const double *>(smem + s * STB + COFF + sl * SEG_O);
        // Phase A, before plane q+1 is waited for: the in-plane neighbours and,
        // on the interior fast path, the reduceat chain up to its last term
        // (z+1 enters second to last), so the wait overlaps the DP latency.
        if (!FR && !BOX && BS_EASY) {
            const int gk = B.plo[2] + lz;
            bool e = true;
#pragma unroll
            for (int r = 0; r < RY; ++r) e = e && (!row_in[r] || box_dist1(B, gi, gjr[r], gk) < B.overlap);
            easy = __all_sync(0xffffffffu, e);
        }
        // Fast path = stencil7's z-present branch, which never tests the x / y
        // flags: an absent x-1 / y-1 neighbour of a box (or easy) row lies
        // outside the padded box, where TMA zero-fills, and an exact zero
        // inside the chain leaves every partial sum unchanged.  So only the
        // z-1 presence selects it — tiles on the low x / y faces stream as
        // fast as interior ones (they used to finish each sweep last).
        const bool fast = FR || (easy && lz > 0);
        double xm_[RY], xp_[RY], ym_[RY], yp_[RY], pre_[RY];
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int gj = gjr[r];
            xm_[r] = uval_p(st, own[r] - 1, -1, gj, lz, pd);
            xp_[r] = uval_p(st, own[r] + 1, 1, gj, lz, pd);
            ym_[r] = r > 0 ? u_cur[r > 0 ? r - 1 : 0] : uval_p(st, own[r] - SX, 0, gj - 1, lz, pd);
            yp_[r] = r < RY - 1 ? u_cur[r < RY - 1 ? r + 1 : 0] : uval_p(st, own[r] + SX, 0, gj + 1, lz, pd);
            pre_[r] = fast ? add(add(add(add(-ym_[r], -xm_[r]), mul(6.0, u_cur[r])), -xp_[r]), -yp_[r]) : 0.0;
            // reversed: z+1 is the plane behind, so it enters the chain now
            if (REV && fast) pre_[r] = add(pre_[r], -u_prev[r]);
        }
        if (wait_next) mbar_wait(&full[sn], par_n & 1u);
        double u_next[RY];
#pragma unroll
        for (int r = 0; r < RY; ++r)
            u_next[r] = uval_p(smem + sn * STB + sln * (SC * 8), own[r], 0, gjr[r], lz + DZ, pd);
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            const int ly = ly_0 + r;
            const int gj = gjr[r];
            const bool here =
                FR || ((BOX || easy) ? row_in[r] : (row_in[r] && in_region(B, gi, gj, B.plo[2] + lz)));
            if (!here) continue;
            const double xm = xm_[r], xp = xp_[r], ym = ym_[r], yp = yp_[r];
            const double zm = REV ? u_next[r] : u_prev[r], zp = REV ? u_prev[r] : u_next[r];
            const long long sxr = sx + (long long)r * pitch;
            double au, od = 0.0;
            if (fast) {
                // = stencil7(zm, ym, xm, u_cur, xp, yp, zp, true, true, true), same association
                au = REV ? add(-zm, pre_[r]) : add(-zm, add(pre_[r], -zp));
                if (OP == OP_JAC) od = offdiag6(zm, ym, xm, xp, yp, zp, true, true, true, true, true, true);
            } else {
                bool pz, py, px;
                if (BOX || easy) {
                    pz = lz > 0;
                    py = ly > 0;
                    px = px_box;
                } else {
                    const int gk = B.plo[2] + lz;
                    pz = in_region(B, gi, gj, gk - 1);
                    py = in_region(B, gi, gj - 1, gk);
                    px = in_region(B, gi - 1, gj, gk);
                }
                au = stencil7(zm, ym, xm, u_cur[r], xp, yp, zp, pz, py, px);
                if (OP == OP_JAC) {
                    bool qz, qy, qx;
                    if (BOX || easy) {
                        qz = lz < pdz - 1;
                        qy = ly < pdy - 1;
                        qx = lx < pdx - 1;
                    } else {
                        const int gk = B.plo[2] + lz;
                        qz = in_region(B, gi, gj, gk + 1);
                        qy = in_region(B, gi, gj + 1, gk);
                        qx = in_region(B, gi + 1, gj, gk);
                    }
                    od = offdiag6(zm, ym, xm, xp, yp, zp, pz, py, px, qx, qy, qz);
                }
            }
            const int ci = (ty * RY + r) * TX + tx;  // bare-tile cell
            if (OP == OP_APPLY) {
                out_y[sxr] = au;
            } else if (OP == OP_GSPMV) {  // w = A v_j ; h_0j = v_0 . w (inner_solvers.py:187-190)
                out_w[sxr] = au;
                const double v0 = first ? u_cur[r] : cst[ci];
                acc[0] = add(acc[0], mul(v0, au));
            } else if (OP == OP_S2) {
                const double rnv = sub(cst[ci], mul(alpha, au));
                out_r[sxr] = rnv;
                acc[0] = add(acc[0], mul(rnv, rnv));
            } else if (OP == OP_S1) {
                out_p[sxr] = u_cur[r];
                if (pend)
                    out_x[sxr] = add(cst[ci], mul(alpha_pend, reinterpret_cast<const double *>(st + BOFF)[own[r]]));
                acc[0] = add(acc[0], mul(u_cur[r], au));
            } else if (FR) {  // lean round of OP_RESID / OP_JAC: no coupled row, rhs = b
                const double bv = cst[ci];
                const double rv = sub(bv, au);
                acc[0] = add(acc[0], mul(bv, bv));
                const double r2 = mul(rv, rv);
                acc[1] = add(acc[1], r2);
                if (OP == OP_JAC) {
                    out_p[sxr] = div6(sub(bv, od));
                } else {
                    out_r[sxr] = rv;
                    acc[3] = add(acc[3], r2);  // b - (global row) = rv bit for bit; acc[2]: see the tile's end
                }
            } else {  // OP_RESID: r = (b - C*halo) - A_ii u ; OP_JAC: also the Jacobi update
                const double bv = cst[ci];
                const int gk = B.plo[2] + lz;
                const bool face = BOX ? (lx == 0 || ly == 0 || lz == 0 || lx == pdx - 1 || ly == pdy - 1 ||
                                         lz == pdz - 1)
                                      : !easy;
                double rhs = bv, rg_au = au;
                if (face) {
                    if (BOX)
                        face_coupling_box(B, lx, ly, lz, bv, zm, ym, xm, u_cur[r], xp, yp, zp,
                                          OP == OP_RESID, rhs, rg_au);
                    else  // out of line: keeps the interior path lean
                        face_coupling(B, gi, gj, gk, bv, zm, ym, xm, u_cur[r], xp, yp, zp,
                                      OP == OP_RESID, rhs, rg_au);
                }
                const double rv = sub(rhs, au);
                if (OP == OP_JAC) {
                    // x_{k+1} = (rhs - offd x_k) / d (inner_solvers.py:88) ; ||rhs - A x_k||
                    out_p[sxr] = div6(sub(rhs, od));
                    acc[0] = add(acc[0], mul(rhs, rhs));
                    acc[1] = add(acc[1], mul(rv, rv));
                } else {
                    out_r[sxr] = rv;
                    acc[0] = add(acc[0], mul(rhs, rhs));
                    const double r2 = mul(rv, rv);
                    acc[1] = add(acc[1], r2);
                    if (BOX || in_owned(B, gi, gj, gk)) {
                        // box blocks own every row: acc[2] would repeat acc[1]
                        // add for add, so it is copied at the tile's end
                        if (!BOX) acc[2] = add(acc[2], r2);
                        const double rg = sub(bv, rg_au);
                        acc[3] = add(acc[3], mul(rg, rg));
                    }
                }
            }
        }
        sx += DZ * plane;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            u_prev[r] = u_cur[r];
            u_cur[r] = u_next[r];
        }
        if (release) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    };
    // q = 1 .. nplanes-2 in rounds of NS stages (NS*ZP planes) aligned to stage 0
    uint32_t par = par0;  // completion parity of the stages of this round
    const bool tile_full = lx0 + TX <= pdx && ly0 + TY <= pdy;
    // the computed plane with lz == 0 (no z-1 neighbour), if the tile has one
    const int q_zero = lz0 == 0 ? (REV ? lz1 : 1) : -1;
    // Residual / Jacobi sweeps: a fast round must not hold a coupled row
    // (rhs = b - C*halo, global row != block row).  Couplings sit on block
    // faces that are not grid faces: the tile's x / y face columns (tile_cpl)
    // and the planes lz == 0 (q_zero) and lz == pdz - 1 (q_top).
    constexpr bool LEAN = OP == OP_RESID || OP == OP_JAC;
    bool tile_cpl = false;
    int q_top = -1;
    if constexpr (LEAN && BOX) {
        tile_cpl = (lx0 == 0 && B.plo[0] > 0) || (lx0 + TX >= pdx && B.plo[0] + pdx < B.gn[0]) ||
                   (ly0 == 0 && B.plo[1] > 0) || (ly0 + TY >= pdy && B.plo[1] + pdy < B.gn[1]);
        if (lz1 == pdz && B.plo[2] + pdz < B.gn[2]) q_top = REV ? 1 : nplanes - 2;
    }
    for (int q0 = -o * ZP; q0 <= nplanes - 2; q0 += NS * ZP, par ^= 1u) {
        constexpr int QR = NS * ZP;  // planes per round
        // measured per op: the CG sweeps take both fast variants; the residual,
        // Jacobi and GMRES sweeps only the unguarded one (a third unrolled
        // copy makes them spill); the standalone SpMV none (its general path
        // is already short)
        constexpr bool FAST_ROUNDS = BOX && OP != OP_APPLY;
        constexpr bool GUARDED_FAST = OP == OP_S1 || OP == OP_S2;
        bool fround = false;
        if constexpr (FAST_ROUNDS)
            fround = tile_full && !(q_zero >= q0 && q_zero < q0 + QR) &&
                     !(LEAN && (tile_cpl || (q_top >= q0 && q_top < q0 + QR)));
        if (fround && q0 >= 1 && q0 + QR - 1 <= nplanes - 2) {  // interior round: no guards at all
            if (OP == OP_RESID && pend) {
#pragma unroll
                for (int u = 0; u < QR; ++u) {
                    const int un = u + 1;
                    single_step(std::true_type{}, IntC<1>{}, q0 + u, u / ZP, slot(u), (un / ZP) % NS, slot(un),
                                un % ZP == 0, un == QR ? par ^ 1u : par, u % ZP == ZP - 1);
                }
            } else {
#pragma unroll
                for (int u = 0; u < QR; ++u) {
                    const int un = u + 1;
                    single_step(std::true_type{}, IntC<(OP == OP_RESID ? 0 : -1)>{}, q0 + u, u / ZP, slot(u),
                                (un / ZP) % NS, slot(un), un % ZP == 0, un == QR ? par ^ 1u : par, u % ZP == ZP - 1);
                }
            }
        } else if (GUARDED_FAST && fround) {  // first / last round: the uniform plane-range guard only
#pragma unroll
            for (int u = 0; u < QR; ++u) {
                const int q = q0 + u;
                const int un = u + 1;
                if (q >= 1 && q <= nplanes - 2)
                    single_step(std::true_type{}, IntC<-1>{}, q, u / ZP, slot(u), (un / ZP) % NS, slot(un), un % ZP == 0,
                                un == QR ? par ^ 1u : par, u % ZP == ZP - 1);
            }
        } else {
#pragma unroll
            for (int u = 0; u < QR; ++u) {
                const int q = q0 + u;
                const int un = u + 1;
                if (q >= 1 && q <= nplanes - 2)
                    single_step(std::false_type{}, IntC<-1>{}, q, u / ZP, slot(u), (un / ZP) % NS, slot(un), un % ZP == 0,
                                un == QR ? par ^ 1u : par, u % ZP == ZP - 1);
            }
        }
    }
    // box blocks own every row: the owned-row sum is the all-row sum
    if (OP == OP_RESID && BOX) acc[2] = acc[1];
    if (tid == 0) BS_STAMP(2);
    if (shared_ring) {
        // release the stages the plane loop did not (the one holding only the
        // last, never computed, plane) — after waiting for each, so no
        // barrier can run a phase ahead of the producer's wait
        const int released = (nplanes - 1 - ZP) / ZP + 1;
        __syncwarp();
        for (int k = released; k < nst; ++k) {
            const int kg = k0 + k;
            mbar_wait(&full[kg % NS], (uint32_t)((kg / NS) & 1));
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[kg % NS]);
        }
        return nst;
    }
    return 0;
}

// ------------------------------------------------------------------ scalars

// ---- restarted GMRES(m) scalar recurrences (inner_solvers.py:149-251)

__device__ void gmres_start_cycle(DState &S, GState &G, double beta, double rel) {
    S.cycle_start = rel;  // inner_solvers.py:159
    G.g[0] = beta;
    S.gnrm = beta;        // v_0 = r / beta
    S.gj = 0;
    S.gi = 0;
    S.gflag = GF_NONE;
    S.phase = PH_G_NORM;
}

// y = H[:j+1,:j+1] \ g[:j+1] (inner_solvers.py:246-251)
__device__ void gmres_back_substitute(GState &G, int j) {
    for (int i = j; i >= 0; --i) {
        double s = 0.0;
        for (int k = i + 1; k <= j; ++k) s = add(s, mul(G.H[i * MAXM + k], G.y[k]));
        G.y[i] = __ddiv_rn(sub(G.g[i], s), G.H[i * MAXM + i]);
    }
}

__device__ __noinline__ void gmres_transition(const DBlock &B, DState &S, GState &G, int ph, const double *q) {
    switch (ph) {
        case PH_INIT: {  // inner_solvers.py:153-164
            for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
            const double bn = sqrt(q[0]);
            S.scale = bn > 0.0 ? bn : 1.0;
            const double beta = sqrt(q[1]);
            const double rel = beta / S.scale;
            S.rel = rel;
            S.tol_eff = S.basis == BS_BASIS_INITIAL ? S.tol * rel : S.tol;
            S.it = 0;
            if (rel <= S.tol_eff) {
                S.stop = BS_STOP_TOLERANCE_MET;
                S.phase = PH_DONE;
            } else {
                gmres_start_cycle(S, G, beta, rel);
            }
            break;
        }
        case PH_G_NORM:
            S.phase = PH_G_SPMV;
            break;
        case PH_G_SPMV:
            G.H[0 * MAXM + S.gj] = q[0];
            if (S.gj >= 1) {
                S.gi = 1;
                S.phase = PH_G_MGS;
            } else {
                S.phase = PH_G_FINAL;
            }
            break;
        case PH_G_MGS:
            G.H[S.gi * MAXM + S.gj] = q[0];
            if (S.gi < S.gj) S.gi += 1;
            else S.phase = PH_G_FINAL;
            break;
        case PH_G_FINAL: {  // inner_solvers.py:194-236
            const int j = S.gj;
            const double wnorm = sqrt(q[0]);
            G.H[(j + 1) * MAXM + j] = wnorm;
            double cn = 0.0;
            for (int r = 0; r <= j + 1; ++r) cn = add(cn, mul(G.H[r * MAXM + j], G.H[r * MAXM + j]));
            const bool happy = wnorm <= 1e-14 * fmax(sqrt(cn), 1e-300);
            for (int i = 0; i < j; ++i) {
                const double hi = G.H[i * MAXM + j], hi1 = G.H[(i + 1) * MAXM + j];
                const double hij = add(mul(G.cs[i], hi), mul(G.sn[i], hi1));
                G.H[(i + 1) * MAXM + j] = add(mul(-G.sn[i], hi), mul(G.cs[i], hi1));
                G.H[i * MAXM + j] = hij;
            }
            const double hjj = G.H[j * MAXM + j], hj1 = G.H[(j + 1) * MAXM + j];
            const double denom = hypot(hjj, hj1);
            G.cs[j] = __ddiv_rn(hjj, denom);
            G.sn[j] = __ddiv_rn(hj1, denom);
            G.H[j * MAXM + j] = denom;
            G.H[(j + 1) * MAXM + j] = 0.0;
            G.g[j + 1] = mul(-G.sn[j], G.g[j]);
            G.g[j] = mul(G.cs[j], G.g[j]);
            S.it += 1;
            const double rel = fabs(G.g[j + 1]) / S.scale;
            S.rel = rel;
            if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel;
            int flag = GF_NONE;
            if (happy) flag = GF_HAPPY;
            else if (rel <= S.tol_eff || S.it >= S.max_its) flag = GF_CHECK;
            else if (j == S.gm - 1) flag = GF_CYCLE;
            if (flag != GF_NONE) {
                gmres_back_substitute(G, j);
                S.gflag = flag;
                S.phase = PH_G_FORM;
            } else {
                S.gnrm = wnorm;  // v_{j+1} = w / wnorm (inner_solvers.py:237)
                S.gj = j + 1;
                S.gi = 0;
                S.phase = PH_G_NORM;
            }
            break;
        }
        case PH_G_FORM:
            S.phase = PH_G_RESID;
            break;
        case PH_G_RESID: {  // inner_solvers.py:215-243
            for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
            const double rel_true = sqrt(q[1]) / S.scale;
            S.rel = rel_true;
            if (S.gflag == GF_HAPPY) {
                if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel_true;
                S.stop = BS_STOP_TOLERANCE_MET;
                S.phase = PH_DONE;
                break;
            }
            if (S.gflag == GF_CHECK) {
                if (rel_true <= S.tol_eff) {
                    if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel_true;
                    S.stop = BS_STOP_TOLERANCE_MET;
                    S.phase = PH_DONE;
                    break;
                }
                if (S.it >= S.max_its) {
                    S.stop = BS_STOP_MAX_ITERATIONS;
                    S.phase = PH_DONE;
                    break;
                }
            }
            if (!isfinite(rel_true) || S.cycle_start - rel_true < 1e-14 * S.cycle_start) {
                S.stop = BS_STOP_BREAKDOWN;  // non-finite or stagnation over a cycle
                S.phase = PH_DONE;
                break;
            }
            gmres_start_cycle(S, G, sqrt(q[1]), rel_true);  // restart from r = b - A x
            break;
        }
        default:
            break;
    }
}

// rec = false: a redundant copy of the transition (the persistent kernel's
// non-recording CTAs) that must not write the block's history.
__device__ __noinline__ void cg_transition(const DBlock &B, DState &S, int ph, const double *q, bool rec = true) {
    const int hist_cap = rec ? B.hist_cap : 0;
    switch (ph) {
        case PH_INIT: {
            for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
            const double bn = sqrt(q[0]);
            S.scale = bn > 0.0 ? bn : 1.0;  // inner_solvers.py:70-72
            const double rel = sqrt(q[1]) / S.scale;
            S.rel = rel;
            S.tol_eff = S.basis == BS_BASIS_INITIAL ? S.tol * rel : S.tol;
            S.it = 0;
            if (rel <= S.tol_eff) {  // inner_solvers.py:110-113
                S.stop = BS_STOP_TOLERANCE_MET;
                S.phase = PH_DONE;
            } else {
                S.rr = q[1];
                S.first = 1;
                S.phase = PH_S1;
            }
            break;
        }
        case PH_S1: {  // inner_solvers.py:118-122
            const double pap = q[0];
            S.pend = 0;  // the deferred update was applied in this sweep
            S.pcur ^= 1;
            S.first = 0;
            if (!(pap > 0.0) || isinf(pap)) {
                S.stop = BS_STOP_BREAKDOWN;
                S.phase = PH_DONE;
            } else {
                S.alpha = S.rr / pap;
                S.phase = PH_S2;
            }
            break;
        }
        case PH_S2: {  // inner_solvers.py:123-145
            const double rr_new = q[0];
            S.it += 1;
            S.pend = 1;  // x += alpha p deferred to the next sweep
            S.alpha_pend = S.alpha;
            const double rel = sqrt(rr_new) / S.scale;
            S.rel = rel;
            if (S.it - 1 < hist_cap) B.hist[S.it - 1] = rel;
            if (!isfinite(rel)) {
                S.stop = BS_STOP_BREAKDOWN;
                S.phase = PH_DONE;
            } else if (rel <= S.tol_eff) {
                S.phase = PH_VERIFY;
            } else {
                S.beta = rr_new / S.rr;
                S.rr = rr_new;
                if (S.it >= S.max_its) {
                    S.stop = BS_STOP_MAX_ITERATIONS;
                    S.phase = PH_DONE;
                } else {
                    S.phase = PH_S1;
                }
            }
            break;
        }
        case PH_VERIFY: {  // inner_solvers.py:132-142
            const double rel_true = sqrt(q[1]) / S.scale;
            if (rel_true <= S.tol_eff) {
                S.rel = rel_true;
                if (S.it - 1 < hist_cap) B.hist[S.it - 1] = rel_true;
                S.stop = BS_STOP_TOLERANCE_MET;
                S.phase = PH_DONE;
            } else {
                const double rr_new = q[1];  // r = r_true
                const double rel = sqrt(rr_new) / S.scale;
                S.rel = rel;
                if (S.it - 1 < hist_cap) B.hist[S.it - 1] = rel;
                S.beta = rr_new / S.rr;
                S.rr = rr_new;
                if (S.it >= S.max_its) {
                    S.stop = BS_STOP_MAX_ITERATIONS;
                    S.phase = PH_DONE;
                } else {
                    S.phase = PH_S1;
                }
            }
            break;
        }
        case PH_RESID:
        case PH_OWNRES: {
            for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
            S.phase = PH_DONE;
            break;
        }
        default:
            break;
    }
}

// ---- point Jacobi (inner_solvers.py:75-99).  Sweep k reads x_k from
// buf[xin] (x or p[0]), reports ||rhs - A x_k|| and writes x_{k+1} into the
// other buffer; the solve stops at the first k whose x_k passes a test, so the
// answer is buf[xin] and k the iteration count.
__device__ __noinline__ void jacobi_transition(const DBlock &B, DState &S, int ph, const double *q) {
    const double rel_in = [&] {
        if (S.it == 0) {
            const double bn = sqrt(q[0]);
            S.scale = bn > 0.0 ? bn : 1.0;  // inner_solvers.py:70-72
        }
        return sqrt(q[1]) / S.scale;
    }();
    if (ph == PH_INIT) {  // residual sweep of the outer driver doubles as the initial check
        for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
        S.rel = rel_in;
        S.tol_eff = S.basis == BS_BASIS_INITIAL ? S.tol * rel_in : S.tol;
        S.xin = 0;
        if (rel_in <= S.tol_eff) {  // inner_solvers.py:85-87
            S.stop = BS_STOP_TOLERANCE_MET;
            S.phase = PH_DONE;
        } else {
            S.phase = PH_JAC;
        }
        return;
    }
    // PH_JAC, sweep k = S.it
    const int k = S.it;
    if (k == 0) S.tol_eff = S.basis == BS_BASIS_INITIAL ? S.tol * rel_in : S.tol;
    S.rel = rel_in;
    if (k > 0 && k - 1 < B.hist_cap) B.hist[k - 1] = rel_in;
    int stop = BS_STOP_NONE;
    if (k > 0 && !isfinite(rel_in)) stop = BS_STOP_BREAKDOWN;           // inner_solvers.py:93-94
    else if (rel_in <= S.tol_eff) stop = BS_STOP_TOLERANCE_MET;        // 85-87, 95-96
    else if (k >= S.max_its) stop = BS_STOP_MAX_ITERATIONS;             // 97
    if (stop != BS_STOP_NONE) {
        S.stop = stop;
        S.phase = PH_DONE;  // x_k stays in buf[xin]
    } else {
        S.xin ^= 1;  // x_{k+1} was written to the other buffer
        S.it = k + 1;
    }
}

__device__ void transition(const DBlock &B, DState &S, GState *G, int ph, const double *q, bool rec = true) {
    if (ph == PH_JAC || (ph == PH_INIT && S.kind == KIND_JACOBI)) {
        jacobi_transition(B, S, ph, q);
        return;
    }
    const bool gm = (ph >= PH_G_NORM && ph <= PH_G_RESID) || (ph == PH_INIT && S.kind == KIND_GMRES);
    if (gm) gmres_transition(B, S, *G, ph, q);
    else cg_transition(B, S, ph, q, rec);
}

// Does a launch of sweep op OPK (or pointwise pass PK when OPK < 0) serve this block?
template <int OPK, int PKK>
__device__ __forceinline__ bool serves(const DState &S, const KParams &P) {
    const int ph = S.phase;
    if (OPK == OP_S1) return ph == PH_S1;
    if (OPK == OP_S2) return ph == PH_S2;
    if (OPK == OP_RESID) return ph == PH_INIT || ph == PH_VERIFY || ph == PH_RESID || ph == PH_G_RESID;
    if (OPK == OP_GSPMV) return ph == PH_G_SPMV && S.gj == P.launch_j;
    if (OPK == OP_JAC) return ph == PH_JAC;
    if (PKK == PK_NORM) return ph == PH_G_NORM && S.gj == P.launch_j;
    if (PKK == PK_MGS) return ph == PH_G_MGS && S.gj == P.launch_j && S.gi == P.launch_i;
    if (PKK == PK_FINAL) return ph == PH_G_FINAL && S.gj == P.launch_j;
    if (PKK == PK_FORM) return ph == PH_G_FORM;
    if (PKK == PK_OWNRES) return ph == PH_OWNRES;
    return false;
}

// Per-tile partials -> the block's last CTA reduces them in tile order and
// advances the block's recurrence.  Every CTA then counts into the launch;
// the launch's last CTA publishes the loop conditions.  NTH = CTA threads.
// Block state as the other CTAs left it: L2 loads (a persistent kernel must
// not see a stale L1 copy from an earlier sweep).
__device__ __forceinline__ DState ld_state(const DState *p) {
    DState S;
    const int4 *src = reinterpret_cast<const int4 *>(p);
    int4 *dst = reinterpret_cast<int4 *>(&S);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(DState) / 16); ++i) dst[i] = __ldcg(src + i);
    return S;
}

// Only the head (what a sweep needs): 4 loads instead of sizeof/16, which
// matters when every CTA of a persistent grid reads the same block state.
__device__ __forceinline__ DState ld_state_head(const DState *p) {
    DState S;
    const int4 *src = reinterpret_cast<const int4 *>(p);
    int4 *dst = reinterpret_cast<int4 *>(&S);
#pragma unroll
    for (int i = 0; i < DSTATE_HEAD / 16; ++i) dst[i] = __ldcg(src + i);
    return S;
}

// Block-level part of a sweep's epilogue for tile `vcta` (the CTA index in a
// launch, or the tile a persistent CTA just swept).
template <int NTH, bool POINT = false>
__device__ void finish_block(const KParams &P, int b, int ph, bool served, double (&acc)[NQ], int nq,
                             unsigned char *smem, int vcta) {
    const int nctas = POINT ? P.npctas : P.nctas;
    const int tid = threadIdx.x;
    double *red = reinterpret_cast<double *>(smem);
    double *scratch = red + NQ * (NTH / 32);
    int *flag = reinterpret_cast<int *>(scratch + 256);
    if (served) {
        const DBlock &B = P.blocks[b];
        cta_sum<NTH>(acc, red);
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) P.partials[(size_t)q * nctas + vcta] = acc[q];
            __threadfence();
            const unsigned prev = atomicAdd(&P.blk_counter[b], 1u);
            const int span = POINT ? B.pcta_end - B.pcta_begin : B.cta_end - B.cta_begin;
            *flag = (prev == (unsigned)span - 1u);
        }
        __syncthreads();
        if (*flag) {  // last tile of block b
            __threadfence();
            const int c0 = POINT ? B.pcta_begin : B.cta_begin, c1 = POINT ? B.pcta_end : B.cta_end;
            double q[NQ];
            for (int i = 0; i < NQ; ++i)
                q[i] = i < nq ? range_sum<NTH>(P.partials + (size_t)i * nctas, c0, c1, scratch) : 0.0;
            if (tid == 0) {
                DState Sn = ld_state(P.states + b);
                transition(B, Sn, P.gstates ? P.gstates + b : nullptr, ph, q);
                P.states[b] = Sn;
                P.blk_counter[b] = 0u;
                __threadfence();
            }
        }
        __syncthreads();
    }
}

// Launch-level epilogue of a sweep: every CTA counts into the launch; the
// launch's last CTA publishes the loop conditions and rewinds the tile
// counter (flag: one int of shared memory).
template <int OPK>
__device__ void finish_launch(const KParams &P, int *flag) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(P.launch_counter, 1u);
        *flag = (prev == gridDim.x - 1u);
    }
    __syncthreads();
    if (!*flag || tid != 0) return;
    __threadfence();
    int active = 0, verify = 0;
    for (int bb = 0; bb < P.nblocks; ++bb) {
        const int p2 = ((volatile DState *)P.states)[bb].phase;
        if (p2 != PH_DONE && p2 != PH_IDLE) ++active;
        if (p2 == PH_VERIFY || p2 == PH_INIT || p2 == PH_RESID) ++verify;
    }
    if (OPK == OP_S2 || OPK == OP_JAC) {
        Control &ctl = *P.ctl;
        ctl.cycles += 1;
        if (ctl.max_cycles > 0 && ctl.cycles > ctl.max_cycles && active) {
            // runaway guard: never let a device-side loop spin forever
            for (int bb = 0; bb < P.nblocks; ++bb) {
                DState &Sb = P.states[bb];
                if (Sb.phase != PH_DONE && Sb.phase != PH_IDLE) {
                    Sb.phase = PH_DONE;
                    Sb.stop = STOP_STALLED;
                }
            }
            ctl.stalled = 1;
            active = 0;
            verify = 0;
        }
    }
    if (OPK == OP_RESID && P.use_graph) P.ctl->resid_runs += 1;
    *P.n_active = active;
    *P.launch_counter = 0u;
    *P.tile_counter = 0u;
    if (P.use_graph) {
        cudaGraphSetConditional(P.h_loop, active ? 1u : 0u);
        if (OPK == OP_S2) cudaGraphSetConditional(P.h_verify, verify ? 1u : 0u);
    }
}

// Tile epilogue of a multi-tile sweep, on the consumer warps only (the
// producer is streaming the next tile): the tile partial with cta_sum<NTHR>'s
// exact order (warps 0..NCW-1, then the producer warp's +0.0), and the
// block's last tile reduces the block in tile order and advances it — the
// same numbers as finish_block.
__device__ void tile_epilogue(const KParams &P, int b, int ph, double (&acc)[NQ], int nq, int cta, double *red,
                              double *scratch, int *flag) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q * NCW + warp] = v;
    }
    consumer_sync();
    const DBlock &B = P.blocks[b];
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double sum = red[q * NCW];
            for (int w = 1; w < NCW; ++w) sum = add(sum, red[q * NCW + w]);
            P.partials[(size_t)q * P.nctas + cta] = add(sum, 0.0);
        }
        __threadfence();
        const unsigned prev = atomicAdd(&P.blk_counter[b], 1u);
        *flag = (prev == (unsigned)(B.cta_end - B.cta_begin) - 1u);
    }
    consumer_sync();
    if (*flag) {  // last tile of block b
        __threadfence();
        double q[NQ];
        for (int i = 0; i < NQ; ++i)
            q[i] = i < nq ? range_sum<NT, true>(P.partials + (size_t)i * P.nctas, B.cta_begin, B.cta_end, scratch) : 0.0;
        if (tid == 0) {
            DState Sn = ld_state(P.states + b);
            transition(B, Sn, P.gstates ? P.gstates + b : nullptr, ph, q);
            P.states[b] = Sn;
            P.blk_counter[b] = 0u;
            __threadfence();
        }
    }
    consumer_sync();  // red / flag are reused by the next tile
}

template <int NTH, int OPK, bool POINT = false>
__device__ void finish(const KParams &P, int b, int ph, bool served, double (&acc)[NQ], int nq,
                       unsigned char *smem, int vcta) {
    finish_block<NTH, POINT>(P, b, ph, served, acc, nq, smem, vcta);
    // Pointwise (GMRES) passes are host-sequenced and never end a loop: the
    // launch-level bookkeeping (one atomic per CTA on a single counter) is
    // only needed by sweeps.
    if (POINT) return;
    finish_launch<OPK>(P, reinterpret_cast<int *>(reinterpret_cast<double *>(smem) + NQ * (NTH / 32) + 256));
}

// One sweep over every block whose phase this kernel serves.
template <int OPK>
__device__ __forceinline__ SweepCtx make_ctx(const KParams &P, int b, const DBlock &B, const DState &S) {
        const CUtensorMap *tm = P.tmaps + (size_t)b * NTM;
        SweepCtx C;
        C.B = &B;
        C.pend = S.pend != 0;
        C.first = S.first != 0;
        C.want_global = true;
        C.alpha_pend = S.alpha_pend;
        C.alpha = S.alpha;
        C.beta = S.beta;
        C.yout = nullptr;
        C.pout = B.p[S.pcur ^ 1];
        const CUtensorMap *tm_p1 = tm + (S.pcur ? TM_P1H_S1 : TM_P0H_S1);
        if (OPK == OP_RESID) {
            C.map_a = tm + (S.xin ? TM_P0H_R : TM_XH_R);
            C.map_b = C.pend ? tm + (S.pcur ? TM_P1H_R : TM_P0H_R) : nullptr;
            C.map_c = tm + TM_BO_R;
        } else if (OPK == OP_JAC) {  // x_k haloed from buf[xin], b bare; x_{k+1} -> other buffer
            C.map_a = tm + (S.xin ? TM_P0H_J : TM_XH_J);
            C.map_b = nullptr;
            C.map_c = tm + TM_BO_J;
            C.pout = S.xin ? B.x : B.p[0];
        } else if (OPK == OP_S1) {
            C.map_a = tm + TM_RH_S1;
            C.map_b = (!C.first || C.pend) ? tm_p1 : nullptr;
            C.map_c = C.pend ? tm + TM_XO_S1 : nullptr;
        } else if (OPK == OP_S2) {
            C.map_a = tm + (S.pcur ? TM_P1H_S2 : TM_P0H_S2);
            C.map_b = nullptr;
            C.map_c = tm + TM_RO_S2;
        } else {  // OP_GSPMV: u = v_j (haloed), epilogue operand v_0 (bare)
            const CUtensorMap *gm = P.gmaps + (size_t)b * (MAXM + 1);
            C.first = S.gj == 0;
            C.map_a = gm + S.gj;
            C.map_b = nullptr;
            C.map_c = C.first ? nullptr : gm + MAXM;
        }
        return C;
}

template <int OPK>
__host__ __device__ constexpr int op_nq() { return OPK == OP_RESID ? NQ : (OPK == OP_JAC ? 2 : 1); }

__host__ __device__ constexpr int op_minblocks(int op) {
    return (op == OP_RESID || op == OP_JAC) ? BS_MINBLOCKS_HEAVY : BS_MINBLOCKS;
}

template <int OPK, bool BOX>
__global__ void __launch_bounds__(NTHR, op_minblocks(OPK)) k_sweep(const KParams P) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ double s_red[NQ * NCW];
    __shared__ double s_scratch[256];
    __shared__ int s_flag, s_tile[2];
    __shared__ __align__(8) uint64_t s_tfull[2], s_tempty[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) BS_STAMP(0);
#ifdef BS_TRACE
    if (tid == 0 && blockIdx.x < TRACE_CTAS) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace[4][blockIdx.x] = sm;
    }
#endif
    // Each CTA streams tiles back to back through ONE ring: the producer runs
    // into the next tile while the consumers finish the last planes and the
    // epilogue of this one (no per-tile ring fill or CTA launch).  Tiles are
    // handed out dynamically (one counter per launch), so CTAs on busier SMs
    // simply take fewer; the producer lane fetches the next index and passes
    // it to the consumer warps through a two-slot mailbox.  Reversed sweeps
    // take the tiles in reverse order (the previous sweep's last tiles are
    // still in L2).  Results do not depend on the assignment: partials are
    // per tile.
    if (tid == 0) {
        uint64_t *full = reinterpret_cast<uint64_t *>(smem + op_stages(OPK) * op_stage_bytes(OPK));
        for (int s = 0; s < op_stages(OPK); ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&full[op_stages(OPK) + s], NCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_tfull[s], 1);
            mbar_init(&s_tempty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const int T = P.ntiles;
    int gstage = 0;  // ring-global stage of the next tile
    for (int n = 0;; ++n) {
        const int slot = n & 1;
        const uint32_t ph = (uint32_t)((n >> 1) & 1);
        int i = 0;
        if (warp == NCW) {
            if (lane == 0) {
                if (n >= 2) mbar_wait(&s_tempty[slot], ph ^ 1u);  // the slot's previous index was read
                i = (int)atomicAdd(P.tile_counter, 1u);
                s_tile[slot] = i;
                mbar_arrive(&s_tfull[slot]);
            }
            i = __shfl_sync(0xffffffffu, i, 0);
        } else {
            mbar_wait(&s_tfull[slot], ph);
            i = s_tile[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_tempty[slot]);
        }
        if (i >= T) break;
        const int cta = P.cta_base + (op_rev(OPK) ? T - 1 - i : i);
        const int b = P.cta_block[cta];
        const DBlock &B = P.blocks[b];
        const DState S = P.states[b];  // constant until every tile of b is done
        if (!serves<OPK, -1>(S, P)) continue;
        double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
        const SweepCtx C = make_ctx<OPK>(P, b, B, S);
        gstage += sweep_tile<OPK, BOX>(C, cta - B.cta_begin, smem, acc, gstage);
        if (tid < NT) tile_epilogue(P, b, S.phase, acc, op_nq<OPK>(), cta, s_red, s_scratch, &s_flag);
    }
    __syncthreads();
    finish_launch<OPK>(P, &s_flag);
    if (tid == 0) BS_STAMP(3);
}

// ---- persistent CG: the whole solve in one cooperative launch.  Each CTA
// sweeps tiles blockIdx.x, +gridDim.x, ...; sweeps are separated by a
// software grid barrier whose last arriver evaluates the loop conditions that
// the graph's conditional nodes evaluate otherwise.  Removes the per-launch
// fill/drain and launch gaps (~14 us per sweep at 256^3) from every sweep.

// central: the grid barrier's last arriver reduces every block (few blocks);
// otherwise each block's last tile does (finish_block).  Both sum the tile
// partials with range_sum in tile order, so results match the launch path.
constexpr int CENTRAL_MAX = 4;

template <int OPK, bool BOX>
__device__ void persist_sweep(const KParams &P, unsigned char *smem, const DState *s_states, bool central,
                              int sw, double *part, bool local = false) {
    BS_PSTAMP(sw, 0);
    for (int t0 = blockIdx.x; t0 < P.nctas; t0 += gridDim.x) {
        const int t = op_rev(OPK) ? P.nctas - 1 - t0 : t0;  // as k_sweep
        const int b = P.cta_block[t];
        const DBlock &B = P.blocks[b];
        const DState S = local ? s_states[b] : central ? ld_state_head(P.states + b) : ld_state(P.states + b);
        const int ph = S.phase;
        const bool served = serves<OPK, -1>(S, P);
        double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
        if (served) {
            const SweepCtx C = make_ctx<OPK>(P, b, B, S);
            sweep_tile<OPK, BOX>(C, t - B.cta_begin, smem, acc);
            __syncthreads();
            BS_PSTAMP(sw, 1);
            // retire this op's mbarriers: the next sweep reuses the memory
            // (other ops place their ring and barriers differently)
            if (threadIdx.x == 0) {
                uint64_t *bars = reinterpret_cast<uint64_t *>(smem + op_stages(OPK) * op_stage_bytes(OPK));
                for (int i = 0; i < 2 * op_stages(OPK); ++i)
                    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + i)) : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (central) {
            if (served) {
                cta_sum<NTHR>(acc, reinterpret_cast<double *>(smem));
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) part[(size_t)q * P.nctas + t] = acc[q];
                }
                BS_PSTAMP(sw, 2);
            }
        } else {
            finish_block<NTHR>(P, b, ph, served, acc, op_nq<OPK>(), smem, t);
        }
    }
}

// Grid barrier after a sweep of op OPK (the cooperative-groups pattern:
// CTA barrier, one release/acquire round on a counter and a generation word
// per CTA).  Generic-proxy stores of this sweep are fenced against the next
// sweep's TMA (async-proxy) reads on both sides.  Central mode: the last
// arriver reduces and advances every block on its shared-memory copies of
// the block states and publishes them with the loop conditions.  On return
// s_states holds every block's new state (central mode).
template <int OPK>
__device__ void grid_sync(const KParams &P, unsigned char *smem, DState *s_states, bool central, unsigned &gen_ref,
                          int sw) {
    __shared__ int s_last;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    Control *ctl = P.ctl;
    volatile unsigned *gen = &ctl->bar_gen;
    const unsigned g = gen_ref;
    if (threadIdx.x == 0) {
#ifdef BS_BAR_FENCES
        __threadfence();
        s_last = atomicAdd(&ctl->bar_count, 1u) == gridDim.x - 1;
        if (!s_last)
            while (*gen == g) {
            }
        __threadfence();
#else
        // arrive: one acq_rel RMW (release: this CTA's writes, ordered by the
        // CTA barrier, before the count; acquire: everything the earlier
        // arrivals released, for the last arriver)
        unsigned prev;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&ctl->bar_count) : "memory");
        s_last = prev == gridDim.x - 1;
        if (!s_last) {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&ctl->bar_gen) : "memory");
            } while (cur == g);
        }
#endif
    }
    __syncthreads();
    if (s_last) {
        if (central) {
            double *scratch = reinterpret_cast<double *>(smem);
            if (threadIdx.x < P.nblocks) s_states[threadIdx.x] = ld_state(P.states + threadIdx.x);
            __syncthreads();
            for (int b = 0; b < P.nblocks; ++b) {
                if (serves<OPK, -1>(s_states[b], P)) {
                    const DBlock &B = P.blocks[b];
                    double q[NQ];
                    for (int i = 0; i < NQ; ++i)
                        q[i] = i < op_nq<OPK>()
                                   ? range_sum<NTHR>(P.partials + (size_t)i * P.nctas, B.cta_begin, B.cta_end, scratch)
                                   : 0.0;
                    if (threadIdx.x == 0) transition(B, s_states[b], nullptr, s_states[b].phase, q);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            int active = 0, verify = 0;
            for (int bb = 0; bb < P.nblocks; ++bb) {
                const int p2 = central ? s_states[bb].phase : ((volatile DState *)P.states)[bb].phase;
                if (p2 != PH_DONE && p2 != PH_IDLE) ++active;
                if (p2 == PH_VERIFY || p2 == PH_INIT || p2 == PH_RESID) ++verify;
            }
            if (OPK == OP_S2) {
                ctl->cycles += 1;
                if (ctl->max_cycles > 0 && ctl->cycles > ctl->max_cycles && active) {
                    for (int bb = 0; bb < P.nblocks; ++bb) {
                        DState &Sb = central ? s_states[bb] : P.states[bb];
                        if (Sb.phase != PH_DONE && Sb.phase != PH_IDLE) {
                            Sb.phase = PH_DONE;
                            Sb.stop = STOP_STALLED;
                        }
                    }
                    ctl->stalled = 1;
                    active = 0;
                    verify = 0;
                }
            }
            if (central)
                for (int bb = 0; bb < P.nblocks; ++bb) P.states[bb] = s_states[bb];
            if (OPK == OP_RESID) ctl->resid_runs += 1;
            *(volatile int *)&ctl->active = active;
            *(volatile int *)&ctl->verify = verify;
            *(volatile int *)P.n_active = active;
            ctl->bar_count = 0u;
#ifdef BS_BAR_FENCES
            __threadfence();
            atomicExch(&ctl->bar_gen, g + 1u);
#else
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&ctl->bar_gen), "r"(g + 1u) : "memory");
#endif
        }
    }
    gen_ref = g + 1u;
    __syncthreads();
    BS_PSTAMP(sw, 3);
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

#ifndef BS_BAR_LOCAL
#define BS_BAR_LOCAL 1
#endif

// Loop conditions of the local-decision barrier, one copy per CTA.
struct LocalCtl {
    int active, verify, cycles, resid_runs, stalled, max_cycles;
};

// Local-decision grid barrier (central mode): every CTA arrives once on a
// monotonic counter and, when all have, reduces the sweep's tile partials
// ITSELF (range_sum in tile order: the same numbers in every CTA) and
// advances its own shared-memory copy of the block states and loop
// conditions.  Nothing is published on the critical path — one L2 round trip
// and a state re-read fewer than the last-arriver barrier.  Partials
// alternate between two buffers by sweep parity: a CTA overwrites a buffer
// only after the NEXT barrier, which every CTA reaches after reading it.
// Only CTA 0 records the residual history (the others' transitions are
// redundant copies).
template <int OPK>
__device__ void grid_sync_local(const KParams &P, unsigned char *smem, DState *s_states, const double *part,
                                unsigned &target, LocalCtl &L, int sw) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned prev;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&P.ctl->bar_count) : "memory");
        unsigned cur = prev + 1u;
        while ((int)(cur - target) < 0)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&P.ctl->bar_count) : "memory");
    }
    __syncthreads();
    BS_PSTAMP(sw, 3);
    double *scratch = reinterpret_cast<double *>(smem);
    for (int b = 0; b < P.nblocks; ++b) {
        if (serves<OPK, -1>(s_states[b], P)) {
            double q[NQ];
#pragma unroll
            for (int i = 0; i < NQ; ++i)
                q[i] = i < op_nq<OPK>() ? range_sum<NTHR>(part + (size_t)i * P.nctas, P.blocks[b].cta_begin,
                                                         P.blocks[b].cta_end, scratch)
                                        : 0.0;
            if (threadIdx.x == 0)
                transition(P.blocks[b], s_states[b], nullptr, s_states[b].phase, q, blockIdx.x == 0);
        }
    }
    if (threadIdx.x == 0) {
        int active = 0, verify = 0;
        for (int bb = 0; bb < P.nblocks; ++bb) {
            const int p2 = s_states[bb].phase;
            if (p2 != PH_DONE && p2 != PH_IDLE) ++active;
            if (p2 == PH_VERIFY || p2 == PH_INIT || p2 == PH_RESID) ++verify;
        }
        if (OPK == OP_S2) {
            L.cycles += 1;
            if (L.max_cycles > 0 && L.cycles > L.max_cycles && active) {
                for (int bb = 0; bb < P.nblocks; ++bb) {
                    DState &Sb = s_states[bb];
                    if (Sb.phase != PH_DONE && Sb.phase != PH_IDLE) {
                        Sb.phase = PH_DONE;
                        Sb.stop = STOP_STALLED;
                    }
                }
                L.stalled = 1;
                active = 0;
                verify = 0;
            }
        }
        if (OPK == OP_RESID) L.resid_runs += 1;
        L.active = active;
        L.verify = verify;
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <bool BOX>
__device__ void cg_persistent_local(const KParams &P, unsigned char *smem, DState *s_states) {
    __shared__ LocalCtl L;
    if (threadIdx.x < P.nblocks) s_states[threadIdx.x] = ld_state(P.states + threadIdx.x);
    if (threadIdx.x == 0) L = LocalCtl{0, 0, 0, 0, 0, *(volatile int *)&P.ctl->max_cycles};
    __syncthreads();
    double *part[2] = {P.partials, P.partials + (size_t)NQ * P.nctas};
    unsigned target = 0;  // bar_count is zeroed by k_reset_control before the launch
    int sw = 0;
    persist_sweep<OP_RESID, BOX>(P, smem, s_states, true, sw, part[sw & 1], true);
    grid_sync_local<OP_RESID>(P, smem, s_states, part[sw & 1], target, L, sw);
    ++sw;
    while (L.active) {
        persist_sweep<OP_S1, BOX>(P, smem, s_states, true, sw, part[sw & 1], true);
        grid_sync_local<OP_S1>(P, smem, s_states, part[sw & 1], target, L, sw);
        ++sw;
        persist_sweep<OP_S2, BOX>(P, smem, s_states, true, sw, part[sw & 1], true);
        grid_sync_local<OP_S2>(P, smem, s_states, part[sw & 1], target, L, sw);
        ++sw;
        if (L.verify) {
            persist_sweep<OP_RESID, BOX>(P, smem, s_states, true, sw, part[sw & 1], true);
            grid_sync_local<OP_RESID>(P, smem, s_states, part[sw & 1], target, L, sw);
            ++sw;
        }
    }
    if (blockIdx.x == 0) {
        if (threadIdx.x < P.nblocks) P.states[threadIdx.x] = s_states[threadIdx.x];
        if (threadIdx.x == 0) {
            Control *ctl = P.ctl;
            ctl->cycles = L.cycles;
            ctl->stalled = L.stalled;
            ctl->resid_runs = L.resid_runs;
            ctl->active = L.active;
            ctl->verify = L.verify;
            *P.n_active = L.active;
        }
    }
}

template <bool BOX>
__global__ void __launch_bounds__(NTHR, 2) k_cg_persistent(const KParams P) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ DState s_states[CENTRAL_MAX];
    __shared__ unsigned s_gen0;
    const bool central = P.nblocks <= CENTRAL_MAX;
    if (BS_BAR_LOCAL && central) {
        cg_persistent_local<BOX>(P, smem, s_states);
        return;
    }
    if (threadIdx.x == 0) s_gen0 = *(volatile unsigned *)&P.ctl->bar_gen;  // no barrier completes before all read it
    __syncthreads();
    unsigned gen = s_gen0;
    int sw = 0;  // sweep counter (tracing only)
    persist_sweep<OP_RESID, BOX>(P, smem, s_states, central, sw, P.partials);  // INIT (and any armed residual sweep)
    grid_sync<OP_RESID>(P, smem, s_states, central, gen, sw++);
    while (*(volatile int *)&P.ctl->active) {
        persist_sweep<OP_S1, BOX>(P, smem, s_states, central, sw, P.partials);
        grid_sync<OP_S1>(P, smem, s_states, central, gen, sw++);
        persist_sweep<OP_S2, BOX>(P, smem, s_states, central, sw, P.partials);
        grid_sync<OP_S2>(P, smem, s_states, central, gen, sw++);
        if (*(volatile int *)&P.ctl->verify) {
            persist_sweep<OP_RESID, BOX>(P, smem, s_states, central, sw, P.partials);
            grid_sync<OP_RESID>(P, smem, s_states, central, gen, sw++);
        }
    }
}

// ---- streaming persistent CG: many tiles (and up to MAXB_STREAM blocks) per
// launch.  When the tiles outnumber the co-resident CTAs (config 3: eight
// 512^2 x 64 slabs = 8192 tiles, or one slab = 1024 tiles per GPU at 8 GPUs),
// the whole inner solve is still ONE cooperative launch of exactly LANES = 256
// CTAs.  CTA c owns reduction lane c of every block: the tiles
// cta_begin + c + 256 k (k = 0, 1, ...), streamed back to back through one
// ring (sweep_tile's shared-ring mode: no gap between tiles), and it sums
// their tile partials in k order itself — exactly range_sum's lane c.  So a
// sweep publishes one value per (block, quantity, lane), every CTA reduces a
// block from 256 lane sums with range_sum's tree after a software grid
// barrier (local decision, as cg_persistent_local), and the numbers are bit
// for bit the graph path's.  The static assignment gives every CTA the same
// work (1024 tiles -> 4 per CTA) and keeps the 256 CTAs marching through the
// same band of each plane together.
constexpr int MAXB_STREAM = 16;
constexpr int LANES = 256;          // = range_sum's virtual lanes = the grid
constexpr int MAXK_STREAM = 64;     // tiles per lane and block (s_tp capacity)

// The partials of one tile (consumer warps only; the producer may already be
// streaming the next tile): cta_sum<NTHR>'s order — warps 0..NCW-1, then the
// producer warp's +0.0 — exactly as tile_epilogue; thread 0 stores them at out.
__device__ __forceinline__ void tile_partial(double (&acc)[NQ], double *red, double *out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[q * NCW + warp] = v;
    }
    consumer_sync();
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double sum = red[q * NCW];
            for (int w = 1; w < NCW; ++w) sum = add(sum, red[q * NCW + w]);
            out[q] = add(sum, 0.0);
        }
    }
    consumer_sync();  // red is reused by the next tile
}

// Lane sums of one sweep: lanes[(q * nblocks + b) * LANES + c].
template <int OPK, bool BOX>
__device__ __noinline__ void stream_sweep(const KParams &P, unsigned char *smem, const DState *s_states, double *lanes,
                                          double *s_red, double *s_tp, int sw) {
    const int tid = threadIdx.x;
    constexpr int NS = op_stages(OPK);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * op_stage_bytes(OPK));
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&full[NS + s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    BS_SSTAMP(sw, 0);
    const int c = blockIdx.x;
    int gstage = 0;  // ring-global stage of the next tile
    // reversed ops (S2) walk the blocks and their tiles backwards: the
    // previous sweep's last planes are still in L2 (as k_sweep)
    for (int bi = 0; bi < P.nblocks; ++bi) {
        const int b = op_rev(OPK) ? P.nblocks - 1 - bi : bi;
        const DState &S = s_states[b];
        if (!serves<OPK, -1>(S, P)) continue;
        const DBlock &B = P.blocks[b];
        const int span = B.cta_end - B.cta_begin;
        const int nk = span > c ? (span - c + LANES - 1) / LANES : 0;
        if (nk > 0) {
            const SweepCtx C = make_ctx<OPK>(P, b, B, S);
            for (int kk = 0; kk < nk; ++kk) {
                const int k = op_rev(OPK) ? nk - 1 - kk : kk;
                double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
                gstage += sweep_tile<OPK, BOX>(C, c + LANES * k, smem, acc, gstage);
                if (tid < NT) tile_partial(acc, s_red, s_tp + k * NQ);
            }
        }
        if (tid == 0) {  // lane c of block b: its tile partials in k order (range_sum)
#pragma unroll
            for (int q = 0; q < op_nq<OPK>(); ++q) {
                double sum = 0.0;
                for (int k = 0; k < nk; ++k) sum = add(sum, s_tp[k * NQ + q]);
                lanes[((size_t)q * P.nblocks + b) * LANES + c] = sum;
            }
        }
    }
    BS_SSTAMP(sw, 1);
    __syncthreads();
    if (tid == 0)  // the next sweep re-initialises this memory for its own ring
        for (int s = 0; s < 2 * NS; ++s)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Local-decision barrier of the streaming kernel: arrive, wait for all, then
// warp w folds (block, quantity) pairs w, w + 9, ...: the 256 lane sums of a
// pair with range_sum's tree (8 loads in flight per lane), and one thread per
// served block advances its shared-memory state.
template <int OPK>
__device__ void grid_sync_stream(const KParams &P, DState *s_states, const double *lanes, unsigned &target, LocalCtl &L,
                                 int *s_list, double *s_q, int sw) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    target += gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        unsigned prev;
        BS_SSTAMP(sw, 2);
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&P.ctl->bar_count) : "memory");
        unsigned cur = prev + 1u;
        while ((int)(cur - target) < 0)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&P.ctl->bar_count) : "memory");
        BS_SSTAMP(sw, 3);
        int n = 0;
        for (int b = 0; b < P.nblocks; ++b)
            if (serves<OPK, -1>(s_states[b], P)) s_list[n++] = b;
        s_list[MAXB_STREAM] = n;
    }
    __syncthreads();
    BS_SSTAMP(sw, 4);
    constexpr int NQK = op_nq<OPK>();
    const int nserved = s_list[MAXB_STREAM];
    for (int pp = warp; pp < nserved * NQK; pp += NTHR / 32) {
        const double *src = lanes + ((size_t)(pp % NQK) * P.nblocks + s_list[pp / NQK]) * LANES;
        double v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = __ldcg(src + lane + 32 * m);
#pragma unroll
        for (int m = 0; m < 4; ++m) v[m] = add(v[m], v[m + 4]);  // range_sum's tree
        v[0] = add(v[0], v[2]);
        v[1] = add(v[1], v[3]);
        double t = add(v[0], v[1]);
#pragma unroll
        for (int w = 16; w > 0; w >>= 1) t = add(t, __shfl_down_sync(0xffffffffu, t, w));
        if (lane == 0) s_q[pp] = t;
    }
    __syncthreads();
    BS_SSTAMP(sw, 5);
    if (tid < nserved) {  // one thread per served block (CTA 0 records the histories)
        const int b = s_list[tid];
        double q[NQ] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < NQK; ++i) q[i] = s_q[tid * NQK + i];
        transition(P.blocks[b], s_states[b], nullptr, s_states[b].phase, q, blockIdx.x == 0);
    }
    __syncthreads();
    if (tid == 0) {
        int active = 0, verify = 0;
        for (int bb = 0; bb < P.nblocks; ++bb) {
            const int p2 = s_states[bb].phase;
            if (p2 != PH_DONE && p2 != PH_IDLE) ++active;
            if (p2 == PH_VERIFY || p2 == PH_INIT || p2 == PH_RESID) ++verify;
        }
        if (OPK == OP_S2) {
            L.cycles += 1;
            if (L.max_cycles > 0 && L.cycles > L.max_cycles && active) {
                for (int bb = 0; bb < P.nblocks; ++bb) {
                    DState &Sb = s_states[bb];
                    if (Sb.phase != PH_DONE && Sb.phase != PH_IDLE) {
                        Sb.phase = PH_DONE;
                        Sb.stop = STOP_STALLED;
                    }
                }
                L.stalled = 1;
                active = 0;
                verify = 0;
            }
        }
        if (OPK == OP_RESID) L.resid_runs += 1;
        L.active = active;
        L.verify = verify;
        BS_SSTAMP(sw, 6);
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

#ifndef BS_STREAM_MINBLOCKS
#define BS_STREAM_MINBLOCKS 2
#endif

template <bool BOX>
__global__ void __launch_bounds__(NTHR, BS_STREAM_MINBLOCKS) k_cg_stream(const KParams P) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ DState s_states[MAXB_STREAM];
    __shared__ LocalCtl L;
    __shared__ double s_red[NQ * NCW];
    __shared__ double s_q[MAXB_STREAM * NQ];
    __shared__ double s_tp[MAXK_STREAM * NQ];
    __shared__ int s_list[MAXB_STREAM + 1];
    if (threadIdx.x < P.nblocks) s_states[threadIdx.x] = ld_state(P.states + threadIdx.x);
    if (threadIdx.x == 0) L = LocalCtl{0, 0, 0, 0, 0, *(volatile int *)&P.ctl->max_cycles};
    __syncthreads();
    // lane sums alternate between two buffers by sweep parity (a buffer is
    // overwritten only after the next barrier, which every CTA reaches after
    // reading it)
    double *lanes[2] = {P.partials, P.partials + (size_t)NQ * P.part_stride};
    unsigned target = 0;  // bar_count is zeroed by k_reset_control before the launch
    int sw = 0;
    stream_sweep<OP_RESID, BOX>(P, smem, s_states, lanes[sw & 1], s_red, s_tp, sw);
    grid_sync_stream<OP_RESID>(P, s_states, lanes[sw & 1], target, L, s_list, s_q, sw);
    ++sw;
    while (L.active) {
        stream_sweep<OP_S1, BOX>(P, smem, s_states, lanes[sw & 1], s_red, s_tp, sw);
        grid_sync_stream<OP_S1>(P, s_states, lanes[sw & 1], target, L, s_list, s_q, sw);
        ++sw;
        stream_sweep<OP_S2, BOX>(P, smem, s_states, lanes[sw & 1], s_red, s_tp, sw);
        grid_sync_stream<OP_S2>(P, s_states, lanes[sw & 1], target, L, s_list, s_q, sw);
        ++sw;
        if (L.verify) {
            stream_sweep<OP_RESID, BOX>(P, smem, s_states, lanes[sw & 1], s_red, s_tp, sw);
            grid_sync_stream<OP_RESID>(P, s_states, lanes[sw & 1], target, L, s_list, s_q, sw);
            ++sw;
        }
    }
    if (blockIdx.x == 0) {
        if (threadIdx.x < P.nblocks) P.states[threadIdx.x] = s_states[threadIdx.x];
        if (threadIdx.x == 0) {
            Control *ctl = P.ctl;
            ctl->cycles = L.cycles;
            ctl->stalled = L.stalled;
            ctl->resid_runs = L.resid_runs;
            ctl->active = L.active;
            ctl->verify = L.verify;
            *P.n_active = L.active;
        }
    }
}

// Pointwise GMRES passes over a block's region, tile by tile (same CTA table
// and deterministic reduction order as the sweeps).
template <int PKK, bool BOX>
__global__ void __launch_bounds__(NPT) k_point(const KParams P) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // Chunk order: consecutive passes of an Arnoldi step alternate direction
    // (MGS pass i reversed when i is odd, FINAL opposite to the last MGS
    // pass, NORM opposite to the FINAL before it), so each pass starts on
    // the chunks the previous one touched last (still in L2).  Partials are
    // indexed by chunk, so the reduction order (and every result) is the
    // same either way.
    bool rev = false;
    if (BS_REV_PASSES) {
        // GSPMV (a z-ascending sweep) precedes MGS pass 1 and FINAL of step 0
        if (PKK == PK_MGS) rev = P.launch_i & 1;
        else if (PKK == PK_FINAL) rev = !(P.launch_j & 1);
        else if (PKK == PK_NORM) rev = P.launch_j > 0 && !(P.launch_j & 1);
    }
    const int pc = P.pcta_base + (rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x);
    const int b = P.pcta_block[pc];
    const DBlock &B = P.blocks[b];
    const DState S = P.states[b];
    const int ph = S.phase;
    const bool served = serves<-1, PKK>(S, P);
    double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
    if (served) {
        // flat, contiguous chunk of the block's pitched padded box: each thread
        // takes element pairs (16-byte loads) at a fixed stride, so the CTA
        // streams PCHUNK consecutive doubles.  Cells outside the region (and
        // the row padding) hold exact zeros in r, W and V, so MGS / FINAL /
        // NORM need no mask; FORM and OWNRES test the region explicitly.
        const GState &G = P.gstates[b];
        const int tid = threadIdx.x;
        const long long n = (long long)B.pitch * B.pdim[1] * B.pdim[2];
        const long long base = (long long)(pc - B.pcta_begin) * PCHUNK;
        const int j = S.gj, i = S.gi;
        const long long vs = B.vstride;
        double *__restrict__ W = B.W;
        const double *__restrict__ V = B.V;
        // element pairs of this CTA: e = base + 2 (it * NPT + tid); the chunk
        // is processed in batches of PB pairs per thread, every load of a
        // batch issued before any use (memory-level parallelism), with no
        // bounds test on full chunks
        constexpr int PITER = PCHUNK / (2 * NPT), PB = 4;
        const long long pair0 = base / 2 + tid;  // in double2 units
        const long long npairs = n / 2;          // n is even (pitch % 4 == 0)
        const bool full_chunk = base + PCHUNK <= n;
        if (PKK == PK_NORM) {  // v_j = src / nrm (inner_solvers.py:164, 237)
            const double2 *src = reinterpret_cast<const double2 *>(j == 0 ? B.r : W);
            double2 *vj = reinterpret_cast<double2 *>(B.V + j * vs);
            const double nrm = S.gnrm;
            for (int it0 = 0; it0 < PITER; it0 += PB) {
                double2 v[PB];
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    const long long e2 = pair0 + (long long)(it0 + u) * NPT;
                    if (full_chunk || e2 < npairs) v[u] = __ldcs(src + e2);
                }
#pragma unroll
                for (int u = 0; u < PB; ++u) {
                    const long long e2 = pair0 + (long long)(it0 + u) * NPT;
                    if (!(full_chunk || e2 < npairs)) continue;
                    const double2 q = make_double2(__ddiv_rn(v[u].x, nrm), __ddiv_rn(v[u].y, nrm));
                    if (BS_MGS_HINT) __stcg(vj + e2, q);
                    else __stcs(vj + e2, q);
                }
            }
        } else if (PKK == PK_MGS || PKK == PK_FINAL) {
            // MGS:   w -= h_{i-1,j} v_{i-1} ; h_ij = v_i . w   (inner_solvers.py:189-193)
            // FINAL: w -= h_jj v_j ; ||w||^2                    (193-195)
            const double h = PKK == PK_MGS ? G.H[(i - 1) * MAXM + j] : G.H[j * MAXM + j];
            const double2 *va = reinterpret_cast<const double2 *>(V + (PKK == PK_MGS ? i - 1 : j) * vs);
            const double2 *vb = reinterpret_cast<const double2 *>(V + i * vs);
            double2 *w2 = reinterpret_cast<double2 *>(W);
            // evict_last tail only when the launch covers one block: in an
            // all-block launch the time-last CTAs may belong to finished blocks
            const bool one_block = P.pcta_block[P.pcta_base] == P.pcta_block[P.pcta_base + (int)gridDim.x - 1];
            const bool pol2 = BS_MGS_HINT == 2 && one_block;
            uint64_t pol_keep = 0, pol_drop = 0;
            if (pol2) {
                // the FINAL pass of a cycle's last step is w's last use in the
                // cycle (FORM reads V and x, and streams V evict-first): demote
                // its lines instead of pinning them in L2 for the FORM, the
                // residual sweep and other blocks' passes
                const bool last_use = PKK == PK_FINAL && j == S.gm - 1;
                pol_keep = l2_policy(!last_use && (int)blockIdx.x >= (int)gridDim.x - BS_MGS_KEEP);
                pol_drop = l2_policy(false);
            }
            // one loop per cache mode (a run-time mode test inside the batch
            // loop costs the batching its memory-level parallelism)
            auto pass = [&](auto mode_c) {
                constexpr int MODE = decltype(mode_c)::value;
                for (int it0 = 0; it0 < PITER; it0 += PB) {
                    double2 w[PB], a[PB], c[PB];
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const long long e2 = pair0 + (long long)(it0 + u) * NPT;
                        if (full_chunk || e2 < npairs) {
                            if (MODE == 2) {
                                w[u] = ld_pol(w2 + e2, pol_keep);
                                a[u] = ld_pol(va + e2, pol_drop);
                                if (PKK == PK_MGS) c[u] = ld_pol(vb + e2, pol_keep);
                            } else if (MODE == 1) {
                                w[u] = __ldcg(w2 + e2);
                                a[u] = __ldcs(va + e2);
                                if (PKK == PK_MGS) c[u] = __ldcg(vb + e2);
                            } else {
                                w[u] = __ldcs(w2 + e2);
                                a[u] = __ldg(va + e2);
                                if (PKK == PK_MGS) c[u] = __ldg(vb + e2);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const long long e2 = pair0 + (long long)(it0 + u) * NPT;
                        if (!(full_chunk || e2 < npairs)) continue;
                        const double w0 = sub(w[u].x, mul(h, a[u].x)), w1 = sub(w[u].y, mul(h, a[u].y));
                        if (MODE == 2) st_pol(w2 + e2, make_double2(w0, w1), pol_keep);
                        else if (MODE == 1) __stcg(w2 + e2, make_double2(w0, w1));
                        else __stcs(w2 + e2, make_double2(w0, w1));
                        if (PKK == PK_MGS) {
                            acc[0] = add(acc[0], mul(c[u].x, w0));
                            acc[0] = add(acc[0], mul(c[u].y, w1));
                        } else {
                            acc[0] = add(acc[0], mul(w0, w0));
                            acc[0] = add(acc[0], mul(w1, w1));
                        }
                    }
                }
            };
            if (pol2) pass(IntC<2>{});
            else pass(IntC<(BS_MGS_HINT ? 1 : 0)>{});
        } else if (PKK == PK_FORM) {
            // x = x + V[:j+1]^T y (inner_solvers.py:173-175), element pairs:
            // 16-byte loads of x and of 8 basis vectors at a time, all issued
            // before their adds (the same left-to-right sum per element).  The
            // coordinates of a thread's pair advance incrementally (no 64-bit
            // division per element); pairs never straddle a row (pitch % 4 == 0).
            const int pitch = B.pitch, pdx = B.pdim[0], pdy = B.pdim[1];
            const double2 *V2 = reinterpret_cast<const double2 *>(V);
            double2 *x2 = reinterpret_cast<double2 *>(B.x);
            const long long vs2 = vs / 2;
            long long e = base + 2 * tid;
            int lx = (int)(e % pitch);
            int row = (int)(e / pitch);
            const double y0 = G.y[0];
            for (int it = 0; it < PCHUNK / (2 * NPT); ++it, e += 2 * NPT) {
                if (it) {
                    lx += 2 * NPT;
                    while (lx >= pitch) {
                        lx -= pitch;
                        ++row;
                    }
                }
                if (e >= n) break;
                bool in0 = lx < pdx, in1 = lx + 1 < pdx;
                if (!BOX && (in0 || in1)) {
                    const int gi = B.plo[0] + lx, gj = B.plo[1] + row % pdy, gk = B.plo[2] + row / pdy;
                    in0 = in0 && in_region(B, gi, gj, gk);
                    in1 = in1 && in_region(B, gi + 1, gj, gk);
                }
                if (!in0 && !in1) continue;
                const long long p2 = e / 2;
                const double2 v0 = __ldcs(V2 + p2);
                double a0 = mul(v0.x, y0), a1 = mul(v0.y, y0);
                int k = 1;
                for (; k + 8 <= j + 1; k += 8) {
                    double2 v8[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v8[u] = __ldcs(V2 + (k + u) * vs2 + p2);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double yk = G.y[k + u];
                        a0 = add(a0, mul(v8[u].x, yk));
                        a1 = add(a1, mul(v8[u].y, yk));
                    }
                }
                for (; k <= j; ++k) {
                    const double2 v = __ldcs(V2 + k * vs2 + p2);
                    a0 = add(a0, mul(v.x, G.y[k]));
                    a1 = add(a1, mul(v.y, G.y[k]));
                }
                double2 xv = x2[p2];
                if (in0) xv.x = add(xv.x, a0);
                if (in1) xv.y = add(xv.y, a1);
                x2[p2] = xv;
            }
        } else {
            const int pitch = B.pitch, pdx = B.pdim[0], pdy = B.pdim[1];
            for (int it = 0; it < PCHUNK / NPT; ++it) {
                const long long e = base + (long long)it * NPT + tid;
                if (e >= n) break;
                const int lx = (int)(e % pitch);
                if (lx >= pdx) continue;
                const long long t2 = e / pitch;
                const int gi = B.plo[0] + lx, gj = B.plo[1] + (int)(t2 % pdy), gk = B.plo[2] + (int)(t2 / pdy);
                {  // PK_OWNRES
                    // Local residual with owner-canonical values (multisplit.py:372-396):
                    // on owned rows every stencil neighbour is a region point (o >= 1),
                    // so this is b - A x_gathered with x_gathered = each owner's
                    // post-solve value (the snapshot in its r).  acc[2] = acc[3].
                    if (!in_owned(B, gi, gj, gk)) continue;
                    const int ni[6] = {gi, gi, gi - 1, gi + 1, gi, gi};
                    const int nj[6] = {gj, gj - 1, gj, gj, gj + 1, gj};
                    const int nk[6] = {gk - 1, gk, gk, gk, gk, gk + 1};
                    double v[6];
                    bool pg[6];
#pragma unroll
                    for (int d = 0; d < 6; ++d) {
                        pg[d] = in_grid(B, ni[d], nj[d], nk[d]);
                        v[d] = 0.0;
                        if (!pg[d]) continue;
                        if (in_owned(B, ni[d], nj[d], nk[d])) {
                            v[d] = B.r[sidx(B, ni[d], nj[d], nk[d])];
                        } else {
                            for (int u = 0; u < B.nnbr; ++u) {
                                const DBlock &U = P.blocks[B.nbr[u]];
                                if (in_owned(U, ni[d], nj[d], nk[d])) {
                                    v[d] = U.r[sidx(U, ni[d], nj[d], nk[d])];
                                    break;
                                }
                            }
                        }
                    }
                    const double ag = stencil7(v[0], v[1], v[2], B.r[e], v[3], v[4], v[5], pg[0], pg[1], pg[2]);
                    const double rg = sub(B.b[e], ag);
                    const double r2 = mul(rg, rg);
                    acc[2] = add(acc[2], r2);
                    acc[3] = add(acc[3], r2);
                }
            }
        }
    }
    finish<NPT, -1, true>(P, b, ph, served, acc, PKK == PK_OWNRES ? NQ : 1, smem, pc);
}

// ---- overlapping merge (multisplit.py:341-369), overlap > 0.  Inputs are the
// post-solve snapshots (each block's r := x over its region); outputs are
// written into x (shared points; coupled halo cells inside the padded box) and
// the face planes (coupled cells just outside it).

// r := x on region cells, 0 elsewhere (non-region cells of x hold halo values;
// r, W and V must stay zero off the region for the unmasked pointwise passes)
__global__ void k_snapshot(const DBlock *__restrict__ blocks) {
    const DBlock &B = blocks[blockIdx.y];
    if (B.remote) return;
    const long long n = (long long)B.pitch * B.pdim[1] * B.pdim[2];
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int lx = (int)(c % B.pitch);
        const long long t = c / B.pitch;
        const bool in = lx < B.pdim[0] && in_region(B, B.plo[0] + lx, B.plo[1] + (int)(t % B.pdim[1]),
                                                    B.plo[2] + (int)(t / B.pdim[1]));
        B.r[c] = in ? B.x[c] : 0.0;
    }
}

// (own? + sum over covering neighbours in ascending id order) / cover count
__device__ __forceinline__ double merged_value(const DBlock *blocks, const DBlock &T, bool own, double own_val,
                                               int i, int j, int k) {
    double acc = own ? own_val : 0.0;
    int m = own ? 1 : 0;
    for (int u = 0; u < T.nnbr; ++u) {
        const DBlock &U = blocks[T.nbr[u]];
        if (in_region(U, i, j, k)) {
            acc = add(acc, U.r[sidx(U, i, j, k)]);
            ++m;
        }
    }
    return m ? __ddiv_rn(acc, (double)m) : 0.0;
}

__global__ void k_merge(const DBlock *__restrict__ blocks) {
    const DBlock &T = blocks[blockIdx.y];
    if (T.remote) return;
    const long long n = (long long)T.pitch * T.pdim[1] * T.pdim[2];
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int lx = (int)(c % T.pitch);
        if (lx >= T.pdim[0]) continue;
        const long long t = c / T.pitch;
        const int i = T.plo[0] + lx, j = T.plo[1] + (int)(t % T.pdim[1]), k = T.plo[2] + (int)(t / T.pdim[1]);
        if (in_owned(T, i, j, k) || !in_grid(T, i, j, k)) continue;
        if (in_region(T, i, j, k)) {  // shared point: own value first, then neighbours
            T.x[c] = merged_value(blocks, T, true, T.r[c], i, j, k);
        } else if (in_region(T, i - 1, j, k) || in_region(T, i + 1, j, k) || in_region(T, i, j - 1, k) ||
                   in_region(T, i, j + 1, k) || in_region(T, i, j, k - 1) || in_region(T, i, j, k + 1)) {
            T.x[c] = merged_value(blocks, T, false, 0.0, i, j, k);  // coupled halo column
        }
    }
}

__global__ void k_merge_faces(const DBlock *__restrict__ blocks) {
    const DBlock &T = blocks[blockIdx.y];
    const int dir = blockIdx.z;
    if (T.remote || !T.ghost[dir]) return;
    int nu, nv;
    if (dir == 0 || dir == 5) {
        nu = T.pdim[0];
        nv = T.pdim[1];
    } else if (dir == 1 || dir == 4) {
        nu = T.pdim[0];
        nv = T.pdim[2];
    } else {
        nu = T.pdim[1];
        nv = T.pdim[2];
    }
    const long long n = (long long)nu * nv;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        const int u = (int)(c % nu), v = (int)(c / nu);
        int i, j, k, di = 0, dj = 0, dk = 0;
        switch (dir) {
            case 0: i = T.plo[0] + u; j = T.plo[1] + v; k = T.plo[2] - 1; dk = 1; break;
            case 5: i = T.plo[0] + u; j = T.plo[1] + v; k = T.plo[2] + T.pdim[2]; dk = -1; break;
            case 1: i = T.plo[0] + u; j = T.plo[1] - 1; k = T.plo[2] + v; dj = 1; break;
            case 4: i = T.plo[0] + u; j = T.plo[1] + T.pdim[1]; k = T.plo[2] + v; dj = -1; break;
            case 2: i = T.plo[0] - 1; j = T.plo[1] + u; k = T.plo[2] + v; di = 1; break;
            default: i = T.plo[0] + T.pdim[0]; j = T.plo[1] + u; k = T.plo[2] + v; di = -1; break;
        }
        if (in_region(T, i + di, j + dj, k + dk)) T.ghost[dir][c] = merged_value(blocks, T, false, 0.0, i, j, k);
    }
}

// y = A_ii x on one block (standalone a1); x, y in the block's pitched layout.
template <bool BOX>
__global__ void __launch_bounds__(NTHR, BS_MINBLOCKS) k_apply(const DBlock *__restrict__ blocks, int b,
                                                   const __grid_constant__ CUtensorMap xmap, double *y) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const DBlock &B = blocks[b];
    SweepCtx C;
    C.B = &B;
    C.pend = C.first = C.want_global = false;
    C.alpha_pend = C.alpha = C.beta = 0.0;
    C.map_a = &xmap;
    C.map_b = nullptr;
    C.map_c = nullptr;
    C.pout = nullptr;
    C.yout = y;
    double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
    sweep_tile<OP_APPLY, BOX>(C, blockIdx.x, smem, acc);
}

// Arm solves / residual sweeps.
__global__ void k_arm(const DBlock *blocks, DState *states, const int *active, int nblocks, int phase, int max_its,
                      double tol, int basis, int kind, int gm) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    if ((active && !active[b]) || blocks[b].remote) return;  // phantoms stay idle
    DState &S = states[b];
    S.phase = phase;
    if (phase == PH_INIT) {
        S.last_it = S.it;
        S.last_stop = S.stop;
        S.stop = BS_STOP_NONE;
        S.it = 0;
        S.first = 1;
        S.max_its = max_its;
        S.tol = tol;
        S.basis = basis;
        S.kind = kind;
        S.gm = gm;
    }
}

__global__ void k_reset_control(Control *ctl, int max_cycles) {
    ctl->cycles = 0;
    ctl->max_cycles = max_cycles;
    ctl->stalled = 0;
    ctl->resid_runs = 0;
    ctl->bar_count = 0u;
    ctl->active = 0;
    ctl->verify = 0;
}

// Deferred x += alpha p over every region point of blocks with a pending update.
__global__ void k_flush(const DBlock *__restrict__ blocks, const DState *states) {
    const int b = blockIdx.y;
    const DBlock &B = blocks[b];
    const DState &S = states[b];
    if (!S.pend && !S.xin) return;
    const long long n = (long long)B.pdim[0] * B.pdim[1] * B.pdim[2];
    const double a = S.alpha_pend;
    const bool jac = S.xin != 0;  // Jacobi iterate left in p[0]: copy it home
    const double *p = B.p[jac ? 0 : S.pcur];
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int i = B.plo[0] + (int)(c % B.pdim[0]);
        const long long t = c / B.pdim[0];
        const int j = B.plo[1] + (int)(t % B.pdim[1]);
        const int k = B.plo[2] + (int)(t / B.pdim[1]);
        if (B.overlap == 0 || in_region(B, i, j, k)) {
            const long long s = sidx(B, i, j, k);
            B.x[s] = jac ? p[s] : add(B.x[s], mul(a, p[s]));
        }
    }
}

__global__ void k_clear_pend(DState *states, int nblocks) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nblocks) {
        states[b].pend = 0;
        states[b].xin = 0;
    }
}

// Sync halo pack: ghost[dir] of dst <- current (flushed-on-the-fly) x of src.
__global__ void k_halo_pack(const DBlock *__restrict__ blocks, const DState *states, const int *plan) {
    const int e = blockIdx.y;
    const int dst = plan[3 * e], dir = plan[3 * e + 1], src = plan[3 * e + 2];
    const DBlock &D = blocks[dst];
    const DBlock &S = blocks[src];
    const DState &SS = states[src];
    int nu, nv;
    if (dir == 0 || dir == 5) {
        nu = D.pdim[0];
        nv = D.pdim[1];
    } else if (dir == 1 || dir == 4) {
        nu = D.pdim[0];
        nv = D.pdim[2];
    } else {
        nu = D.pdim[1];
        nv = D.pdim[2];
    }
    const unsigned n = (unsigned)nu * (unsigned)nv;  // a plane of a block: < 2^31 cells
    const double a = SS.alpha_pend;
    const bool pend = SS.pend != 0;
    const double *p = S.p[SS.pcur];
    const double *xsrc = SS.xin ? S.p[0] : S.x;
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int v = (int)(c / (unsigned)nu), u = (int)(c - (unsigned)v * (unsigned)nu);
        int i, j, k;
        switch (dir) {
            case 0: i = D.plo[0] + u; j = D.plo[1] + v; k = D.plo[2] - 1; break;
            case 5: i = D.plo[0] + u; j = D.plo[1] + v; k = D.plo[2] + D.pdim[2]; break;
            case 1: i = D.plo[0] + u; j = D.plo[1] - 1; k = D.plo[2] + v; break;
            case 4: i = D.plo[0] + u; j = D.plo[1] + D.pdim[1]; k = D.plo[2] + v; break;
            case 2: i = D.plo[0] - 1; j = D.plo[1] + u; k = D.plo[2] + v; break;
            default: i = D.plo[0] + D.pdim[0]; j = D.plo[1] + u; k = D.plo[2] + v; break;
        }
        const long long s = sidx(S, i, j, k);
        const double xv = xsrc[s];
        D.ghost[dir][c] = pend ? add(xv, mul(a, p[s])) : xv;
    }
}

// ------------------------------------------------------------------ async halo mailboxes
// One-sided puts for asynchronous block Jacobi (comm.py:367-418 semantics on
// real hardware): a sender stores its boundary plane (x + pending alpha p)
// into slot seq % R of the receiver's ring and then publishes seq with a
// system-scope release; the receiver picks the freshest published slot newer
// than the one it applied (stale ones are never applied), copies it to its
// halo plane and re-validates the slot's seq (seqlock) before accepting it.

__device__ __forceinline__ void plane_cell(const DBlock &B, int dir, long long c, int nu, int &i, int &j, int &k) {
    const int u = (int)(c % nu), v = (int)(c / nu);
    switch (dir) {  // the block's own boundary plane facing `dir`
        case 0: i = B.plo[0] + u; j = B.plo[1] + v; k = B.plo[2]; break;
        case 5: i = B.plo[0] + u; j = B.plo[1] + v; k = B.plo[2] + B.pdim[2] - 1; break;
        case 1: i = B.plo[0] + u; j = B.plo[1]; k = B.plo[2] + v; break;
        case 4: i = B.plo[0] + u; j = B.plo[1] + B.pdim[1] - 1; k = B.plo[2] + v; break;
        case 2: i = B.plo[0]; j = B.plo[1] + u; k = B.plo[2] + v; break;
        default: i = B.plo[0] + B.pdim[0] - 1; j = B.plo[1] + u; k = B.plo[2] + v; break;
    }
}

__host__ __device__ __forceinline__ int plane_nu(const int *pdim, int dir) {
    return (dir == 2 || dir == 3) ? pdim[1] : pdim[0];
}

__host__ __device__ __forceinline__ long long plane_len(const int *pdim, int dir) {
    if (dir == 0 || dir == 5) return (long long)pdim[0] * pdim[1];
    if (dir == 1 || dir == 4) return (long long)pdim[0] * pdim[2];
    return (long long)pdim[1] * pdim[2];
}

// Seqlock writer side: retire the slot before its payload is overwritten, so
// a reader that picked the slot's previous seq fails its re-validation.
__global__ void k_async_retire(unsigned long long *seqs, int slot) {
    *((volatile unsigned long long *)&seqs[slot]) = 0ull;
    __threadfence_system();
}

// Payload (x + pending alpha p of the boundary plane) into ring slot `sl`;
// the last CTA stamps the delivery iteration (injected-delay model, may be
// null) and then publishes seq+1 with a system-scope release.
__global__ void k_async_post(const DBlock *__restrict__ blocks, const DState *states, int b, int dir, double *ring,
                             unsigned long long *seqs, int sl, unsigned long long seq, long long *deliver,
                             long long deliver_at, unsigned *counter) {
    const DBlock &B = blocks[b];
    const DState &S = states[b];
    const int nu = plane_nu(B.pdim, dir);
    const long long n = plane_len(B.pdim, dir);
    double *slot = ring + (long long)sl * n;
    const double a = S.alpha_pend;
    const bool pend = S.pend != 0;
    const double *p = B.p[S.pcur];
    const double *xsrc = S.xin ? B.p[0] : B.x;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        plane_cell(B, dir, c, nu, i, j, k);
        const long long sx = sidx(B, i, j, k);
        const double xv = xsrc[sx];
        slot[c] = pend ? add(xv, mul(a, p[sx])) : xv;
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        if (deliver) *((volatile long long *)&deliver[sl]) = deliver_at;
        __threadfence_system();  // payload visible system-wide before the seq (release)
        *((volatile unsigned long long *)&seqs[sl]) = seq + 1;  // 0 = empty slot
        *counter = 0u;
    }
}

// pick[0] = chosen seq+1 (0: nothing newer), pick[1] = slot
// Freshest published slot; with a delivery table only slots whose delivery
// iteration the receiver has reached (deliver <= receiver_k) qualify.
__global__ void k_async_pick(const unsigned long long *seqs, const long long *deliver, int R, long long receiver_k,
                             const unsigned long long *applied, unsigned long long *pick) {
    unsigned long long best = 0, slot = 0;
    for (int s = 0; s < R; ++s) {
        const unsigned long long v = ((const volatile unsigned long long *)seqs)[s];
        if (v <= best) continue;
        if (deliver) {
            __threadfence_system();  // the stamp was written before the seq
            if (((const volatile long long *)deliver)[s] > receiver_k) continue;
        }
        best = v;
        slot = s;
    }
    __threadfence_system();  // acquire: payload reads below follow the seq read
    pick[0] = best > *applied ? best : 0ull;
    pick[1] = slot;
}

__global__ void k_async_copy(const DBlock *__restrict__ blocks, int b, int gdir, const double *ring, long long n,
                             const unsigned long long *pick, double *stage) {
    if (pick[0] == 0) return;
    const double *src = ring + (long long)pick[1] * n;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
        stage[c] = ((const volatile double *)src)[c];
}

// seqlock check: the slot must still hold the chosen seq after the copy;
// torn[0] counts rejected (overwritten-while-read) payloads.
__global__ void k_async_check(const unsigned long long *seqs, unsigned long long *pick, unsigned long long *applied,
                              int *torn) {
    if (pick[0] == 0) return;
    __threadfence_system();
    if (((const volatile unsigned long long *)seqs)[pick[1]] != pick[0]) {
        atomicAdd(torn, 1);
        pick[0] = 0;
        return;
    }
    *applied = pick[0];
}

__global__ void k_async_apply(const DBlock *__restrict__ blocks, int b, int gdir, long long n,
                              const unsigned long long *pick, const double *stage) {
    if (pick[0] == 0) return;
    double *g = blocks[b].ghost[gdir];
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x)
        g[c] = stage[c];
}

// ------------------------------------------------------------------ seeded rhs on the device
// numpy's Generator(PCG64).uniform(low, high, n) reproduced bit for bit: PCG64
// = 128-bit LCG (state = state * M + inc) with XSL-RR output of the new state;
// a double is (raw >> 11) * 2^-53 and the sample low + (high - low) * u.  Each
// thread jumps ahead to its chunk (O(log n) LCG power) and steps sequentially.

__device__ __forceinline__ unsigned long long pcg_xsl_rr(unsigned __int128 x) {
    const unsigned rot = (unsigned)(x >> 122);
    const unsigned long long v = (unsigned long long)(x >> 64) ^ (unsigned long long)x;
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

__global__ void k_pcg64_uniform(double *out, long long n, unsigned long long s_hi, unsigned long long s_lo,
                                unsigned long long i_hi, unsigned long long i_lo, double low, double range,
                                int chunk) {
    const unsigned __int128 M = ((unsigned __int128)0x2360ed051fc65da4ull << 64) | 0x4385df649fccf645ull;
    const unsigned __int128 inc = ((unsigned __int128)i_hi << 64) | i_lo;
    unsigned __int128 st = ((unsigned __int128)s_hi << 64) | s_lo;
    const long long start = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * chunk;
    if (start >= n) return;
    // jump ahead `start` steps: (A, C) <- composition of (M, inc) applied start times
    unsigned __int128 acc_mult = 1, acc_plus = 0, cur_mult = M, cur_plus = inc;
    for (unsigned long long d = (unsigned long long)start; d; d >>= 1) {
        if (d & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
    }
    st = acc_mult * st + acc_plus;
    const long long end = min(n, start + chunk);
    for (long long i = start; i < end; ++i) {
        st = st * M + inc;
        const double u = (double)(pcg_xsl_rr(st) >> 11) * (1.0 / 9007199254740992.0);
        out[i] = __dadd_rn(low, __dmul_rn(range, u));
    }
}

// ------------------------------------------------------------------ vector helpers
// Power-iteration support (linalg.py:243-276): ||x||_2 with a fixed
// reduction order (VEC_CTAS grid-stride partials, then one ordered tree), so
// repeats are bitwise identical on any GPU; y = x / d elementwise.
constexpr int VEC_CTAS = 296, VEC_NT = 256;

__global__ void __launch_bounds__(VEC_NT) k_vec_sq_partial(const double *__restrict__ x, long long n,
                                                            double *__restrict__ part) {
    __shared__ double red[VEC_NT / 32];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * VEC_NT + threadIdx.x; i < n; i += (long long)VEC_CTAS * VEC_NT)
        s = add(s, mul(x[i], x[i]));
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < VEC_NT / 32; ++w) t = add(t, red[w]);
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(VEC_NT) k_vec_sq_final(double *work) {
    __shared__ double scratch[256];
    const double v = range_sum<VEC_NT>(work + 1, 0, VEC_CTAS, scratch);
    if (threadIdx.x == 0) work[0] = sqrt(v);
}

__global__ void k_vec_div(const double *__restrict__ x, long long n, double d, double *__restrict__ y) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = __ddiv_rn(x[i], d);
}

// ------------------------------------------------------------------ host helpers

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encoder() {
    if (g_encode) return BS_OK;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
        return fail(BS_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return BS_OK;
}

// 3-D map over a block's pitched padded box; haloed (TX+4 x TY+2) or bare (TX x TY) plane boxes.
// Box starts are 16-byte aligned in x: tile origins are multiples of TX, haloed boxes start at x0-2.
int encode_map(CUtensorMap *m, const void *ptr, const DBlock &B, bool halo, int depth = 1) {
    if (int e = get_encoder()) return e;
    cuuint64_t dims[3] = {(cuuint64_t)B.pdim[0], (cuuint64_t)B.pdim[1], (cuuint64_t)B.pdim[2]};
    cuuint64_t strides[2] = {(cuuint64_t)B.pitch * 8, (cuuint64_t)B.pitch * B.pdim[1] * 8};
    cuuint32_t box[3] = {(cuuint32_t)(halo ? SX : TX), (cuuint32_t)(halo ? HY : TY), (cuuint32_t)depth};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void *>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(BS_EINVAL, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return BS_OK;
}

}  // namespace

// ====================================================================== context

// Kernels launched by this library.  Atomic: the asynchronous driver's block
// threads call into the library concurrently (one context each).
static std::atomic<unsigned long long> g_launches{0};

struct bs_ctx {
    int device = 0;
    bool box = true;  // every block has overlap 0: compile-time box-region kernels
    int nblocks = 0;
    int nctas = 0;
    std::vector<DBlock> hblocks;
    DBlock *dblocks = nullptr;
    DState *dstates = nullptr;
    CUtensorMap *dtmaps = nullptr;
    int *dcta_block = nullptr;
    int *dpcta_block = nullptr;
    int npctas = 0;
    double *dpartials = nullptr;
    unsigned *dblk_counter = nullptr;
    unsigned *dlaunch_counter = nullptr;
    unsigned *dtile_counter = nullptr;     // dynamic tile hand-out of sweep launches
    std::map<const void *, int> sweep_cap;  // co-resident CTAs of each sweep kernel
    int *dnactive = nullptr;
    Control *dctl = nullptr;
    int *dactive = nullptr;
    int *dplan = nullptr;
    int plan_cap = 0;
    std::vector<int32_t> hplan;  // the plan dplan holds (a sweep loop repeats one plan: no copy per sweep)
    int *hpinned = nullptr;  // [0]: n_active, [1..]: active mask staging
    DState *hstates = nullptr;
    Control *hctl = nullptr;
    unsigned *dpost_counter = nullptr;     // async post completion counter
    unsigned long long *dpick = nullptr;   // async receive scratch
    // GMRES(m) workspace (bs_gmres_setup)
    int gm = 0;
    GState *dgstates = nullptr;
    CUtensorMap *dgmaps = nullptr;
    // device-side solve loop: RESID ; WHILE(any active) { S1 ; S2 ; IF(any verify) RESID }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    // point-Jacobi loop: RESID (serves INIT) ; WHILE(any active) { JAC }
    cudaGraph_t jgraph = nullptr;
    cudaGraphExec_t jgraph_exec = nullptr;
    // one GMRES(m) restart cycle (all Arnoldi passes, FORM, RESID) captured once
    cudaGraph_t ggraph = nullptr;
    cudaGraphExec_t ggraph_exec = nullptr;
    std::vector<cudaGraphExec_t> ggraph_blk;  // the same per block (one-block runs)
    long long gcycle_kernels = 0;
    cudaStream_t cap_stream = nullptr;
    int run_kind = KIND_CG;    // solve armed last: bs_run drives its loop
    int pgrid = -1;            // persistent CG grid (co-resident CTAs), -1 = not computed
    int sgrid = -1;            // streaming persistent CG grid (k_cg_stream), -1 = not computed
    int part_stride = 0;       // per-quantity size of a parity buffer of dpartials
    int stream_sumk = 0;       // tiles per lane of a whole sweep (k_cg_stream)
    int run_path = -1;         // bs_ctx_run_path
    bool jac_dirty = false;    // a Jacobi iterate may sit in p[0] (flush before other solves)
    // optional CUDA-event timing of the sweep kernels (launch mode only)
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    double op_ms[3] = {0.0, 0.0, 0.0};
    long long op_n[3] = {0, 0, 0};
};

namespace {

int set_dev(bs_ctx *c) {
    BS_CU(cudaSetDevice(c->device));
    return BS_OK;
}

int upload_active(bs_ctx *c, const int32_t *active, cudaStream_t st, const int **dptr) {
    if (!active) {
        *dptr = nullptr;
        return BS_OK;
    }
    // the pinned staging slot is reused by the next call: finish this copy first
    BS_CU(cudaStreamSynchronize(st));
    std::memcpy(c->hpinned + 1, active, sizeof(int) * c->nblocks);
    BS_CU(cudaMemcpyAsync(c->dactive, c->hpinned + 1, sizeof(int) * c->nblocks, cudaMemcpyHostToDevice, st));
    BS_CU(cudaStreamSynchronize(st));
    *dptr = c->dactive;
    return BS_OK;
}

KParams make_params(bs_ctx *c, bool graph, cudaGraphConditionalHandle hl = 0,
                    cudaGraphConditionalHandle hv = 0) {
    KParams P;
    P.blocks = c->dblocks;
    P.states = c->dstates;
    P.tmaps = c->dtmaps;
    P.cta_block = c->dcta_block;
    P.nblocks = c->nblocks;
    P.nctas = c->nctas;
    P.pcta_block = c->dpcta_block;
    P.npctas = c->npctas;
    P.partials = c->dpartials;
    P.blk_counter = c->dblk_counter;
    P.launch_counter = c->dlaunch_counter;
    P.tile_counter = c->dtile_counter;
    P.n_active = c->dnactive;
    P.ctl = c->dctl;
    P.h_loop = hl;
    P.h_verify = hv;
    P.use_graph = graph ? 1 : 0;
    P.gstates = c->dgstates;
    P.gmaps = c->dgmaps;
    P.launch_j = 0;
    P.launch_i = 0;
    P.cta_base = 0;
    P.pcta_base = 0;
    P.ntiles = c->nctas;
    P.part_stride = c->part_stride;
    return P;
}

// Grid of a sweep over `ntiles` tiles: one CTA per co-resident slot
// (occupancy x SMs), each streaming tiles until the launch's counter runs
// out.  BS_SWEEP_TILES=1 launches one CTA per tile instead (A/B switch).
int sweep_ctas(bs_ctx *c, const void *fn, int smem, int ntiles) {
    static const int one_per_cta = [] {
        const char *e = std::getenv("BS_SWEEP_TILES");
        return e && std::atoi(e) == 1;
    }();
    if (one_per_cta || ntiles <= 0) return std::max(ntiles, 1);
    auto it = c->sweep_cap.find(fn);
    if (it == c->sweep_cap.end()) {
        int per_sm = 0, sms = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHR, smem) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || per_sm < 1) {
            cudaGetLastError();
            per_sm = 0;
        }
        if (const char *e = std::getenv("BS_SWEEP_PER_SM"))  // A/B: fewer resident sweep CTAs per SM
            per_sm = std::min(per_sm, std::max(1, std::atoi(e)));
        it = c->sweep_cap.emplace(fn, per_sm * sms).first;
    }
    return it->second > 0 ? std::min(ntiles, it->second) : ntiles;
}

// Grid of a sweep (pointwise) launch over every block (blk < 0) or only
// block blk's CTA range, with the matching CTA-table base in P.
template <int OPK>
void *sweep_fn(bool box) {
    return box ? (void *)k_sweep<OPK, true> : (void *)k_sweep<OPK, false>;
}

int sweep_grid(bs_ctx *c, KParams &P, int blk, const void *fn, int smem) {
    if (blk >= 0) {
        const DBlock &B = c->hblocks[blk];
        P.cta_base = B.cta_begin;
        P.ntiles = B.cta_end - B.cta_begin;
    }
    return sweep_ctas(c, fn, smem, P.ntiles);
}

int point_grid(bs_ctx *c, KParams &P, int blk) {
    if (blk < 0) return c->npctas;
    const DBlock &B = c->hblocks[blk];
    P.pcta_base = B.pcta_begin;
    return B.pcta_end - B.pcta_begin;
}

template <int PKK>
void launch_point(bs_ctx *c, cudaStream_t st, int j, int i, int blk = -1) {
    KParams P = make_params(c, false);
    P.launch_j = j;
    P.launch_i = i;
    const int grid = point_grid(c, P, blk);
    constexpr int smem = (NQ * (NPT / 32) + 256 + 8) * 8;
    if (c->box)
        k_point<PKK, true><<<grid, NPT, smem, st>>>(P);
    else
        k_point<PKK, false><<<grid, NPT, smem, st>>>(P);
    ++g_launches;
}

void launch_gspmv(bs_ctx *c, cudaStream_t st, int j, int blk = -1) {
    KParams P = make_params(c, false);
    P.launch_j = j;
    const int grid = sweep_grid(c, P, blk, sweep_fn<OP_GSPMV>(c->box), op_smem(OP_GSPMV));
    if (c->box)
        k_sweep<OP_GSPMV, true><<<grid, NTHR, op_smem(OP_GSPMV), st>>>(P);
    else
        k_sweep<OP_GSPMV, false><<<grid, NTHR, op_smem(OP_GSPMV), st>>>(P);
    ++g_launches;
}


template <int OPK>
void launch_sweep(bs_ctx *c, cudaStream_t st, int slot, int blk = -1) {
    KParams P = make_params(c, false);
    const int grid = sweep_grid(c, P, blk, sweep_fn<OPK>(c->box), op_smem(OPK));
    if (c->timing && slot >= 0) cudaEventRecord(c->ev[2 * slot], st);
    if (c->box)
        k_sweep<OPK, true><<<grid, NTHR, op_smem(OPK), st>>>(P);
    else
        k_sweep<OPK, false><<<grid, NTHR, op_smem(OPK), st>>>(P);
    if (c->timing && slot >= 0) cudaEventRecord(c->ev[2 * slot + 1], st);
    ++g_launches;
}

void launch_cycle(bs_ctx *c, cudaStream_t st, int cycle) {
    launch_sweep<OP_RESID>(c, st, 3 * cycle + 0);
    launch_sweep<OP_S1>(c, st, 3 * cycle + 1);
    launch_sweep<OP_S2>(c, st, 3 * cycle + 2);
}

void harvest_timing(bs_ctx *c, int cycles) {
    for (int i = 0; i < cycles; ++i)
        for (int o = 0; o < 3; ++o) {
            float ms = 0.f;
            const int slot = 3 * i + o;
            if (cudaEventElapsedTime(&ms, c->ev[2 * slot], c->ev[2 * slot + 1]) == cudaSuccess) {
                c->op_ms[o] += ms;
                c->op_n[o] += 1;
            }
        }
}

template <int OPK>
int add_sweep_node(bs_ctx *c, cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, int ndeps,
                   cudaGraphConditionalHandle hl, cudaGraphConditionalHandle hv) {
    KParams P = make_params(c, true, hl, hv);  // copied by the runtime at node creation
    void *args[] = {&P};
    cudaKernelNodeParams kp = {};
    kp.func = sweep_fn<OPK>(c->box);
    kp.gridDim = dim3(sweep_ctas(c, kp.func, op_smem(OPK), P.ntiles));
    kp.blockDim = dim3(NTHR);
    kp.sharedMemBytes = op_smem(OPK);
    kp.kernelParams = args;
    BS_CU(cudaGraphAddKernelNode(node, g, deps, ndeps, &kp));
    return BS_OK;
}

// Graph: RESID (serves INIT) -> WHILE(active) { S1 -> S2 -> IF(verify) { RESID } }
int build_graph(bs_ctx *c) {
    if (c->graph_exec) return BS_OK;
    cudaGraph_t g;
    BS_CU(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop;
    BS_CU(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_init;
    if (int e = add_sweep_node<OP_RESID>(c, g, &n_init, nullptr, 0, h_loop, 0)) return e;

    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_loop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t n_while;
    BS_CU(cudaGraphAddNode(&n_while, g, &n_init, 1, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];

    cudaGraphConditionalHandle h_verify;
    BS_CU(cudaGraphConditionalHandleCreate(&h_verify, body, 0, 0));
    cudaGraphNode_t n_s1, n_s2;
    if (int e = add_sweep_node<OP_S1>(c, body, &n_s1, nullptr, 0, h_loop, h_verify)) return e;
    if (int e = add_sweep_node<OP_S2>(c, body, &n_s2, &n_s1, 1, h_loop, h_verify)) return e;
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_verify;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t n_if;
    BS_CU(cudaGraphAddNode(&n_if, body, &n_s2, 1, &ip));
    cudaGraph_t ifbody = ip.conditional.phGraph_out[0];
    cudaGraphNode_t n_v;
    if (int e = add_sweep_node<OP_RESID>(c, ifbody, &n_v, nullptr, 0, h_loop, h_verify)) return e;

    cudaGraphExec_t ex;
    BS_CU(cudaGraphInstantiate(&ex, g, 0));
    c->graph = g;
    c->graph_exec = ex;
    return BS_OK;
}

// Graph: RESID (serves INIT) -> WHILE(active) { JAC }
int build_jacobi_graph(bs_ctx *c) {
    if (c->jgraph_exec) return BS_OK;
    cudaGraph_t g;
    BS_CU(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop;
    BS_CU(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t n_init;
    if (int e = add_sweep_node<OP_RESID>(c, g, &n_init, nullptr, 0, h_loop, 0)) return e;
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_loop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t n_while;
    BS_CU(cudaGraphAddNode(&n_while, g, &n_init, 1, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    cudaGraphNode_t n_j;
    if (int e = add_sweep_node<OP_JAC>(c, body, &n_j, nullptr, 0, h_loop, 0)) return e;
    cudaGraphExec_t ex;
    BS_CU(cudaGraphInstantiate(&ex, g, 0));
    c->jgraph = g;
    c->jgraph_exec = ex;
    return BS_OK;
}

// x := x + alpha_pend p / the Jacobi iterate, for every block with one pending
void launch_flush(bs_ctx *c, cudaStream_t st) {
    g_launches += 2;
    k_flush<<<dim3(592, c->nblocks), 256, 0, st>>>(c->dblocks, c->dstates);
    k_clear_pend<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dstates, c->nblocks);
    c->jac_dirty = false;
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

const char *bs_last_error(void) { return g_err.c_str(); }

int bs_ctx_create(int device, int nblocks, const bs_block_desc *blocks, int z_chunk, bs_ctx **out) {
    if (!out || !blocks || nblocks < 1) return fail(BS_EINVAL, "bs_ctx_create: bad arguments");
    bs_ctx *c = new bs_ctx();
    c->device = device;
    // profiling: BS_LAUNCH_MODE=1 runs every solve in launch mode (one kernel
    // launch per sweep, CUDA events around each) so that ncu sees the sweep
    // kernels, which it cannot profile inside conditional CUDA graphs
    if (const char *e = std::getenv("BS_LAUNCH_MODE")) c->timing = std::atoi(e) != 0;
    c->nblocks = nblocks;
    if (int e = set_dev(c)) {
        delete c;
        return e;
    }
    std::vector<int> cta_block;
    std::vector<CUtensorMap> maps((size_t)nblocks * NTM);
    for (int b = 0; b < nblocks; ++b) {
        const bs_block_desc &d = blocks[b];
        DBlock B;
        std::memset(&B, 0, sizeof(B));
        if (d.overlap < 0) {
            delete c;
            return fail(BS_EINVAL, "bs_ctx_create: overlap must be non-negative");
        }
        for (int a = 0; a < 3; ++a) {
            B.gn[a] = d.global_dims[a];
            B.lo[a] = d.owned_lo[a];
            B.hi[a] = d.owned_hi[a];
            if (B.gn[a] < 1 || B.lo[a] < 0 || B.hi[a] > B.gn[a] || B.lo[a] >= B.hi[a]) {
                delete c;
                return fail(BS_EINVAL,
                            "bs_ctx_create: block " + std::to_string(b) + " has an empty or out-of-grid owned box");
            }
            B.plo[a] = std::max(0, B.lo[a] - d.overlap);
            B.pdim[a] = std::min(B.gn[a], B.hi[a] + d.overlap) - B.plo[a];
        }
        B.pitch = (B.pdim[0] + PITCH_ALIGN - 1) / PITCH_ALIGN * PITCH_ALIGN;
        B.overlap = d.overlap;
        if (d.overlap != 0) c->box = false;
        B.x = d.x;
        B.r = d.r;
        B.p[0] = d.p0;
        B.p[1] = d.p1;
        B.b = d.b;
        for (int q = 0; q < BS_NDIR; ++q) B.ghost[q] = d.ghost[q];
        B.hist = d.history;
        B.hist_cap = d.history_cap;
        B.remote = d.remote != 0;
        if (B.remote) {
            // phantom: geometry + snapshot pointer only; no tiles, no chunks
            if (!B.r || d.overlap == 0 || reinterpret_cast<uintptr_t>(B.r) % 16) {
                delete c;
                return fail(BS_EINVAL, "bs_ctx_create: remote block " + std::to_string(b) +
                                           " needs overlap > 0 and a 16-byte aligned snapshot pointer");
            }
            for (int q = 0; q < BS_NDIR; ++q) B.ghost[q] = nullptr;
            B.tiles_x = B.tiles_y = B.tiles_z = 0;
            B.cz = 1;
            B.cta_begin = B.cta_end = (int)cta_block.size();
            c->hblocks.push_back(B);
            continue;
        }
        if (!B.x || !B.r || !B.p[0] || !B.p[1] || !B.b) {
            delete c;
            return fail(BS_EINVAL, "bs_ctx_create: null vector pointer for block " + std::to_string(b));
        }
        for (const void *ptr :
             {(const void *)B.x, (const void *)B.r, (const void *)B.p[0], (const void *)B.p[1], (const void *)B.b})
            if (reinterpret_cast<uintptr_t>(ptr) % 16) {
                delete c;
                return fail(BS_EINVAL, "bs_ctx_create: vectors must be 16-byte aligned");
            }
        B.tiles_x = (B.pdim[0] + TX - 1) / TX;
        B.tiles_y = (B.pdim[1] + TY - 1) / TY;
        {
            // Tiles: full-depth columns (long z-marches amortise the 2 re-staged
            // planes and the pipeline ramp) when the block has enough columns
            // to fill the GPU, else z split into chunks of >= 32 planes
            // (z_chunk > 0 forces the chunk length).  All tiles stream z in
            // lockstep.  A function of the block alone: tile partials (and so
            // every reduction) do not depend on which blocks share a GPU.
            const long long cols = (long long)B.tiles_x * B.tiles_y;
            long long nch = 1;
            if (z_chunk > 0) nch = (B.pdim[2] + z_chunk - 1) / z_chunk;
            else if (cols < 148 && B.pdim[2] >= 64) nch = std::min<long long>((256 + cols - 1) / cols, B.pdim[2] / 32);
            B.cz = (int)((B.pdim[2] + nch - 1) / nch);
            B.tiles_z = (B.pdim[2] + B.cz - 1) / B.cz;
        }
        B.cta_begin = (int)cta_block.size();
        const long long ntile = (long long)B.tiles_x * B.tiles_y * B.tiles_z;
        for (long long t = 0; t < ntile; ++t) cta_block.push_back(b);
        B.cta_end = (int)cta_block.size();
        CUtensorMap *m = &maps[(size_t)b * NTM];
        int e = 0;
        if (!e) e = encode_map(&m[TM_P0H_S2], B.p[0], B, true, op_zp(OP_S2));
        if (!e) e = encode_map(&m[TM_P1H_S2], B.p[1], B, true, op_zp(OP_S2));
        if (!e) e = encode_map(&m[TM_RO_S2], B.r, B, false, op_zp(OP_S2));
        if (!e) e = encode_map(&m[TM_RH_S1], B.r, B, true, op_zp(OP_S1));
        if (!e) e = encode_map(&m[TM_P0H_S1], B.p[0], B, true, op_zp(OP_S1));
        if (!e) e = encode_map(&m[TM_P1H_S1], B.p[1], B, true, op_zp(OP_S1));
        if (!e) e = encode_map(&m[TM_XO_S1], B.x, B, false, op_zp(OP_S1));
        if (!e) e = encode_map(&m[TM_XH_J], B.x, B, true, op_zp(OP_JAC));
        if (!e) e = encode_map(&m[TM_P0H_J], B.p[0], B, true, op_zp(OP_JAC));
        if (!e) e = encode_map(&m[TM_BO_J], B.b, B, false, op_zp(OP_JAC));
        if (!e) e = encode_map(&m[TM_XH_R], B.x, B, true, op_zp(OP_RESID));
        if (!e) e = encode_map(&m[TM_P0H_R], B.p[0], B, true, op_zp(OP_RESID));
        if (!e) e = encode_map(&m[TM_P1H_R], B.p[1], B, true, op_zp(OP_RESID));
        if (!e) e = encode_map(&m[TM_BO_R], B.b, B, false, op_zp(OP_RESID));
        if (e) {
            delete c;
            return e;
        }
        c->hblocks.push_back(B);
    }
    // pointwise table: fixed contiguous chunks of each block (streaming kernels
    // want many CTAs and long contiguous runs; the chunk -> CTA map is a
    // function of the block alone, so per-block reductions stay independent of
    // the co-resident blocks)
    std::vector<int> pcta_block;
    for (int b = 0; b < nblocks; ++b) {
        DBlock &B = c->hblocks[b];
        const long long n = (long long)B.pitch * B.pdim[1] * B.pdim[2];
        B.pcta_begin = (int)pcta_block.size();
        if (!B.remote)
            for (long long t = 0; t < (n + PCHUNK - 1) / PCHUNK; ++t) pcta_block.push_back(b);
        B.pcta_end = (int)pcta_block.size();
    }
    c->npctas = (int)pcta_block.size();
    // neighbour lists (problems.py:343-349): extended regions within one stencil
    // step, i.e. L1 gap between owned boxes <= 2o+1; ascending block ids
    for (int a = 0; a < nblocks; ++a) {
        DBlock &A = c->hblocks[a];
        A.nnbr = 0;
        for (int b = 0; b < nblocks; ++b) {
            if (b == a) continue;
            const DBlock &Bn = c->hblocks[b];
            int gap = 0;
            for (int d = 0; d < 3; ++d)
                gap += std::max(0, std::max(A.lo[d] - (Bn.hi[d] - 1), Bn.lo[d] - (A.hi[d] - 1)));
            if (gap <= A.overlap + Bn.overlap + 1) {
                if (A.nnbr >= MAXNBR) {
                    delete c;
                    return fail(BS_EINVAL, "bs_ctx_create: too many neighbours for block " + std::to_string(a));
                }
                A.nbr[A.nnbr++] = b;
            }
        }
    }
    c->nctas = (int)cta_block.size();
    cudaError_t e = cudaSuccess;
    e = cudaMalloc(&c->dblocks, sizeof(DBlock) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dstates, sizeof(DState) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dtmaps, sizeof(CUtensorMap) * maps.size());
    if (e == cudaSuccess) e = cudaMalloc(&c->dcta_block, sizeof(int) * c->nctas);
    // per quantity: one partial per sweep tile / pointwise chunk, or one lane
    // sum per (block, lane) for k_cg_stream; x2: persistent parity buffers
    c->part_stride = std::max(std::max(c->nctas, c->npctas), nblocks * LANES);
    if (e == cudaSuccess) e = cudaMalloc(&c->dpartials, 2 * sizeof(double) * NQ * c->part_stride);
    if (e == cudaSuccess) e = cudaMalloc(&c->dpcta_block, sizeof(int) * c->npctas);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dpcta_block, pcta_block.data(), sizeof(int) * c->npctas, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&c->dblk_counter, sizeof(unsigned) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dlaunch_counter, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&c->dtile_counter, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&c->dnactive, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->dctl, sizeof(Control));
    if (e == cudaSuccess) e = cudaMalloc(&c->dactive, sizeof(int) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dpost_counter, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(c->dpost_counter, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&c->dpick, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaHostAlloc(&c->hpinned, sizeof(int) * (nblocks + 1), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&c->hstates, sizeof(DState) * nblocks, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&c->hctl, sizeof(Control), cudaHostAllocDefault);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dblocks, c->hblocks.data(), sizeof(DBlock) * nblocks, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dtmaps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dcta_block, cta_block.data(), sizeof(int) * c->nctas, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(c->dstates, 0, sizeof(DState) * nblocks);
    if (e == cudaSuccess) e = cudaMemset(c->dblk_counter, 0, sizeof(unsigned) * nblocks);
    if (e == cudaSuccess) e = cudaMemset(c->dlaunch_counter, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(c->dtile_counter, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(c->dnactive, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->dctl, 0, sizeof(Control));
    {
        const void *fns[] = {sweep_fn<OP_RESID>(true),    sweep_fn<OP_RESID>(false), sweep_fn<OP_S1>(true),
                             sweep_fn<OP_S1>(false),      sweep_fn<OP_S2>(true),     sweep_fn<OP_S2>(false),
                             sweep_fn<OP_GSPMV>(true),    sweep_fn<OP_GSPMV>(false), sweep_fn<OP_JAC>(true),
                             sweep_fn<OP_JAC>(false),     (const void *)k_apply<true>,
                             (const void *)k_cg_persistent<true>, (const void *)k_cg_persistent<false>,
                             (const void *)k_apply<false>, (const void *)k_cg_stream<true>,
                             (const void *)k_cg_stream<false>};
        for (const void *f : fns)
            if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    }
    if (e != cudaSuccess) {
        bs_ctx_destroy(c);
        return fail(BS_ECUDA, std::string("bs_ctx_create: ") + cudaGetErrorString(e));
    }
    *out = c;
    return BS_OK;
}

int bs_ctx_destroy(bs_ctx *c) {
    if (!c) return BS_OK;
    cudaSetDevice(c->device);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    if (c->graph) cudaGraphDestroy(c->graph);
    if (c->jgraph_exec) cudaGraphExecDestroy(c->jgraph_exec);
    if (c->jgraph) cudaGraphDestroy(c->jgraph);
    if (c->ggraph_exec) cudaGraphExecDestroy(c->ggraph_exec);
    if (c->ggraph) cudaGraphDestroy(c->ggraph);
    for (cudaGraphExec_t e : c->ggraph_blk)
        if (e) cudaGraphExecDestroy(e);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    cudaFree(c->dblocks);
    cudaFree(c->dstates);
    cudaFree(c->dtmaps);
    cudaFree(c->dcta_block);
    cudaFree(c->dpcta_block);
    cudaFree(c->dpartials);
    cudaFree(c->dblk_counter);
    cudaFree(c->dlaunch_counter);
    cudaFree(c->dtile_counter);
    cudaFree(c->dnactive);
    cudaFree(c->dctl);
    cudaFree(c->dactive);
    cudaFree(c->dplan);
    cudaFree(c->dgstates);
    cudaFree(c->dgmaps);
    cudaFree(c->dpost_counter);
    cudaFree(c->dpick);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->hpinned) cudaFreeHost(c->hpinned);
    if (c->hstates) cudaFreeHost(c->hstates);
    if (c->hctl) cudaFreeHost(c->hctl);
    delete c;
    return BS_OK;
}

int bs_ctx_num_ctas(const bs_ctx *c) { return c ? c->nctas : 0; }

int bs_ctx_run_path(const bs_ctx *c) { return c ? c->run_path : -1; }

int bs_block_pitch(const bs_ctx *c, int block) {
    if (!c || block < 0 || block >= c->nblocks) return fail(BS_EINVAL, "bs_block_pitch: bad arguments");
    return c->hblocks[block].pitch;
}

unsigned long long bs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int bs_timing(bs_ctx *c, int enable, double *ms_out, long long *n_out) {
    if (!c) return fail(BS_EINVAL, "bs_timing: null context");
    if (ms_out)
        for (int o = 0; o < 3; ++o) ms_out[o] = c->op_ms[o];
    if (n_out)
        for (int o = 0; o < 3; ++o) n_out[o] = c->op_n[o];
    if (enable >= 0) {
        c->timing = enable != 0;
        for (int o = 0; o < 3; ++o) {
            c->op_ms[o] = 0.0;
            c->op_n[o] = 0;
        }
    }
    return BS_OK;
}

int bs_stencil_apply(bs_ctx *c, int block, const double *x, double *y, void *stream) {
    if (!c || block < 0 || block >= c->nblocks || !x || !y) return fail(BS_EINVAL, "bs_stencil_apply: bad arguments");
    if (reinterpret_cast<uintptr_t>(x) % 16) return fail(BS_EINVAL, "bs_stencil_apply: x must be 16-byte aligned");
    if (int e = set_dev(c)) return e;
    const DBlock &B = c->hblocks[block];
    CUtensorMap xmap;
    if (int e = encode_map(&xmap, x, B, true, op_zp(OP_APPLY))) return e;
    ++g_launches;
    if (B.overlap == 0)
        k_apply<true><<<B.cta_end - B.cta_begin, NTHR, op_smem(OP_APPLY), (cudaStream_t)stream>>>(c->dblocks, block, xmap, y);
    else
        k_apply<false><<<B.cta_end - B.cta_begin, NTHR, op_smem(OP_APPLY), (cudaStream_t)stream>>>(c->dblocks, block, xmap, y);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_cg_begin(bs_ctx *c, int max_iterations, double tolerance, int basis, const int32_t *active,
                void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_cg_begin: null context");
    if (max_iterations < 1) return fail(BS_EINVAL, "max_iterations must be at least 1");
    if (!(tolerance >= 0.0)) return fail(BS_EINVAL, "tolerance must be non-negative");
    if (basis != BS_BASIS_RHS && basis != BS_BASIS_INITIAL) return fail(BS_EINVAL, "unknown tolerance basis");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const int *dact = nullptr;
    if (int e = upload_active(c, active, st, &dact)) return e;
    if (c->jac_dirty) launch_flush(c, st);
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, dact, c->nblocks, PH_INIT, max_iterations,
                                                   tolerance, basis, KIND_CG, 0);
    BS_CU(cudaGetLastError());
    c->run_kind = KIND_CG;
    return BS_OK;
}

int bs_jacobi_begin(bs_ctx *c, int max_iterations, double tolerance, int basis, const int32_t *active,
                    void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_jacobi_begin: null context");
    if (max_iterations < 1) return fail(BS_EINVAL, "max_iterations must be at least 1");
    if (!(tolerance >= 0.0)) return fail(BS_EINVAL, "tolerance must be non-negative");
    if (basis != BS_BASIS_RHS && basis != BS_BASIS_INITIAL) return fail(BS_EINVAL, "unknown tolerance basis");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const int *dact = nullptr;
    if (int e = upload_active(c, active, st, &dact)) return e;
    launch_flush(c, st);  // sweep 0 reads x itself: apply any pending CG update / Jacobi copy
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, dact, c->nblocks, PH_INIT, max_iterations,
                                                   tolerance, basis, KIND_JACOBI, 0);
    BS_CU(cudaGetLastError());
    c->run_kind = KIND_JACOBI;
    c->jac_dirty = true;
    return BS_OK;
}

int bs_sweep_resid(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_sweep_resid: null context");
    if (int e = set_dev(c)) return e;
    launch_sweep<OP_RESID>(c, (cudaStream_t)stream, -1);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_cancel(bs_ctx *c, const int32_t *active, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_cancel: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const int *dact = nullptr;
    if (int e = upload_active(c, active, st, &dact)) return e;
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, dact, c->nblocks, PH_DONE, 0, 0.0, 0, 0, 0);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_residual(bs_ctx *c, const int32_t *active, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_residual: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const int *dact = nullptr;
    if (int e = upload_active(c, active, st, &dact)) return e;
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, dact, c->nblocks, PH_RESID, 0, 0.0, 0, 0, 0);
    launch_sweep<OP_RESID>(c, st, -1);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

namespace {
// Run path of CG solves (BS_PERSIST, default 1): 1 = one persistent launch —
// k_cg_persistent when every tile has its own co-resident CTA, else the
// streaming k_cg_stream (<= MAXB_STREAM blocks); 0 = the CUDA-graph path;
// 2 = k_cg_persistent with tile loops; 3 = k_cg_stream always.  All paths
// give bitwise-identical results.
int persist_mode() {
    const char *env = std::getenv("BS_PERSIST");
    return env ? std::atoi(env) : 1;
}

bool use_persistent(bs_ctx *c) {
    const int mode = persist_mode();
    if (mode == 0 || mode == 3) return false;
    if (c->pgrid < 0) {
        int per_sm = 0, sms = 0, coop = 0;
        const void *fn = c->box ? (const void *)k_cg_persistent<true> : (const void *)k_cg_persistent<false>;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHR, SMEM_MAX) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess ||
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device) != cudaSuccess || !coop) {
            cudaGetLastError();
            c->pgrid = 0;
        } else {
            c->pgrid = std::min(c->nctas, per_sm * sms);
        }
    }
    if (c->pgrid <= 0) return false;
    return mode == 2 || c->pgrid == c->nctas;
}

bool use_stream(bs_ctx *c) {
    const int mode = persist_mode();
    if ((mode != 1 && mode != 3) || c->nblocks > MAXB_STREAM) return false;
    if (c->sgrid < 0) {
        int per_sm = 0, sms = 0, coop = 0;
        const void *fn = c->box ? (const void *)k_cg_stream<true> : (const void *)k_cg_stream<false>;
        int maxk = 0, sumk = 0;  // tiles per lane: of the largest block, of a whole sweep
        for (const DBlock &B : c->hblocks) {
            const int k = (B.cta_end - B.cta_begin + LANES - 1) / LANES;
            maxk = std::max(maxk, k);
            sumk += k;
        }
        // Static lanes put 2 CTAs on 108 SMs and 1 on 40: over long sweeps the
        // SMs with two fall behind, while the graph path's dynamic hand-out
        // over 3 CTAs on every SM stays balanced.  Measured per GPU on the
        // config-3 slabs (scripts/proxy_ab.sh, profiles/r02_stream_proxy.log):
        // stream 88.3 / 89.9 / 87.9 / 87.1 Gpts/s at 1 / 2 / 4 / 8 slabs
        // (4 / 8 / 16 / 32 tiles per lane), graph 80.0 / 89.5 / 92.4 / 93.2.
        c->stream_sumk = sumk;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHR, SMEM_MAX) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess ||
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device) != cudaSuccess || !coop) {
            cudaGetLastError();
            c->sgrid = 0;
        } else {
            // exactly LANES co-resident CTAs (one per reduction lane)
            c->sgrid = (per_sm * sms >= LANES && maxk <= MAXK_STREAM) ? LANES : 0;
        }
    }
    int limit = 8;
    if (const char *e = std::getenv("BS_STREAM_MAXK")) limit = std::atoi(e);
    return c->sgrid > 0 && (mode == 3 || c->stream_sumk <= limit);
}

}  // namespace

namespace {
// Jacobi solves: graph mode (one launch) or launch mode (timing), sweep count out
int run_jacobi(bs_ctx *c, int batch, int max_launches, cudaStream_t st, int64_t *sweeps_out) {
    if (!c->timing) {
        if (int e = build_jacobi_graph(c)) return e;
        ++g_launches;
        k_reset_control<<<1, 1, 0, st>>>(c->dctl, max_launches > 0 ? max_launches : 0);
        BS_CU(cudaGraphLaunch(c->jgraph_exec, st));
        BS_CU(cudaMemcpyAsync(c->hctl, c->dctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        const Control ctl = *c->hctl;
        g_launches += (long long)ctl.resid_runs + ctl.cycles;
        if (sweeps_out) *sweeps_out = (long long)ctl.resid_runs + ctl.cycles;
        if (ctl.stalled) return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
        return BS_OK;
    }
    int64_t launched = 1;
    launch_sweep<OP_RESID>(c, st, -1);
    for (;;) {
        BS_CU(cudaMemcpyAsync(c->hpinned, c->dnactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        if (c->hpinned[0] == 0) break;
        if (max_launches > 0 && launched >= max_launches) {
            if (sweeps_out) *sweeps_out = launched;
            return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
        }
        for (int i = 0; i < batch; ++i) launch_sweep<OP_JAC>(c, st, -1);
        launched += batch;
        BS_CU(cudaGetLastError());
    }
    if (sweeps_out) *sweeps_out = launched;
    return BS_OK;
}
}  // namespace

int bs_run(bs_ctx *c, int batch, int max_launches, void *stream, int64_t *sweeps_out) {
    if (!c) return fail(BS_EINVAL, "bs_run: null context");
    if (batch < 1) batch = 1;
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->run_kind == KIND_JACOBI) {
        c->run_path = c->timing ? 3 : 4;
        return run_jacobi(c, batch, max_launches, st, sweeps_out);
    }
    if (!c->timing && use_persistent(c)) {
        // the whole solve in one cooperative launch (software grid barriers)
        ++g_launches;
        k_reset_control<<<1, 1, 0, st>>>(c->dctl, max_launches > 0 ? (max_launches + 2) / 3 : 0);
        KParams P = make_params(c, false);
        void *args[] = {&P};
        const void *fn = c->box ? (const void *)k_cg_persistent<true> : (const void *)k_cg_persistent<false>;
        if (cudaLaunchCooperativeKernel(fn, dim3(c->pgrid), dim3(NTHR), args, SMEM_MAX, st) != cudaSuccess) {
            // e.g. another context holds SMs the grid needs: the graph path
            // computes the same thing (same tile partials, same order)
            cudaGetLastError();
            c->pgrid = 0;
        } else {
            c->run_path = 1;
            ++g_launches;
            BS_CU(cudaMemcpyAsync(c->hctl, c->dctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
            BS_CU(cudaStreamSynchronize(st));
            const Control ctl = *c->hctl;
            if (sweeps_out) *sweeps_out = (long long)ctl.resid_runs + 2LL * ctl.cycles;
            if (ctl.stalled) return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
            return BS_OK;
        }
    }
    if (!c->timing && use_stream(c)) {
        // the whole solve in one cooperative launch, tiles streamed per CTA
        ++g_launches;
        k_reset_control<<<1, 1, 0, st>>>(c->dctl, max_launches > 0 ? (max_launches + 2) / 3 : 0);
        KParams P = make_params(c, false);
        void *args[] = {&P};
        const void *fn = c->box ? (const void *)k_cg_stream<true> : (const void *)k_cg_stream<false>;
        if (cudaLaunchCooperativeKernel(fn, dim3(c->sgrid), dim3(NTHR), args, SMEM_MAX, st) != cudaSuccess) {
            cudaGetLastError();  // SMs held by another context: the graph path computes the same numbers
            c->sgrid = 0;
        } else {
            c->run_path = 2;
            ++g_launches;
            BS_CU(cudaMemcpyAsync(c->hctl, c->dctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
            BS_CU(cudaStreamSynchronize(st));
            const Control ctl = *c->hctl;
            if (sweeps_out) *sweeps_out = (long long)ctl.resid_runs + 2LL * ctl.cycles;
            if (ctl.stalled) return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
            return BS_OK;
        }
    }
    if (!c->timing) {
        // device-side loop: one graph launch runs the solves to completion
        if (int e = build_graph(c)) return e;
        c->run_path = 0;
        ++g_launches;
        k_reset_control<<<1, 1, 0, st>>>(c->dctl, max_launches > 0 ? (max_launches + 2) / 3 : 0);
        BS_CU(cudaGraphLaunch(c->graph_exec, st));
        BS_CU(cudaMemcpyAsync(c->hctl, c->dctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        const Control ctl = *c->hctl;
        // kernels the graph ran: per cycle S1 + S2, plus every residual sweep
        g_launches += (long long)ctl.resid_runs + 2LL * ctl.cycles;
        if (sweeps_out) *sweeps_out = (long long)ctl.resid_runs + 2LL * ctl.cycles;
        if (ctl.stalled) return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
        return BS_OK;
    }
    // launch mode with per-kernel CUDA events (profiling)
    c->run_path = 3;
    int64_t launched = 0;
    if ((int)c->ev.size() < 6 * batch) {
        for (int i = (int)c->ev.size(); i < 6 * batch; ++i) {
            cudaEvent_t e;
            BS_CU(cudaEventCreate(&e));
            c->ev.push_back(e);
        }
    }
    for (;;) {
        for (int i = 0; i < batch; ++i) launch_cycle(c, st, i);
        launched += 3LL * batch;
        BS_CU(cudaGetLastError());
        BS_CU(cudaMemcpyAsync(c->hpinned, c->dnactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        harvest_timing(c, batch);
        if (c->hpinned[0] == 0) break;
        if (max_launches > 0 && launched >= max_launches) {
            if (sweeps_out) *sweeps_out = launched;
            return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
        }
    }
    if (sweeps_out) *sweeps_out = launched;
    return BS_OK;
}

int bs_gmres_setup(bs_ctx *c, int m, const bs_gmres_desc *descs) {
    if (!c || !descs) return fail(BS_EINVAL, "bs_gmres_setup: bad arguments");
    if (m < 1 || m > MAXM) return fail(BS_EINVAL, "restart: GMRES restart must be in 1.." + std::to_string(MAXM));
    if (int e = set_dev(c)) return e;
    std::vector<CUtensorMap> maps((size_t)c->nblocks * (MAXM + 1));
    for (int b = 0; b < c->nblocks; ++b) {
        DBlock &B = c->hblocks[b];
        const bs_gmres_desc &d = descs[b];
        if (B.remote) continue;  // phantoms never solve
        if (!d.V || !d.W) return fail(BS_EINVAL, "bs_gmres_setup: null V or W");
        const long long n = (long long)B.pitch * B.pdim[1] * B.pdim[2];
        if (d.vstride < n || (d.vstride * 8) % 16) return fail(BS_EINVAL, "bs_gmres_setup: bad V stride");
        B.V = d.V;
        B.vstride = d.vstride;
        B.W = d.W;
        for (int j = 0; j < m; ++j)
            if (int e = encode_map(&maps[(size_t)b * (MAXM + 1) + j], B.V + (size_t)j * d.vstride, B, true,
                                   op_zp(OP_GSPMV)))
                return e;
        if (int e = encode_map(&maps[(size_t)b * (MAXM + 1) + MAXM], B.V, B, false, op_zp(OP_GSPMV))) return e;
    }
    cudaFree(c->dgmaps);
    c->dgmaps = nullptr;
    if (c->ggraph_exec) cudaGraphExecDestroy(c->ggraph_exec);  // captured the old maps
    if (c->ggraph) cudaGraphDestroy(c->ggraph);
    c->ggraph_exec = nullptr;
    c->ggraph = nullptr;
    for (cudaGraphExec_t &e : c->ggraph_blk) {
        if (e) cudaGraphExecDestroy(e);
        e = nullptr;
    }
    if (!c->dgstates) BS_CU(cudaMalloc(&c->dgstates, sizeof(GState) * c->nblocks));
    BS_CU(cudaMalloc(&c->dgmaps, sizeof(CUtensorMap) * maps.size()));
    BS_CU(cudaMemcpy(c->dgmaps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
    BS_CU(cudaMemcpy(c->dblocks, c->hblocks.data(), sizeof(DBlock) * c->nblocks, cudaMemcpyHostToDevice));
    c->gm = m;
    return BS_OK;
}

int bs_gmres_begin(bs_ctx *c, int max_iterations, double tolerance, int basis, const int32_t *active,
                   void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_gmres_begin: null context");
    if (!c->gm) return fail(BS_ESTATE, "bs_gmres_begin: call bs_gmres_setup first");
    if (max_iterations < 1) return fail(BS_EINVAL, "max_iterations must be at least 1");
    if (!(tolerance >= 0.0)) return fail(BS_EINVAL, "tolerance must be non-negative");
    if (basis != BS_BASIS_RHS && basis != BS_BASIS_INITIAL) return fail(BS_EINVAL, "unknown tolerance basis");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const int *dact = nullptr;
    if (int e = upload_active(c, active, st, &dact)) return e;
    if (c->jac_dirty) launch_flush(c, st);
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, dact, c->nblocks, PH_INIT, max_iterations,
                                                   tolerance, basis, KIND_GMRES, c->gm);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

namespace {
// Restart cycles of the armed GMRES solves of every block (blk < 0) or of
// block blk alone (launches cover only its CTAs; its cycle graph is
// captured once per block).  The one-block form lets blocks share one
// Krylov basis, solved one after another.
int gmres_run(bs_ctx *c, int blk, int max_cycles, cudaStream_t st, int64_t *kernels_out) {
    const unsigned long long l0 = g_launches;
    if (blk >= 0) {
        // W may hold another block's values (shared workspace): off-region
        // cells and row padding must read as exact zeros (see k_point)
        const DBlock &B = c->hblocks[blk];
        BS_CU(cudaMemsetAsync(B.W, 0, sizeof(double) * (size_t)B.vstride, st));
    }
    launch_sweep<OP_RESID>(c, st, -1, blk);  // INIT: rhs assembly + r0 (inner_solvers.py:153-159)
    if (blk >= 0 && c->ggraph_blk.size() != (size_t)c->nblocks) c->ggraph_blk.assign(c->nblocks, nullptr);
    cudaGraphExec_t &exec = blk < 0 ? c->ggraph_exec : c->ggraph_blk[blk];
    if (!exec) {
        // one restart cycle as a CUDA graph: m Arnoldi steps (NORM, SPMV + h0j,
        // MGS passes, FINAL), FORM, true residual — 3m + m(m-1)/2 + 2 kernels
        // replayed per cycle without host launch overhead
        if (!c->cap_stream) BS_CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = c->cap_stream;
        const unsigned long long g0 = g_launches;
        BS_CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int j = 0; j < c->gm; ++j) {  // one Arnoldi step per j; finished blocks skip
            launch_point<PK_NORM>(c, cs, j, 0, blk);
            launch_gspmv(c, cs, j, blk);
            for (int i = 1; i <= j; ++i) launch_point<PK_MGS>(c, cs, j, i, blk);
            launch_point<PK_FINAL>(c, cs, j, 0, blk);
        }
        launch_point<PK_FORM>(c, cs, 0, 0, blk);
        launch_sweep<OP_RESID>(c, cs, -1, blk);  // true residual -> stop or restart
        cudaGraph_t g = nullptr;
        BS_CU(cudaStreamEndCapture(cs, &g));
        c->gcycle_kernels = (long long)(g_launches - g0);
        g_launches = g0;  // captured, not launched
        BS_CU(cudaGraphInstantiate(&exec, g, 0));
        BS_CU(cudaGraphDestroy(g));
    }
    int cycles = 0;
    for (;;) {
        BS_CU(cudaGraphLaunch(exec, st));
        g_launches += c->gcycle_kernels;
        BS_CU(cudaGetLastError());
        if (blk < 0)
            BS_CU(cudaMemcpyAsync(c->hpinned, c->dnactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        else
            BS_CU(cudaMemcpyAsync(c->hpinned, &c->dstates[blk].phase, sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        ++cycles;
        const bool done = blk < 0 ? c->hpinned[0] == 0 : (c->hpinned[0] == PH_DONE || c->hpinned[0] == PH_IDLE);
        if (done) break;
        if (max_cycles > 0 && cycles >= max_cycles) {
            if (kernels_out) *kernels_out = (int64_t)(g_launches - l0);
            return fail(BS_ESTATE, "bs_gmres_run: solves still active after max_cycles restart cycles");
        }
    }
    if (kernels_out) *kernels_out = (int64_t)(g_launches - l0);
    return BS_OK;
}

}  // namespace

int bs_gmres_run(bs_ctx *c, int max_cycles, void *stream, int64_t *kernels_out) {
    if (!c) return fail(BS_EINVAL, "bs_gmres_run: null context");
    if (!c->gm) return fail(BS_ESTATE, "bs_gmres_run: call bs_gmres_setup first");
    if (int e = set_dev(c)) return e;
    return gmres_run(c, -1, max_cycles, (cudaStream_t)stream, kernels_out);
}

int bs_gmres_run_block(bs_ctx *c, int block, int max_cycles, void *stream, int64_t *kernels_out) {
    if (!c) return fail(BS_EINVAL, "bs_gmres_run_block: null context");
    if (!c->gm) return fail(BS_ESTATE, "bs_gmres_run_block: call bs_gmres_setup first");
    if (block < 0 || block >= c->nblocks) return fail(BS_EINVAL, "bs_gmres_run_block: block out of range");
    if (int e = set_dev(c)) return e;
    return gmres_run(c, block, max_cycles, (cudaStream_t)stream, kernels_out);
}

int bs_overlap_merge(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_overlap_merge: null context");
    if (int e = bs_overlap_snapshot(c, stream)) return e;
    return bs_overlap_combine(c, stream);
}

int bs_overlap_snapshot(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_overlap_snapshot: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches += 1;
    k_snapshot<<<dim3(296, c->nblocks), 256, 0, st>>>(c->dblocks);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_overlap_combine(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_overlap_combine: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    g_launches += 2;
    k_merge<<<dim3(296, c->nblocks), 256, 0, st>>>(c->dblocks);
    k_merge_faces<<<dim3(64, c->nblocks, BS_NDIR), 256, 0, st>>>(c->dblocks);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_owner_residual(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_owner_residual: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dblocks, c->dstates, nullptr, c->nblocks, PH_OWNRES, 0, 0.0, 0, 0, 0);
    launch_point<PK_OWNRES>(c, st, 0, 0);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_async_post_slot(bs_ctx *c, int block, int dir, double *ring, uint64_t *seqs, int64_t *deliver, int slot,
                       uint64_t seq, int64_t deliver_at, void *stream) {
    if (!c || block < 0 || block >= c->nblocks || dir < 0 || dir >= BS_NDIR || !ring || !seqs || slot < 0)
        return fail(BS_EINVAL, "bs_async_post: bad arguments");
    if (int e = set_dev(c)) return e;
    g_launches += 2;
    k_async_retire<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long *)seqs, slot);
    k_async_post<<<64, 256, 0, (cudaStream_t)stream>>>(c->dblocks, c->dstates, block, dir, ring,
                                                       (unsigned long long *)seqs, slot, (unsigned long long)seq,
                                                       (long long *)deliver, (long long)deliver_at,
                                                       c->dpost_counter);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_async_post(bs_ctx *c, int block, int dir, double *ring, uint64_t *seqs, int R, uint64_t seq,
                  void *stream) {
    if (R < 1) return fail(BS_EINVAL, "bs_async_post: bad arguments");
    return bs_async_post_slot(c, block, dir, ring, seqs, nullptr, (int)(seq % (uint64_t)R), seq, 0, stream);
}

int bs_async_receive(bs_ctx *c, int block, int ghost_dir, const double *ring, const uint64_t *seqs, int R,
                     uint64_t *applied, double *stage, int *torn, void *stream) {
    return bs_async_receive_at(c, block, ghost_dir, ring, seqs, nullptr, R, 0, applied, stage, torn, stream);
}

int bs_async_receive_at(bs_ctx *c, int block, int ghost_dir, const double *ring, const uint64_t *seqs,
                        const int64_t *deliver, int R, int64_t receiver_k, uint64_t *applied, double *stage,
                        int *torn, void *stream) {
    if (!c || block < 0 || block >= c->nblocks || ghost_dir < 0 || ghost_dir >= BS_NDIR || !ring || !seqs || R < 1 ||
        !applied || !stage || !torn)
        return fail(BS_EINVAL, "bs_async_receive: bad arguments");
    if (!c->hblocks[block].ghost[ghost_dir]) return fail(BS_EINVAL, "bs_async_receive: no ghost plane");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = plane_len(c->hblocks[block].pdim, ghost_dir);
    g_launches += 4;
    k_async_pick<<<1, 1, 0, st>>>((const unsigned long long *)seqs, (const long long *)deliver, R,
                                  (long long)receiver_k, (const unsigned long long *)applied, c->dpick);
    k_async_copy<<<64, 256, 0, st>>>(c->dblocks, block, ghost_dir, ring, n, c->dpick, stage);
    k_async_check<<<1, 1, 0, st>>>((const unsigned long long *)seqs, c->dpick, (unsigned long long *)applied, torn);
    k_async_apply<<<64, 256, 0, st>>>(c->dblocks, block, ghost_dir, n, c->dpick, stage);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_uniform_pcg64(double *out, int64_t n, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, double low, double high, void *stream) {
    if (!out || n < 0) return fail(BS_EINVAL, "bs_uniform_pcg64: bad arguments");
    if (n == 0) return BS_OK;
    const int chunk = 256;
    const long long threads = (n + chunk - 1) / chunk;
    ++g_launches;
    k_pcg64_uniform<<<(unsigned)((threads + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        out, n, state_hi, state_lo, inc_hi, inc_lo, low, high - low, chunk);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

#ifdef BS_TRACE
int bs_strace_read(unsigned long long *out) {  // PT_SWEEPS x 8 x PT_CTAS (BS_TRACE builds)
    if (!out) return fail(BS_EINVAL, "bs_strace_read: bad arguments");
    BS_CU(cudaMemcpyFromSymbol(out, g_strace, sizeof(g_strace)));
    return BS_OK;
}

int bs_ptrace_read(unsigned long long *out) {  // PT_SWEEPS x 5 x PT_CTAS
    if (!out) return fail(BS_EINVAL, "bs_ptrace_read: bad arguments");
    BS_CU(cudaMemcpyFromSymbol(out, g_ptrace, sizeof(g_ptrace)));
    return BS_OK;
}

int bs_trace_read(unsigned long long *out, int nctas) {
    if (!out || nctas < 0 || nctas > TRACE_CTAS) return fail(BS_EINVAL, "bs_trace_read: bad arguments");
    for (int i = 0; i < 5; ++i)
        BS_CU(cudaMemcpyFromSymbol(out + (size_t)i * nctas, g_trace, sizeof(unsigned long long) * nctas,
                                   sizeof(unsigned long long) * TRACE_CTAS * i));
    return BS_OK;
}
#endif

int bs_vec_nrm2(const double *x, int64_t n, double *work, void *stream) {
    if (!work || n < 0 || (n > 0 && !x)) return fail(BS_EINVAL, "bs_vec_nrm2: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    g_launches += 2;
    k_vec_sq_partial<<<VEC_CTAS, VEC_NT, 0, st>>>(x, n, work + 1);
    k_vec_sq_final<<<1, VEC_NT, 0, st>>>(work);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_vec_scale(const double *x, int64_t n, double denom, double *y, void *stream) {
    if (n < 0 || (n > 0 && (!x || !y))) return fail(BS_EINVAL, "bs_vec_scale: bad arguments");
    if (n == 0) return BS_OK;
    ++g_launches;
    const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
    k_vec_div<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, denom, y);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_ipc_export(const void *ptr, unsigned char *handle_out, uint64_t *offset_out) {
    if (!ptr || !handle_out || !offset_out) return fail(BS_EINVAL, "bs_ipc_export: bad arguments");
    static PFN_cuMemGetAddressRange_v3020 range_fn = nullptr;
    if (!range_fn) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(BS_ECUDA, "cuMemGetAddressRange unavailable from the driver");
        range_fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range_fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(BS_ECUDA, "bs_ipc_export: not a device allocation");
    cudaIpcMemHandle_t h;
    BS_CU(cudaIpcGetMemHandle(&h, (void *)base));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((CUdeviceptr)ptr - base);
    return BS_OK;
}

int bs_ipc_open(const unsigned char *handle, uint64_t offset, void **ptr_out) {
    if (!handle || !ptr_out) return fail(BS_EINVAL, "bs_ipc_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    BS_CU(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr_out = (unsigned char *)base + offset;
    return BS_OK;
}

int bs_ipc_close(void *base) {
    if (!base) return BS_OK;
    BS_CU(cudaIpcCloseMemHandle(base));
    return BS_OK;
}

int bs_flush(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_flush: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    launch_flush(c, st);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_halo_pack(bs_ctx *c, int nplan, const int32_t *plan, void *stream) {
    if (!c || nplan < 0 || (nplan > 0 && !plan)) return fail(BS_EINVAL, "bs_halo_pack: bad arguments");
    if (nplan == 0) return BS_OK;
    if (int e = set_dev(c)) return e;
    for (int e = 0; e < nplan; ++e) {
        const int dst = plan[3 * e], dir = plan[3 * e + 1], src = plan[3 * e + 2];
        if (dst < 0 || dst >= c->nblocks || src < 0 || src >= c->nblocks || dir < 0 || dir >= BS_NDIR)
            return fail(BS_EINVAL, "bs_halo_pack: plan entry out of range");
        if (!c->hblocks[dst].ghost[dir]) return fail(BS_EINVAL, "bs_halo_pack: destination has no ghost plane");
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (nplan > c->plan_cap) {
        BS_CU(cudaStreamSynchronize(st));
        cudaFree(c->dplan);
        c->dplan = nullptr;
        BS_CU(cudaMalloc(&c->dplan, sizeof(int) * 3 * nplan));
        c->plan_cap = nplan;
        c->hplan.clear();
    }
    if (c->hplan.size() != (size_t)(3 * nplan) || memcmp(c->hplan.data(), plan, sizeof(int32_t) * 3 * nplan) != 0) {
        // the copy stages `plan` before returning (pageable host memory); kernels
        // already launched with the old plan run before it in stream order
        BS_CU(cudaMemcpyAsync(c->dplan, plan, sizeof(int) * 3 * nplan, cudaMemcpyHostToDevice, st));
        c->hplan.assign(plan, plan + 3 * nplan);
    }
    ++g_launches;
    // 256 CTAs per plane: four cells per thread at 512^2 (the grid-stride loop is a chain of dependent
    // load -> store rounds, so more threads in flight is what shortens it)
    k_halo_pack<<<dim3(256, nplan), 256, 0, st>>>(c->dblocks, c->dstates, c->dplan);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_read_reports(bs_ctx *c, bs_block_report *out, void *stream) {
    if (!c || !out) return fail(BS_EINVAL, "bs_read_reports: bad arguments");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    BS_CU(cudaMemcpyAsync(c->hstates, c->dstates, sizeof(DState) * c->nblocks, cudaMemcpyDeviceToHost, st));
    BS_CU(cudaStreamSynchronize(st));
    for (int b = 0; b < c->nblocks; ++b) {
        const DState &S = c->hstates[b];
        bs_block_report &R = out[b];
        R.phase = S.phase;
        R.stop_reason = S.stop;
        R.iterations_used = S.it;
        R.pending_flush = S.pend;
        R.final_relative_residual = S.rel;
        R.rhs_sq = S.q[0];
        R.r_sq = S.q[1];
        R.r_owned_sq = S.q[2];
        R.rglob_owned_sq = S.q[3];
        R.scale = S.scale;
        R.last_iterations = S.last_it;
        R.last_stop_reason = S.last_stop;
    }
    return BS_OK;
}

}  // extern "C"
