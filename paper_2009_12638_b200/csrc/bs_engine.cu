// bs_engine.cu — sm_100a engine for the block-Jacobi / CG 7-point stencil path.
//
// One translation unit: the matrix-free stencil sweep machinery, the fused CG
// phase machine with device-side stopping, halo packing, and the C ABI
// declared in include/blocksolve_b200.h.
//
// Reference algorithm (file:line into /root/reference/pkg/src/blocksolve):
//   SpMV            linalg.py:178-194 on the block system of problems.py:362-406
//   CG              inner_solvers.py:102-146 (scale = ||rhs||, 70-72)
//   rhs assembly    multisplit.py:333-338
//   local residual  multisplit.py:372-396, true residual 404-406
//   sync halo       comm.py:332-365 + merge multisplit.py:341-369 (overlap 0)
//
// Design:
//   * Every vector lives over the block's padded box, x-fastest.  A CTA owns a
//     TX x TY column tile and marches CZ planes in z: the stencil input field
//     u of plane k+1 is staged (tile + 1-cell x/y halo) into a 3-deep shared
//     ring while plane k is computed; z-neighbours ride in registers.
//   * The stencil input is produced on the fly: u = r + beta*p_old in CG
//     sweep 1 (so p is written once and never re-read in the same sweep),
//     u = p in sweep 2, u = x + alpha*p in residual sweeps (deferred x update).
//     => one CG iteration moves 64 B/point of compulsory HBM traffic.
//   * Reductions are fixed-order (per-thread z order, xor-butterfly warps,
//     sequential warps, strided+tree across CTAs) so results are deterministic
//     and independent of how many blocks share a GPU.
//   * The scalar recurrences (alpha, beta, stop tests) run in the last CTA of
//     every sweep launch ("last block" pattern), so the host only polls one
//     counter per batch of sweeps.
//   * All floating-point arithmetic is explicit round-to-nearest with no FMA
//     contraction (__dadd_rn/__dmul_rn, and -fmad=false) to reproduce the
//     reference's rounding: the SpMV is bit-identical.

#include "blocksolve_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
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

constexpr int TX = 32;
constexpr int TY = 8;
constexpr int NT = TX * TY;
constexpr int HX = TX + 2;
constexpr int HY = TY + 2;
constexpr int NHALO = 2 * TX + 2 * TY;
constexpr int NQ = 4;  // partial sums per CTA

enum Phase : int {
    PH_IDLE = 0,
    PH_INIT = 1,    // residual sweep that starts a CG solve
    PH_S1 = 2,      // p = r + beta p_old ; x += alpha_pend p_old ; p.Ap
    PH_S2 = 3,      // r -= alpha A p ; r.r
    PH_VERIFY = 4,  // true-residual check on claimed convergence
    PH_DONE = 5,
    PH_RESID = 6,   // standalone residual sweep (outer residual / checks)
};

enum Op : int { OP_RESID = 0, OP_S1 = 1, OP_S2 = 2, OP_APPLY = 3 };

struct DBlock {
    int gn[3];
    int lo[3], hi[3];        // owned box
    int plo[3], pdim[3];     // padded box
    int overlap;
    int cta_begin, cta_end;  // CTA range in sweep launches
    int tiles_x, tiles_y, tiles_z, cz;
    double *x, *r, *p[2];
    const double *b;
    double *ghost[BS_NDIR];
    double *hist;
    int hist_cap;
};

struct DState {
    int phase, stop, it, first, pend, pcur, max_its, basis;
    double tol, tol_eff, scale, rel, rr, alpha, beta, alpha_pend;
    double q[NQ];
};

// ------------------------------------------------------------------ geometry

__device__ __forceinline__ long long sidx(const DBlock &B, int i, int j, int k) {
    return (long long)(i - B.plo[0]) +
           (long long)B.pdim[0] * ((long long)(j - B.plo[1]) + (long long)B.pdim[1] * (long long)(k - B.plo[2]));
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
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

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

// ------------------------------------------------------------------ reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic CTA reduction of NQ values; result valid in thread 0.
__device__ __forceinline__ void cta_sum(double (&acc)[NQ], double (*red)[NT / 32]) {
    const int tid = threadIdx.y * TX + threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double v = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = v;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double s = red[q][0];
            for (int w = 1; w < NT / 32; ++w) s = add(s, red[q][w]);
            acc[q] = s;
        }
    }
}

// Sum of partials[begin:end) with a fixed strided + tree order (whole CTA).
__device__ double range_sum(const double *part, int begin, int end, double *scratch) {
    const int tid = threadIdx.y * TX + threadIdx.x;
    double s = 0.0;
    for (int c = begin + tid; c < end; c += NT) s = add(s, __ldcg(part + c));
    scratch[tid] = s;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
        if (tid < w) scratch[tid] = add(scratch[tid], scratch[tid + w]);
        __syncthreads();
    }
    double out = scratch[0];
    __syncthreads();
    return out;
}

// ------------------------------------------------------------------ sweep

struct SweepCtx {
    const DBlock *B;
    int op;
    bool pend, first, want_global;
    double alpha_pend, beta, alpha;
    const double *pin;  // p[pcur]
    double *pout;       // p[1-pcur]
    const double *xin;  // OP_APPLY input
    double *yout;       // OP_APPLY output
};

// Stencil input field at storage index s of an in-region point.
template <int OP>
__device__ __forceinline__ double field(const SweepCtx &C, long long s) {
    const DBlock &B = *C.B;
    switch (OP) {
        case OP_RESID: {
            double v = B.x[s];
            return C.pend ? add(v, mul(C.alpha_pend, C.pin[s])) : v;
        }
        case OP_S1: {
            double v = B.r[s];
            return C.first ? v : add(v, mul(C.beta, C.pin[s]));
        }
        case OP_S2:
            return C.pin[s];
        default:
            return C.xin[s];
    }
}

template <int OP>
__device__ __forceinline__ double field_at(const SweepCtx &C, int i, int j, int k) {
    return in_region(*C.B, i, j, k) ? field<OP>(C, sidx(*C.B, i, j, k)) : 0.0;
}

// Process one tile: accumulate partial sums into acc.
template <int OP>
__device__ void sweep_tile(const SweepCtx &C, int tile, double (*sm)[HY][HX], double (&acc)[NQ]) {
    const DBlock &B = *C.B;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    int t = tile;
    const int ix = t % B.tiles_x;
    t /= B.tiles_x;
    const int iy = t % B.tiles_y;
    const int iz = t / B.tiles_y;
    const int x0 = B.plo[0] + ix * TX, y0 = B.plo[1] + iy * TY;
    const int z0 = B.plo[2] + iz * B.cz;
    const int z1 = min(z0 + B.cz, B.plo[2] + B.pdim[2]);
    const int gi = x0 + tx, gj = y0 + ty;
    const bool col_in = gi < B.plo[0] + B.pdim[0] && gj < B.plo[1] + B.pdim[1];

    int hci = 0, hcj = 0;
    const bool has_halo = tid < NHALO;
    if (tid < TX) {
        hci = tid;
        hcj = -1;
    } else if (tid < 2 * TX) {
        hci = tid - TX;
        hcj = TY;
    } else if (tid < 2 * TX + TY) {
        hci = -1;
        hcj = tid - 2 * TX;
    } else {
        hci = TX;
        hcj = tid - 2 * TX - TY;
    }

    double u_prev = col_in ? field_at<OP>(C, gi, gj, z0 - 1) : 0.0;
    int bc = 0;
    double u_cur = col_in ? field_at<OP>(C, gi, gj, z0) : 0.0;
    sm[bc][ty + 1][tx + 1] = u_cur;
    if (has_halo) sm[bc][hcj + 1][hci + 1] = field_at<OP>(C, x0 + hci, y0 + hcj, z0);

    for (int k = z0; k < z1; ++k) {
        const int bn = bc == 2 ? 0 : bc + 1;
        const double u_next = col_in ? field_at<OP>(C, gi, gj, k + 1) : 0.0;
        sm[bn][ty + 1][tx + 1] = u_next;
        if (has_halo) sm[bn][hcj + 1][hci + 1] = field_at<OP>(C, x0 + hci, y0 + hcj, k + 1);
        __syncthreads();
        if (col_in && in_region(B, gi, gj, k)) {
            const double xm = sm[bc][ty + 1][tx], xp = sm[bc][ty + 1][tx + 2];
            const double ym = sm[bc][ty][tx + 1], yp = sm[bc][ty + 2][tx + 1];
            const bool pz = in_region(B, gi, gj, k - 1);
            const bool py = in_region(B, gi, gj - 1, k);
            const bool px = in_region(B, gi - 1, gj, k);
            const double au = stencil7(u_prev, ym, xm, u_cur, xp, yp, u_next, pz, py, px);
            const long long s = sidx(B, gi, gj, k);
            if (OP == OP_APPLY) {
                C.yout[s] = au;
            } else if (OP == OP_S2) {
                const double rn = sub(B.r[s], mul(C.alpha, au));
                B.r[s] = rn;
                acc[0] = add(acc[0], mul(rn, rn));
            } else if (OP == OP_S1) {
                C.pout[s] = u_cur;
                if (C.pend) B.x[s] = add(B.x[s], mul(C.alpha_pend, C.pin[s]));
                acc[0] = add(acc[0], mul(u_cur, au));
            } else {  // OP_RESID: r = (b - C*halo) - A_ii u
                const double bv = B.b[s];
                // neighbours in ascending column order
                const int ni[6] = {gi, gi, gi - 1, gi + 1, gi, gi};
                const int nj[6] = {gj, gj - 1, gj, gj, gj + 1, gj};
                const int nk[6] = {k - 1, k, k, k, k, k + 1};
                // coupling row sum C*halo (multisplit.py:333-338): entries of
                // -1 in ascending column order, reduceat rule first + seq(rest)
                double first = 0.0, rest = 0.0;
                int cnt = 0;
#pragma unroll
                for (int d = 0; d < 6; ++d) {
                    if (in_grid(B, ni[d], nj[d], nk[d]) && !in_region(B, ni[d], nj[d], nk[d])) {
                        const double term = -ghost_at(B, ni[d], nj[d], nk[d], d);
                        if (cnt == 0) first = term;
                        else if (cnt == 1) rest = term;
                        else rest = add(rest, term);
                        ++cnt;
                    }
                }
                const double rhs = cnt == 0 ? bv : sub(bv, cnt == 1 ? first : add(first, rest));
                const double rv = sub(rhs, au);
                B.r[s] = rv;
                acc[0] = add(acc[0], mul(rhs, rhs));
                const double r2 = mul(rv, rv);
                acc[1] = add(acc[1], r2);
                if (in_owned(B, gi, gj, k)) {
                    acc[2] = add(acc[2], r2);
                    if (C.want_global) {
                        // global operator row (residual_norms on the gathered
                        // iterate): couplings enter the stencil as present terms
                        double v[6] = {u_prev, ym, xm, xp, yp, u_next};
                        bool pg[6];
#pragma unroll
                        for (int d = 0; d < 6; ++d) {
                            pg[d] = in_grid(B, ni[d], nj[d], nk[d]);
                            if (pg[d] && !in_region(B, ni[d], nj[d], nk[d]))
                                v[d] = ghost_at(B, ni[d], nj[d], nk[d], d);
                        }
                        const double ag =
                            stencil7(v[0], v[1], v[2], u_cur, v[3], v[4], v[5], pg[0], pg[1], pg[2]);
                        const double rg = sub(bv, ag);
                        acc[3] = add(acc[3], mul(rg, rg));
                    }
                }
            }
        }
        u_prev = u_cur;
        u_cur = u_next;
        bc = bn;
    }
    __syncthreads();  // ring reuse by the next tile of this CTA (none today)
}

// ------------------------------------------------------------------ scalars

__device__ void transition(const DBlock &B, DState &S, int ph, const double *q) {
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
            if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel;
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
                if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel_true;
                S.stop = BS_STOP_TOLERANCE_MET;
                S.phase = PH_DONE;
            } else {
                const double rr_new = q[1];  // r = r_true
                const double rel = sqrt(rr_new) / S.scale;
                S.rel = rel;
                if (S.it - 1 < B.hist_cap) B.hist[S.it - 1] = rel;
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
        case PH_RESID: {
            for (int i = 0; i < NQ; ++i) S.q[i] = q[i];
            S.phase = PH_DONE;
            break;
        }
        default:
            break;
    }
}


// Which phases a sweep kernel of op OPK serves.
template <int OPK>
__device__ __forceinline__ bool serves(int ph) {
    if (OPK == OP_S1) return ph == PH_S1;
    if (OPK == OP_S2) return ph == PH_S2;
    return ph == PH_INIT || ph == PH_VERIFY || ph == PH_RESID;
}

// One sweep over every block whose phase this kernel serves; the last CTA
// to finish runs the scalar recurrences of those blocks.  Launched as the
// cycle RESID -> S1 -> S2, each block advances through its own phase machine
// (a block in S1 at the start of a cycle completes one CG iteration).
template <int OPK>
__global__ void __launch_bounds__(NT) k_sweep(const DBlock *__restrict__ blocks, DState *states,
                                              const int *__restrict__ cta_block, int nblocks, int nctas,
                                              double *partials, unsigned *counter, int *n_active,
                                              int want_global) {
    __shared__ double sm[3][HY][HX];
    __shared__ double red[NQ][NT / 32];
    __shared__ double scratch[NT];
    __shared__ bool am_last;
    const int tid = threadIdx.y * TX + threadIdx.x;
    const int b = cta_block[blockIdx.x];
    const DBlock &B = blocks[b];
    const int ph = states[b].phase;

    double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
    if (serves<OPK>(ph)) {
        const DState S = states[b];
        SweepCtx C;
        C.B = &B;
        C.op = OPK;
        C.pend = S.pend != 0;
        C.first = S.first != 0;
        C.want_global = want_global != 0;
        C.alpha_pend = S.alpha_pend;
        C.alpha = S.alpha;
        C.beta = S.beta;
        C.pin = B.p[S.pcur];
        C.pout = B.p[S.pcur ^ 1];
        C.xin = nullptr;
        C.yout = nullptr;
        sweep_tile<OPK>(C, blockIdx.x - B.cta_begin, sm, acc);
    }
    cta_sum(acc, red);
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) partials[(size_t)q * nctas + blockIdx.x] = acc[q];
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        am_last = (prev == (unsigned)nctas - 1u);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    int active = 0;
    for (int bb = 0; bb < nblocks; ++bb) {
        const int phb = states[bb].phase;
        if (serves<OPK>(phb)) {
            const DBlock &BB = blocks[bb];
            double q[NQ];
            const int nq = (OPK == OP_RESID) ? NQ : 1;
            for (int i = 0; i < NQ; ++i)
                q[i] = i < nq ? range_sum(partials + (size_t)i * nctas, BB.cta_begin, BB.cta_end, scratch) : 0.0;
            if (tid == 0) {
                DState S = states[bb];
                transition(BB, S, phb, q);
                states[bb] = S;
            }
            __syncthreads();
        }
        if (tid == 0) {
            const int p2 = states[bb].phase;
            if (p2 != PH_DONE && p2 != PH_IDLE) ++active;
        }
    }
    if (tid == 0) {
        *n_active = active;
        *counter = 0u;
    }
}

// y = A_ii x on one block (standalone a1).
__global__ void __launch_bounds__(NT) k_apply(const DBlock *__restrict__ blocks, int b, const double *x,
                                              double *y) {
    __shared__ double sm[3][HY][HX];
    const DBlock &B = blocks[b];
    SweepCtx C;
    C.B = &B;
    C.op = OP_APPLY;
    C.pend = C.first = C.want_global = false;
    C.alpha_pend = C.alpha = C.beta = 0.0;
    C.pin = nullptr;
    C.pout = nullptr;
    C.xin = x;
    C.yout = y;
    double acc[NQ] = {0.0, 0.0, 0.0, 0.0};
    sweep_tile<OP_APPLY>(C, blockIdx.x, sm, acc);
}

// Arm solves / residual sweeps.
__global__ void k_arm(DState *states, const int *active, int nblocks, int phase, int max_its, double tol,
                      int basis) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    if (active && !active[b]) return;
    DState &S = states[b];
    S.phase = phase;
    if (phase == PH_INIT) {
        S.stop = BS_STOP_NONE;
        S.it = 0;
        S.first = 1;
        S.max_its = max_its;
        S.tol = tol;
        S.basis = basis;
    }
}

// Deferred x += alpha p over every region point of blocks with a pending update.
__global__ void k_flush(const DBlock *__restrict__ blocks, const DState *states, int nblocks) {
    const int b = blockIdx.y;
    const DBlock &B = blocks[b];
    const DState &S = states[b];
    if (!S.pend) return;
    const long long n = (long long)B.pdim[0] * B.pdim[1] * B.pdim[2];
    const double a = S.alpha_pend;
    const double *p = B.p[S.pcur];
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (long long)gridDim.x * blockDim.x) {
        const int i = B.plo[0] + (int)(s % B.pdim[0]);
        const long long t = s / B.pdim[0];
        const int j = B.plo[1] + (int)(t % B.pdim[1]);
        const int k = B.plo[2] + (int)(t / B.pdim[1]);
        if (B.overlap == 0 || in_region(B, i, j, k)) B.x[s] = add(B.x[s], mul(a, p[s]));
    }
}

__global__ void k_clear_pend(DState *states, int nblocks) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nblocks) states[b].pend = 0;
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
    const long long n = (long long)nu * nv;
    const double a = SS.alpha_pend;
    const bool pend = SS.pend != 0;
    const double *p = S.p[SS.pcur];
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (long long)gridDim.x * blockDim.x) {
        const int u = (int)(c % nu), v = (int)(c / nu);
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
        const double xv = S.x[s];
        D.ghost[dir][c] = pend ? add(xv, mul(a, p[s])) : xv;
    }
}

}  // namespace

// ====================================================================== C ABI

static unsigned long long g_launches = 0;  // kernels launched by this library

struct bs_ctx {
    int device = 0;
    // optional CUDA-event timing of the S1 / S2 / RESID sweep kernels in bs_run
    bool timing = false;
    std::vector<cudaEvent_t> ev;   // pairs, reused across batches
    double op_ms[3] = {0.0, 0.0, 0.0};
    long long op_n[3] = {0, 0, 0};
    int nblocks = 0;
    int nctas = 0;
    std::vector<DBlock> hblocks;
    DBlock *dblocks = nullptr;
    DState *dstates = nullptr;
    int *dcta_block = nullptr;
    double *dpartials = nullptr;
    unsigned *dcounter = nullptr;
    int *dnactive = nullptr;
    int *dactive = nullptr;
    int *dplan = nullptr;
    int plan_cap = 0;
    int *hpinned = nullptr;  // [0]: n_active, [1..]: active mask staging
    DState *hstates = nullptr;
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
    std::memcpy(c->hpinned + 1, active, sizeof(int) * c->nblocks);
    BS_CU(cudaMemcpyAsync(c->dactive, c->hpinned + 1, sizeof(int) * c->nblocks, cudaMemcpyHostToDevice, st));
    *dptr = c->dactive;
    return BS_OK;
}

template <int OPK>
static void launch_sweep(bs_ctx *c, cudaStream_t st, int slot) {
    if (c->timing) cudaEventRecord(c->ev[2 * slot], st);
    k_sweep<OPK><<<c->nctas, dim3(TX, TY), 0, st>>>(c->dblocks, c->dstates, c->dcta_block, c->nblocks, c->nctas,
                                                    c->dpartials, c->dcounter, c->dnactive, 1);
    if (c->timing) cudaEventRecord(c->ev[2 * slot + 1], st);
    ++g_launches;
}

static void launch_cycle(bs_ctx *c, cudaStream_t st, int cycle) {
    launch_sweep<OP_RESID>(c, st, 3 * cycle + 0);
    launch_sweep<OP_S1>(c, st, 3 * cycle + 1);
    launch_sweep<OP_S2>(c, st, 3 * cycle + 2);
}

// After the batch's stream sync: fold the recorded event pairs into the totals.
static void harvest_timing(bs_ctx *c, int cycles) {
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

}  // namespace

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

const char *bs_last_error(void) { return g_err.c_str(); }

int bs_ctx_create(int device, int nblocks, const bs_block_desc *blocks, int z_chunk, bs_ctx **out) {
    if (!out || !blocks || nblocks < 1) return fail(BS_EINVAL, "bs_ctx_create: bad arguments");
    bs_ctx *c = new bs_ctx();
    c->device = device;
    c->nblocks = nblocks;
    if (int e = set_dev(c)) {
        delete c;
        return e;
    }
    std::vector<int> cta_block;
    for (int b = 0; b < nblocks; ++b) {
        const bs_block_desc &d = blocks[b];
        DBlock B;
        std::memset(&B, 0, sizeof(B));
        for (int a = 0; a < 3; ++a) {
            B.gn[a] = d.global_dims[a];
            B.lo[a] = d.owned_lo[a];
            B.hi[a] = d.owned_hi[a];
            if (B.gn[a] < 1 || B.lo[a] < 0 || B.hi[a] > B.gn[a] || B.lo[a] >= B.hi[a]) {
                delete c;
                return fail(BS_EINVAL, "bs_ctx_create: block " + std::to_string(b) + " has an empty or out-of-grid owned box");
            }
            B.plo[a] = std::max(0, B.lo[a] - d.overlap);
            B.pdim[a] = std::min(B.gn[a], B.hi[a] + d.overlap) - B.plo[a];
        }
        if (d.overlap < 0) {
            delete c;
            return fail(BS_EINVAL, "bs_ctx_create: overlap must be non-negative");
        }
        B.overlap = d.overlap;
        B.x = d.x;
        B.r = d.r;
        B.p[0] = d.p0;
        B.p[1] = d.p1;
        B.b = d.b;
        for (int q = 0; q < BS_NDIR; ++q) B.ghost[q] = d.ghost[q];
        B.hist = d.history;
        B.hist_cap = d.history_cap;
        if (!B.x || !B.r || !B.p[0] || !B.p[1] || !B.b) {
            delete c;
            return fail(BS_EINVAL, "bs_ctx_create: null vector pointer for block " + std::to_string(b));
        }
        B.tiles_x = (B.pdim[0] + TX - 1) / TX;
        B.tiles_y = (B.pdim[1] + TY - 1) / TY;
        int cz = z_chunk;
        if (cz <= 0) {
            // aim for >= ~16 resident CTAs' worth of work per SM without
            // chopping z into slivers (each chunk re-stages 2 planes)
            const long long cols = (long long)B.tiles_x * B.tiles_y * nblocks;
            const long long want = 148LL * 12;
            long long chunks = (want + cols - 1) / cols;
            cz = (int)std::max<long long>(16, (B.pdim[2] + chunks - 1) / chunks);
        }
        B.cz = std::min(cz, B.pdim[2]);
        B.tiles_z = (B.pdim[2] + B.cz - 1) / B.cz;
        B.cta_begin = (int)cta_block.size();
        const long long ntile = (long long)B.tiles_x * B.tiles_y * B.tiles_z;
        for (long long t = 0; t < ntile; ++t) cta_block.push_back(b);
        B.cta_end = (int)cta_block.size();
        c->hblocks.push_back(B);
    }
    c->nctas = (int)cta_block.size();
    cudaError_t e = cudaSuccess;
    e = cudaMalloc(&c->dblocks, sizeof(DBlock) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dstates, sizeof(DState) * nblocks);
    if (e == cudaSuccess) e = cudaMalloc(&c->dcta_block, sizeof(int) * c->nctas);
    if (e == cudaSuccess) e = cudaMalloc(&c->dpartials, sizeof(double) * NQ * c->nctas);
    if (e == cudaSuccess) e = cudaMalloc(&c->dcounter, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&c->dnactive, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->dactive, sizeof(int) * nblocks);
    if (e == cudaSuccess) e = cudaHostAlloc(&c->hpinned, sizeof(int) * (nblocks + 1), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&c->hstates, sizeof(DState) * nblocks, cudaHostAllocDefault);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dblocks, c->hblocks.data(), sizeof(DBlock) * nblocks, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(c->dcta_block, cta_block.data(), sizeof(int) * c->nctas, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(c->dstates, 0, sizeof(DState) * nblocks);
    if (e == cudaSuccess) e = cudaMemset(c->dcounter, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(c->dnactive, 0, sizeof(int));
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
    cudaFree(c->dblocks);
    cudaFree(c->dstates);
    cudaFree(c->dcta_block);
    cudaFree(c->dpartials);
    cudaFree(c->dcounter);
    cudaFree(c->dnactive);
    cudaFree(c->dactive);
    cudaFree(c->dplan);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->hpinned) cudaFreeHost(c->hpinned);
    if (c->hstates) cudaFreeHost(c->hstates);
    delete c;
    return BS_OK;
}

int bs_ctx_num_ctas(const bs_ctx *c) { return c ? c->nctas : 0; }

unsigned long long bs_launch_count(void) { return g_launches; }

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
    if (int e = set_dev(c)) return e;
    const DBlock &B = c->hblocks[block];
    ++g_launches;
    k_apply<<<B.cta_end - B.cta_begin, dim3(TX, TY), 0, (cudaStream_t)stream>>>(c->dblocks, block, x, y);
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
    ++g_launches;
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dstates, dact, c->nblocks, PH_INIT, max_iterations,
                                                   tolerance, basis);
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
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dstates, dact, c->nblocks, PH_RESID, 0, 0.0, 0);
    ++g_launches;
    k_sweep<OP_RESID><<<c->nctas, dim3(TX, TY), 0, st>>>(c->dblocks, c->dstates, c->dcta_block, c->nblocks,
                                                         c->nctas, c->dpartials, c->dcounter, c->dnactive, 1);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_sweep_resid(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_sweep_resid: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    launch_sweep<OP_RESID>(c, st, 0);
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
    k_arm<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dstates, dact, c->nblocks, PH_DONE, 0, 0.0, 0);
    BS_CU(cudaGetLastError());
    return BS_OK;
}

int bs_run(bs_ctx *c, int batch, int max_launches, void *stream, int64_t *sweeps_out) {
    if (!c) return fail(BS_EINVAL, "bs_run: null context");
    if (batch < 1) batch = 1;
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t launched = 0;
    for (;;) {
        if (c->timing && (int)c->ev.size() < 6 * batch) {
            for (int i = (int)c->ev.size(); i < 6 * batch; ++i) {
                cudaEvent_t e;
                BS_CU(cudaEventCreate(&e));
                c->ev.push_back(e);
            }
        }
        for (int i = 0; i < batch; ++i) launch_cycle(c, st, i);
        launched += 3LL * batch;
        BS_CU(cudaGetLastError());
        BS_CU(cudaMemcpyAsync(c->hpinned, c->dnactive, sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_CU(cudaStreamSynchronize(st));
        if (c->timing) harvest_timing(c, batch);
        if (c->hpinned[0] == 0) break;
        if (max_launches > 0 && launched >= max_launches) {
            if (sweeps_out) *sweeps_out = launched;
            return fail(BS_ESTATE, "bs_run: solves still active after max_launches sweeps");
        }
    }
    if (sweeps_out) *sweeps_out = launched;
    return BS_OK;
}

int bs_flush(bs_ctx *c, void *stream) {
    if (!c) return fail(BS_EINVAL, "bs_flush: null context");
    if (int e = set_dev(c)) return e;
    cudaStream_t st = (cudaStream_t)stream;
    ++g_launches;
    k_flush<<<dim3(592, c->nblocks), 256, 0, st>>>(c->dblocks, c->dstates, c->nblocks);
    ++g_launches;
    k_clear_pend<<<(c->nblocks + 127) / 128, 128, 0, st>>>(c->dstates, c->nblocks);
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
    }
    BS_CU(cudaMemcpyAsync(c->dplan, plan, sizeof(int) * 3 * nplan, cudaMemcpyHostToDevice, st));
    ++g_launches;
    k_halo_pack<<<dim3(64, nplan), 256, 0, st>>>(c->dblocks, c->dstates, c->dplan);
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
    }
    return BS_OK;
}

}  // extern "C"
