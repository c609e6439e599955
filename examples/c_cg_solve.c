/* Minimal non-Python host of the C ABI (include/blocksolve_b200.h): one CG
 * solve of the 7-point Laplacian on an n^3 grid with the seeded rhs of
 * SURVEY §8(d), exactly what blocksolve's cg_solve(A, b, 0, spec) computes
 * (inner_solvers.py:102-146).
 *
 *   gcc -O2 -I include examples/c_cg_solve.c -o c_cg_solve \
 *       -L paper_2009_12638_b200/_lib -lbsgpu -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2009_12638_b200/_lib -Wl,-rpath,/usr/local/cuda/lib64
 *   ./c_cg_solve 64        # prints "its=231 stop=1 rel=..."
 *
 * With no GPU it still exercises the error path: "error: ..." and exit 2. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "blocksolve_b200.h"

static int die(const char *what) {
    fprintf(stderr, "error: %s: %s\n", what, bs_last_error());
    return 2;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 64;
    if (bs_abi_version() != BS_ABI_VERSION) return die("abi");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        /* argument validation works without a device */
        if (bs_ctx_create(0, 0, NULL, 0, NULL) != BS_EINVAL) return 3;
        fprintf(stderr, "error: no CUDA device (%s)\n", bs_last_error());
        return 2;
    }
    const int pitch = (n + 3) / 4 * 4;
    const size_t cells = (size_t)pitch * n * n, bytes = cells * sizeof(double);
    double *x, *r, *p0, *p1, *b, *flat, *hist;
    if (cudaMalloc((void **)&x, bytes) || cudaMalloc((void **)&r, bytes) || cudaMalloc((void **)&p0, bytes) ||
        cudaMalloc((void **)&p1, bytes) || cudaMalloc((void **)&b, bytes) ||
        cudaMalloc((void **)&flat, (size_t)n * n * n * sizeof(double)) ||
        cudaMalloc((void **)&hist, 4096 * sizeof(double)))
        return die("cudaMalloc");
    cudaMemset(x, 0, bytes);
    cudaMemset(r, 0, bytes);
    cudaMemset(p0, 0, bytes);
    cudaMemset(p1, 0, bytes);
    cudaMemset(b, 0, bytes);
    /* numpy.random.default_rng(0).bit_generator.state after seeding */
    const unsigned long long s_hi = 0x1aa1b5345996452dULL, s_lo = 0x09585eb7a69561e3ULL;
    const unsigned long long i_hi = 0x418ddadb3af71a82ULL, i_lo = 0x588133bc447873a9ULL;
    if (bs_uniform_pcg64(flat, (int64_t)n * n * n, s_hi, s_lo, i_hi, i_lo, -1.0, 1.0, NULL)) return die("rhs");
    /* x-fastest rows -> pitched rows */
    if (cudaMemcpy2D(b, pitch * sizeof(double), flat, n * sizeof(double), n * sizeof(double), (size_t)n * n,
                     cudaMemcpyDeviceToDevice))
        return die("cudaMemcpy2D");
    bs_block_desc d;
    memset(&d, 0, sizeof(d));
    d.global_dims[0] = d.global_dims[1] = d.global_dims[2] = n;
    d.owned_hi[0] = d.owned_hi[1] = d.owned_hi[2] = n;
    d.x = x;
    d.r = r;
    d.p0 = p0;
    d.p1 = p1;
    d.b = b;
    d.history = hist;
    d.history_cap = 4096;
    bs_ctx *ctx = NULL;
    if (bs_ctx_create(0, 1, &d, 0, &ctx)) return die("bs_ctx_create");
    if (bs_cg_begin(ctx, 4096, 1e-8, BS_BASIS_RHS, NULL, NULL)) return die("bs_cg_begin");
    if (bs_run(ctx, 8, 0, NULL, NULL)) return die("bs_run");
    if (bs_flush(ctx, NULL)) return die("bs_flush");
    bs_block_report rep;
    if (bs_read_reports(ctx, &rep, NULL)) return die("bs_read_reports");
    printf("its=%d stop=%d rel=%.17g\n", rep.iterations_used, rep.stop_reason, rep.final_relative_residual);
    bs_ctx_destroy(ctx);
    return rep.stop_reason == BS_STOP_TOLERANCE_MET ? 0 : 1;
}
