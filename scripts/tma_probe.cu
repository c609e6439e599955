// Bisect TMA usage on sm_100a: ./tma_probe <variant>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0: param map; 1: global map; bit 2: with fence.mbarrier_init; bit 3: skip sync fence
__global__ void probe(const __grid_constant__ CUtensorMap pmap, const CUtensorMap *gmap, double *out, int c0, int c1,
                      int c2, int nbytes) {
    __shared__ __align__(128) double buf[36 * 10];
    __shared__ __align__(8) uint64_t bar;
    const CUtensorMap *map = (MODE & 1) ? gmap : &pmap;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
        if (MODE & 4) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(nbytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su(buf)),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su(&bar))
            : "memory");
    }
    uint32_t ok = 0;
    for (long it = 0; it < (1L << 26) && !ok; ++it)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(su(&bar)), "r"(0)
            : "memory");
    for (int i = threadIdx.x; i < 360; i += blockDim.x) out[i] = ok ? buf[i] : -12345.0;
}

int main(int argc, char **argv) {
    int v = argc > 1 ? atoi(argv[1]) : 0;
    int nx = 40, ny = 20, nz = 3, pitch = 40;
    std::vector<double> h(pitch * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *out;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&out, 360 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t str[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * ny * 8};
    cuuint32_t box[3] = {36, 10, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d encode=%d\n", v, (int)r);
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    int c0 = (v & 8) ? -2 : 0, c1 = (v & 8) ? -1 : 0, c2 = (v & 16) ? -1 : 0;
    switch (v & 7) {
        case 0: probe<0><<<1, 128>>>(m, gm, out, c0, c1, c2, 2880); break;
        case 1: probe<1><<<1, 128>>>(m, gm, out, c0, c1, c2, 2880); break;
        case 4: probe<4><<<1, 128>>>(m, gm, out, c0, c1, c2, 2880); break;
        case 5: probe<5><<<1, 128>>>(m, gm, out, c0, c1, c2, 2880); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> ho(360);
    cudaMemcpy(ho.data(), out, 360 * 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %s; out[0..3]=%g %g %g %g out[37]=%g out[38]=%g\n", v, cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[3],
           ho[37], ho[38]);
    return 0;
}
