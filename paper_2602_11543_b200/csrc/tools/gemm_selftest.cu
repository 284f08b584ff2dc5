// Standalone check of the grouped tcgen05 GEMM against a naive FP32 kernel on the
// same bf16 inputs, plus a throughput probe. Developer tool (not the product path).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../grouped_gemm.cuh"
#include "../tmap.hpp"

using namespace spes_dev;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__global__ void ref_gemm(const __nv_bfloat16* A, const __nv_bfloat16* B, const GemmGroup* groups,
                         int ng, float* out, int BN, int lda) {
    // one thread per output element of every group (slow; test sizes only)
    int g = blockIdx.y;
    if (g >= ng) return;
    const GemmGroup gg = groups[g];
    int M = gg.m_tiles * 128, N = gg.n_tiles * BN;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < M * N;
         idx += gridDim.x * blockDim.x) {
        int m = idx / N, n = idx % N;
        float s = 0.f;
        // lda/ldb passed through ldo==K convention below
        for (int k = 0; k < gg.k_len; ++k)
            s += __bfloat162float(A[(int64_t)(gg.a_row0 + m) * lda + gg.k0 + k]) *
                 __bfloat162float(B[(int64_t)(gg.b_row0 + n) * lda + gg.bk0 + k]);
        out[(gg.out_row0 + m) * gg.ldo + n] = s;
    }
}

__global__ void fill_rand(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = __float2bfloat16(((x & 0xFFFF) / 65536.f - 0.5f));
    }
}

template <int BN>
int run_case(const char* name, int K_total, int a_rows, int b_rows, std::vector<GemmGroup> groups,
             int out_rows, int out_cols, bool timeit) {
    __nv_bfloat16 *A, *B;
    CK(cudaMalloc(&A, (size_t)a_rows * K_total * 2));
    CK(cudaMalloc(&B, (size_t)b_rows * K_total * 2));
    fill_rand<<<1024, 256>>>(A, (size_t)a_rows * K_total, 1234);
    fill_rand<<<1024, 256>>>(B, (size_t)b_rows * K_total, 777);
    float *out, *ref;
    CK(cudaMalloc(&out, (size_t)out_rows * out_cols * 4));
    CK(cudaMalloc(&ref, (size_t)out_rows * out_cols * 4));
    CK(cudaMemset(out, 0xFF, (size_t)out_rows * out_cols * 4));
    CK(cudaMemset(ref, 0, (size_t)out_rows * out_cols * 4));
    int tiles = 0;
    for (auto& g : groups) {
        g.tile_start = tiles;
        tiles += g.m_tiles * g.n_tiles;
        g.out0 = out;
        g.ldo = out_cols;
        g.bk0 = g.k0;
    }
    GemmGroup* dg;
    CK(cudaMalloc(&dg, groups.size() * sizeof(GemmGroup)));
    CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    int* dtiles;
    CK(cudaMalloc(&dtiles, 4));
    CK(cudaMemcpy(dtiles, &tiles, 4, cudaMemcpyHostToDevice));

    CUtensorMap ma = spes_host::make_tmap_bf16(A, a_rows, K_total, 128);
    CUtensorMap mb = spes_host::make_tmap_bf16(B, b_rows, K_total, BN);
    auto kern = grouped_gemm_kernel<BN, EpiStoreF32<BN>>;
    int smem = GemmCfg<BN>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = tiles < 148 ? tiles : 148;
    kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                       EpiStoreF32<BN>{});
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());

    std::vector<GemmGroup> rg = groups;
    for (auto& g : rg) g.out0 = ref;
    CK(cudaMemcpy(dg, rg.data(), rg.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    ref_gemm<<<dim3(256, groups.size()), 256>>>(A, B, dg, (int)groups.size(), ref, BN, K_total);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());

    std::vector<float> ho((size_t)out_rows * out_cols), hr((size_t)out_rows * out_cols);
    CK(cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), ref, hr.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    size_t bad = 0;
    for (auto& g : groups) {
        for (int m = 0; m < g.m_tiles * 128; ++m)
            for (int n = 0; n < g.n_tiles * BN; ++n) {
                size_t i = (size_t)(g.out_row0 + m) * out_cols + n;
                double e = fabs((double)ho[i] - hr[i]);
                if (!(e <= 1e-2 + 1e-3 * fabs(hr[i]))) ++bad;
                if (e > maxerr || e != e) maxerr = e;
                if (fabs(hr[i]) > maxref) maxref = fabs(hr[i]);
            }
    }
    printf("[%s] BN=%d tiles=%d max_abs_err=%.3e max_ref=%.3e bad=%zu -> %s\n", name, BN, tiles,
           maxerr, maxref, bad, bad == 0 ? "PASS" : "FAIL");
    if (timeit) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
        for (int i = 0; i < 3; ++i)
            kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                               EpiStoreF32<BN>{});
        cudaEventRecord(e0);
        const int iters = 20;
        for (int i = 0; i < iters; ++i)
            kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                               EpiStoreF32<BN>{});
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 0;
        for (auto& g : groups) flops += 2.0 * g.m_tiles * 128.0 * g.n_tiles * BN * g.k_len;
        printf("[%s] %.3f us/launch  %.1f TFLOP/s\n", name, ms * 1e3 / iters,
               flops / (ms / iters * 1e-3) / 1e12);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(out);
    cudaFree(ref);
    cudaFree(dg);
    cudaFree(dtiles);
    return bad == 0 ? 0 : 1;
}

// MN-major (weight-gradient) form: D[m][n] = sum_k A[k0+k][acol+m] * B[k0+k][bcol+n]
__global__ void ref_gemm_mn(const __nv_bfloat16* A, const __nv_bfloat16* B, const GemmGroup* groups,
                            int ng, float* out, int BN, int Mtot, int Ntot) {
    int g = blockIdx.y;
    if (g >= ng) return;
    const GemmGroup gg = groups[g];
    int M = gg.m_tiles * 128, N = gg.n_tiles * BN;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < M * N;
         idx += gridDim.x * blockDim.x) {
        int m = idx / N, n = idx % N;
        float s = 0.f;
        for (int k = 0; k < gg.k_len; ++k)
            s += __bfloat162float(A[(int64_t)(gg.k0 + k) * Mtot + gg.a_row0 + m]) *
                 __bfloat162float(B[(int64_t)(gg.k0 + k) * Ntot + gg.b_row0 + n]);
        out[(gg.out_row0 + m) * gg.ldo + n] = s;
    }
}

template <int BN>
int run_case_mn(const char* name, int K_total, int Mtot, int Ntot, std::vector<GemmGroup> groups,
                int out_rows, int out_cols, bool timeit) {
    __nv_bfloat16 *A, *B;
    CK(cudaMalloc(&A, (size_t)K_total * Mtot * 2));
    CK(cudaMalloc(&B, (size_t)K_total * Ntot * 2));
    fill_rand<<<1024, 256>>>(A, (size_t)K_total * Mtot, 99);
    fill_rand<<<1024, 256>>>(B, (size_t)K_total * Ntot, 4242);
    float *out, *ref;
    CK(cudaMalloc(&out, (size_t)out_rows * out_cols * 4));
    CK(cudaMalloc(&ref, (size_t)out_rows * out_cols * 4));
    CK(cudaMemset(out, 0xFF, (size_t)out_rows * out_cols * 4));
    CK(cudaMemset(ref, 0, (size_t)out_rows * out_cols * 4));
    int tiles = 0;
    for (auto& g : groups) {
        g.tile_start = tiles;
        tiles += g.m_tiles * g.n_tiles;
        g.out0 = out;
        g.ldo = out_cols;
        g.bk0 = g.k0;
    }
    GemmGroup* dg;
    CK(cudaMalloc(&dg, groups.size() * sizeof(GemmGroup)));
    CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    int* dtiles;
    CK(cudaMalloc(&dtiles, 4));
    CK(cudaMemcpy(dtiles, &tiles, 4, cudaMemcpyHostToDevice));
    CUtensorMap ma = spes_host::make_tmap_bf16(A, K_total, Mtot, 64);
    CUtensorMap mb = spes_host::make_tmap_bf16(B, K_total, Ntot, 64);
    auto kern = grouped_gemm_kernel<BN, EpiStoreF32<BN>, true, true>;
    int smem = GemmCfg<BN>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = tiles < 148 ? tiles : 148;
    kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                       EpiStoreF32<BN>{});
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<GemmGroup> rg = groups;
    for (auto& g : rg) g.out0 = ref;
    CK(cudaMemcpy(dg, rg.data(), rg.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    ref_gemm_mn<<<dim3(256, groups.size()), 256>>>(A, B, dg, (int)groups.size(), ref, BN, Mtot, Ntot);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> ho((size_t)out_rows * out_cols), hr((size_t)out_rows * out_cols);
    CK(cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), ref, hr.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    size_t bad = 0;
    for (auto& g : groups)
        for (int m = 0; m < g.m_tiles * 128; ++m)
            for (int n = 0; n < g.n_tiles * BN; ++n) {
                size_t i = (size_t)(g.out_row0 + m) * out_cols + n;
                double e = fabs((double)ho[i] - hr[i]);
                if (!(e <= 1e-2 + 1e-3 * fabs(hr[i]))) ++bad;
                if (e > maxerr || e != e) maxerr = e;
            }
    printf("[%s] MN BN=%d tiles=%d max_abs_err=%.3e bad=%zu -> %s\n", name, BN, tiles, maxerr, bad,
           bad == 0 ? "PASS" : "FAIL");
    if (timeit) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
        for (int i = 0; i < 3; ++i)
            kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                               EpiStoreF32<BN>{});
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i)
            kern<<<grid, GEMM_THREADS, smem>>>(ma, mb, dg, (int)groups.size(), dtiles, tiles,
                                               EpiStoreF32<BN>{});
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 0;
        for (auto& g : groups) flops += 2.0 * g.m_tiles * 128.0 * g.n_tiles * BN * g.k_len;
        printf("[%s] %.3f us/launch  %.1f TFLOP/s\n", name, ms * 1e3 / 20,
               flops / (ms / 20 * 1e-3) / 1e12);
    }
    cudaFree(A);
    cudaFree(B);
    cudaFree(out);
    cudaFree(ref);
    cudaFree(dg);
    cudaFree(dtiles);
    return bad == 0 ? 0 : 1;
}

static GemmGroup G(int a_row0, int b_row0, int k0, int k_len, int mt, int nt, int out_row0) {
    GemmGroup g{};
    g.a_row0 = a_row0;
    g.b_row0 = b_row0;
    g.k0 = k0;
    g.k_len = k_len;
    g.m_tiles = mt;
    g.n_tiles = nt;
    g.out_row0 = out_row0;
    return g;
}

int main() {
    int fails = 0;
    // single tile
    fails += run_case<128>("single", 64, 128, 128, {G(0, 0, 0, 64, 1, 1, 0)}, 128, 128, false);
    fails += run_case<256>("single256", 128, 128, 256, {G(0, 0, 0, 128, 1, 1, 0)}, 128, 256, false);
    // routed-style: 3 experts with 2,1,3 m-tiles, K=256, N=512 (two n tiles of 256)
    fails += run_case<256>("routed", 256, 6 * 128, 3 * 512,
                           {G(0, 0, 0, 256, 2, 2, 0), G(256, 512, 0, 256, 1, 2, 256),
                            G(384, 1024, 0, 256, 3, 2, 384)},
                           6 * 128, 512, false);
    // dW-style: K ranges differ per group, one empty
    fails += run_case<128>("dw", 1024, 256, 256,
                           {G(0, 0, 0, 384, 2, 2, 0), G(0, 0, 384, 0, 2, 2, 256),
                            G(0, 0, 384, 640, 2, 2, 512)},
                           768, 256, false);
    // throughput probe: cfg2 gate||up forward shape (16 experts x 2048 rows, N=2048, K=1024)
    {
        std::vector<GemmGroup> gs;
        for (int j = 0; j < 16; ++j) gs.push_back(G(j * 2048, j * 2048, 0, 1024, 16, 8, j * 2048));
        fails += run_case<256>("cfg2_fwd1", 1024, 16 * 2048, 16 * 2048, gs, 16 * 2048, 2048, true);
    }
    // MN-major (dW) form: tiny, offsets, empty K range, then the cfg2 dW gate||up shape
    fails += run_case_mn<128>("mn_single", 64, 128, 128, {G(0, 0, 0, 64, 1, 1, 0)}, 128, 128, false);
    fails += run_case_mn<256>("mn_groups", 1024, 256, 512,
                              {G(0, 0, 0, 384, 2, 2, 0), G(0, 0, 384, 0, 2, 2, 256),
                               G(128, 256, 384, 640, 1, 1, 512)},
                              640, 512, false);
    {
        std::vector<GemmGroup> gs;  // 16 owned experts, 2048 tokens each: [1024 x 2048] per expert
        for (int j = 0; j < 16; ++j) gs.push_back(G(0, 0, j * 2048, 2048, 8, 8, j * 1024));
        fails += run_case_mn<256>("cfg2_dw1", 16 * 2048, 1024, 2048, gs, 16 * 1024, 2048, true);
    }
    printf(fails ? "SELFTEST FAILED\n" : "SELFTEST OK\n");
    return fails;
}
