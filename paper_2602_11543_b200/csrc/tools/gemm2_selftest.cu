// Standalone check + throughput probe of the 2-CTA (cta_group::2) grouped GEMM for all
// operand-major combinations used by the library. Developer tool.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../grouped_gemm_2cta.cuh"
#include "../tmap.hpp"

using namespace spes_dev;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

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

// A: K-major [arows x K] (a[row*lda + k]) or MN-major [K x Mtot] (a[k*lda + col])
__global__ void ref_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, const GemmGroup* gs,
                           int ng, float* out, int BN, int lda, int ldb, int a_mn, int b_mn) {
    int g = blockIdx.y;
    if (g >= ng) return;
    const GemmGroup gg = gs[g];
    int M = gg.m_tiles * 256, N = gg.n_tiles * BN;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < M * N;
         idx += gridDim.x * blockDim.x) {
        int m = idx / N, n = idx % N;
        float s = 0.f;
        for (int k = 0; k < gg.k_len; ++k) {
            float a = a_mn ? __bfloat162float(A[(int64_t)(gg.k0 + k) * lda + gg.a_row0 + m])
                           : __bfloat162float(A[(int64_t)(gg.a_row0 + m) * lda + gg.k0 + k]);
            float b = b_mn ? __bfloat162float(B[(int64_t)(gg.bk0 + k) * ldb + gg.b_row0 + n])
                           : __bfloat162float(B[(int64_t)(gg.b_row0 + n) * ldb + gg.bk0 + k]);
            s += a * b;
        }
        out[(gg.out_row0 + m) * gg.ldo + n] = s;
    }
}

template <int BN, bool AMN, bool BMN>
int run(const char* name, int a_rows, int a_cols, int b_rows, int b_cols,
        std::vector<GemmGroup> groups, int out_rows, int out_cols, bool timeit) {
    __nv_bfloat16 *A, *B;
    CK(cudaMalloc(&A, (size_t)a_rows * a_cols * 2));
    CK(cudaMalloc(&B, (size_t)b_rows * b_cols * 2));
    fill_rand<<<1024, 256>>>(A, (size_t)a_rows * a_cols, 321);
    fill_rand<<<1024, 256>>>(B, (size_t)b_rows * b_cols, 654);
    float *out, *ref;
    CK(cudaMalloc(&out, (size_t)out_rows * out_cols * 4));
    CK(cudaMalloc(&ref, (size_t)out_rows * out_cols * 4));
    CK(cudaMemset(out, 0xFF, (size_t)out_rows * out_cols * 4));
    int tiles = 0;
    for (auto& g : groups) {
        g.tile_start = tiles;
        tiles += g.m_tiles * g.n_tiles;
        g.out0 = out;
        g.ldo = out_cols;
    }
    GemmGroup* dg;
    CK(cudaMalloc(&dg, groups.size() * sizeof(GemmGroup)));
    CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    int* dtiles;
    CK(cudaMalloc(&dtiles, 4));
    CK(cudaMemcpy(dtiles, &tiles, 4, cudaMemcpyHostToDevice));
    CUtensorMap ma = spes_host::make_tmap_bf16(A, a_rows, a_cols, AMN ? 64 : 128);
    CUtensorMap mb = spes_host::make_tmap_bf16(B, b_rows, b_cols, BMN ? 64 : BN / 2);
    auto kern = grouped_gemm_2cta_kernel<BN, EpiStoreF32<BN>, AMN, BMN>;
    const int smem = Gemm2Cfg<BN>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int pairs = tiles < 74 ? tiles : 74;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GemmGroup* dgc = dg;
    const int* dtc = dtiles;
    int ng = (int)groups.size();
    CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dgc, ng, dtc, tiles,
                          EpiStoreF32<BN>{}));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<GemmGroup> rg = groups;
    for (auto& g : rg) g.out0 = ref;
    CK(cudaMemcpy(dg, rg.data(), rg.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    ref_kernel<<<dim3(512, groups.size()), 256>>>(A, B, dg, ng, ref, BN, a_cols, b_cols, AMN, BMN);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> ho((size_t)out_rows * out_cols), hr((size_t)out_rows * out_cols);
    CK(cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), ref, hr.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    size_t bad = 0;
    for (auto& g : groups)
        for (int m = 0; m < g.m_tiles * 256; ++m)
            for (int n = 0; n < g.n_tiles * BN; ++n) {
                size_t i = (size_t)(g.out_row0 + m) * out_cols + n;
                double e = fabs((double)ho[i] - hr[i]);
                if (!(e <= 1e-2 + 1e-3 * fabs(hr[i]))) ++bad;
                if (e > maxerr || e != e) maxerr = e;
            }
    printf("[%s] 2CTA BN=%d A_MN=%d B_MN=%d tiles=%d max_abs_err=%.3e bad=%zu -> %s\n", name, BN,
           (int)AMN, (int)BMN, tiles, maxerr, bad, bad == 0 ? "PASS" : "FAIL");
    if (timeit && bad == 0) {
        CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int i = 0; i < 3; ++i)
            CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dgc, ng, dtc, tiles,
                                  EpiStoreF32<BN>{}));
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i)
            CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dgc, ng, dtc, tiles,
                                  EpiStoreF32<BN>{}));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 0;
        for (auto& g : groups) flops += 2.0 * g.m_tiles * 256.0 * g.n_tiles * BN * g.k_len;
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

struct EpiNull {
    static constexpr int SLOTS = 1;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup&, int, int, int, uint32_t, bool, int, EpiOut&) const {}
};

// epilogue cost decomposition probes (fp32 tile of 128 x 256 per CTA)
struct EpiTmemOnly {  // TMEM -> registers only (results kept alive via an impossible store)
    static constexpr int SLOTS = 1;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int, int, int r, uint32_t taddr, bool empty,
                               int half, EpiOut&) const {
        float acc = 0.f;
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += v[i];
        }
        if (acc == 1234.5f && r == 999) static_cast<float*>(g.out0)[0] = acc;
    }
};
struct EpiTmemSmem {  // TMEM -> registers -> smem slot (no global stores)
    static constexpr int SLOTS = 1;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup&, int, int, int, uint32_t taddr, bool empty,
                               int half, EpiOut& out) const {
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
            uint4* row = out.my_row(0);
#pragma unroll
            for (int i = 0; i < 8; ++i) row[i] = reinterpret_cast<const uint4*>(v)[i];
            __syncwarp();
        }
    }
};

// TMA-store epilogue probe: each warp writes its 32 x 32 fp32 piece into a 128B-swizzled
// 4 KiB box and one lane issues cp.async.bulk.tensor.2d (global <- shared), double-buffered
__device__ CUtensorMap g_out_map;
__device__ float* g_out_ptr;
struct EpiTmaF32 {
    static constexpr int SLOTS = 2;
    __device__ void prefetch(const GemmGroup&, int, int, int, int) const {}
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr, bool empty,
                               int half, EpiOut& out) const {
        const int lane = out.lane;
        uint8_t* base = reinterpret_cast<uint8_t*>(
            (reinterpret_cast<uintptr_t>(out.base) + 1023) & ~static_cast<uintptr_t>(1023));
        const int row0 = static_cast<int>(g.out_row0) + mt * 128 + (r - lane);
        int slot = 0;
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
            uint8_t* box = base + slot * 4096;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            const uint4* src = reinterpret_cast<const uint4*>(v);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                reinterpret_cast<uint4*>(box + lane * 128)[j ^ (lane & 7)] = src[j];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&g_out_map)),
                    "r"(nt * 256 + c), "r"(row0), "r"(smem_u32(box))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            slot ^= 1;
        }
    }
};

template <int BN, bool AMN, bool BMN, class Epi>
void probe(const char* name, int a_rows, int a_cols, int b_rows, int b_cols,
           std::vector<GemmGroup> groups, int grid_pairs) {
    __nv_bfloat16 *A, *B;
    CK(cudaMalloc(&A, (size_t)a_rows * a_cols * 2));
    CK(cudaMalloc(&B, (size_t)b_rows * b_cols * 2));
    fill_rand<<<1024, 256>>>(A, (size_t)a_rows * a_cols, 1);
    fill_rand<<<1024, 256>>>(B, (size_t)b_rows * b_cols, 2);
    int tiles = 0;
    for (auto& g : groups) {
        g.tile_start = tiles;
        tiles += g.m_tiles * g.n_tiles;
    }
    GemmGroup* dg;
    CK(cudaMalloc(&dg, groups.size() * sizeof(GemmGroup)));
    CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    int* dtiles;
    CK(cudaMalloc(&dtiles, 4));
    CK(cudaMemcpy(dtiles, &tiles, 4, cudaMemcpyHostToDevice));
    CUtensorMap ma = spes_host::make_tmap_bf16(A, a_rows, a_cols, AMN ? 64 : 128);
    CUtensorMap mb = spes_host::make_tmap_bf16(B, b_rows, b_cols, BMN ? 64 : BN / 2);
    auto kern = grouped_gemm_2cta_kernel<BN, Epi, AMN, BMN>;
    const int smem = Gemm2Cfg<BN, Epi::SLOTS>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    {  // output for the store probes: [a_rows x b_cols] fp32 (groups write their own rows)
        float* outp;
        CK(cudaMalloc(&outp, (size_t)a_rows * b_cols * 4));
        for (auto& gg : groups) { gg.out0 = outp; gg.ldo = b_cols; }
        CK(cudaMemcpy(dg, groups.data(), groups.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
        CUtensorMap om;
        cuuint64_t dims[2] = {(cuuint64_t)b_cols, (cuuint64_t)a_rows};
        cuuint64_t strides[1] = {(cuuint64_t)b_cols * 4};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t es[2] = {1, 1};
        if (spes_host::tmap_encoder()(&om, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, outp, dims, strides, box,
                                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            printf("out map failed\n");
        CK(cudaMemcpyToSymbol(g_out_map, &om, sizeof(om)));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * grid_pairs);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ng = (int)groups.size();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dg, ng, (const int*)dtiles, tiles, Epi{}));
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i)
        CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dg, ng, (const int*)dtiles, tiles, Epi{}));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 0;
    for (auto& g : groups) flops += 2.0 * g.m_tiles * 256.0 * g.n_tiles * BN * g.k_len;
    printf("[probe %s] pairs=%d %.3f us/launch  %.1f TFLOP/s\n", name, grid_pairs, ms * 1e3 / 20,
           flops / (ms / 20 * 1e-3) / 1e12);
    cudaFree(A); cudaFree(B); cudaFree(dg); cudaFree(dtiles);
}

static GemmGroup G(int a_row0, int b_row0, int k0, int bk0, int k_len, int mt, int nt,
                   int out_row0) {
    GemmGroup g{};
    g.a_row0 = a_row0;
    g.b_row0 = b_row0;
    g.k0 = k0;
    g.bk0 = bk0;
    g.k_len = k_len;
    g.m_tiles = mt;
    g.n_tiles = nt;
    g.out_row0 = out_row0;
    return g;
}

int l2probe_main();
int mma_probe_main();
int main() {
    l2probe_main();
    mma_probe_main();
    int fails = 0;
    // K-major A and B: one pair tile, then routed-style groups (3 experts)
    fails += run<256, false, false>("kk_single", 256, 128, 256, 128, {G(0, 0, 0, 0, 128, 1, 1, 0)},
                                    256, 256, false);
    fails += run<256, false, false>("kk_routed", 1024, 256, 3 * 512, 256,
                                    {G(0, 0, 0, 0, 256, 1, 2, 0), G(256, 512, 0, 0, 256, 2, 2, 256),
                                     G(768, 1024, 0, 0, 0, 1, 2, 768)},
                                    1024, 512, false);
    // A K-major, B row-major weight (MN-major), expert offset via bk0
    fails += run<256, false, true>("kmn_routed", 768, 256, 3 * 256, 512,
                                   {G(0, 0, 0, 0, 256, 1, 2, 0), G(256, 0, 0, 256, 256, 2, 2, 256)},
                                   768, 512, false);
    // weight-gradient form
    fails += run<256, true, true>("mnmn", 1024, 512, 1024, 512,
                                  {G(0, 0, 0, 0, 384, 2, 2, 0), G(0, 0, 384, 384, 640, 2, 2, 512)},
                                  1024, 512, false);
    // throughput probes at cfg2 shapes
    {
        std::vector<GemmGroup> gs;  // gate||up forward: 16 experts x 2048 rows, N = 2048, K = 1024
        for (int j = 0; j < 16; ++j) gs.push_back(G(j * 2048, 0, 0, j * 1024, 1024, 8, 8, j * 2048));
        fails += run<256, false, true>("cfg2_fwd1", 16 * 2048, 1024, 16 * 1024, 2048, gs, 16 * 2048,
                                       2048, true);
    }
    {
        std::vector<GemmGroup> gs;  // dW gate||up: 16 experts, [1024 x 2048] over 2048 tokens each
        for (int j = 0; j < 16; ++j) gs.push_back(G(0, 0, j * 2048, j * 2048, 2048, 4, 8, j * 1024));
        fails += run<256, true, true>("cfg2_dw1", 16 * 2048, 1024, 16 * 2048, 2048, gs, 16 * 1024,
                                      2048, true);
    }
    {
        std::vector<GemmGroup> gs;  // dX: A = dGU [rows x 2048], B = W1 [d x 2048] K-major
        for (int j = 0; j < 16; ++j) gs.push_back(G(j * 2048, j * 1024, 0, 0, 2048, 8, 4, j * 2048));
        fails += run<256, false, false>("cfg2_dx", 16 * 2048, 2048, 16 * 1024, 2048, gs, 16 * 2048,
                                        1024, true);
    }
    {
        std::vector<GemmGroup> gs;
        for (int j = 0; j < 16; ++j) gs.push_back(G(j * 2048, 0, 0, j * 1024, 1024, 8, 8, j * 2048));
        probe<256, false, true, EpiNull>("fwd1_nullepi", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
        probe<256, false, true, EpiTmemOnly>("fwd1_tmem_only", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
        probe<256, false, true, EpiTmemSmem>("fwd1_tmem_smem", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
        probe<256, false, true, EpiStoreF32<256>>("fwd1_put_f32", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
        probe<256, false, true, EpiTmaF32>("fwd1_tma_f32", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
        probe<256, false, true, EpiNull>("fwd1_nullepi_p37", 16 * 2048, 1024, 16 * 1024, 2048, gs, 37);
    }
    printf(fails ? "SELFTEST2 FAILED\n" : "SELFTEST2 OK\n");
    return fails;
}
// (appended) L2-resident operand probe: every group reads the same A rows and B expert
int l2probe_main() {
    std::vector<GemmGroup> gs;
    for (int j = 0; j < 16; ++j) gs.push_back(G(0, 0, 0, 0, 1024, 8, 8, j * 2048));
    probe<256, false, true, EpiNull>("fwd1_l2resident_null", 16 * 2048, 1024, 16 * 1024, 2048, gs, 74);
    return 0;
}
// (appended) MMA-issue-rate probe: operands loaded once, MMAs stream from smem
template <int BN>
void mma_rate_probe() {
    std::vector<GemmGroup> gs;
    for (int j = 0; j < 16; ++j) gs.push_back(G(0, 0, 0, 0, 1024, 8, 8, j * 2048));
    int tiles = 0;
    for (auto& g : gs) { g.tile_start = tiles; tiles += g.m_tiles * g.n_tiles; }
    __nv_bfloat16 *A, *B;
    CK(cudaMalloc(&A, (size_t)32768 * 1024 * 2));
    CK(cudaMalloc(&B, (size_t)16384 * 2048 * 2));
    GemmGroup* dg; CK(cudaMalloc(&dg, gs.size() * sizeof(GemmGroup)));
    CK(cudaMemcpy(dg, gs.data(), gs.size() * sizeof(GemmGroup), cudaMemcpyHostToDevice));
    int* dt; CK(cudaMalloc(&dt, 4)); CK(cudaMemcpy(dt, &tiles, 4, cudaMemcpyHostToDevice));
    CUtensorMap ma = spes_host::make_tmap_bf16(A, 32768, 1024, 128);
    CUtensorMap mb = spes_host::make_tmap_bf16(B, 16384, 2048, 64);
    auto kern = grouped_gemm_2cta_kernel<BN, EpiNull, false, true>;
    const int smem = Gemm2Cfg<BN>::SMEM_BYTES;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(GEMM_THREADS); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int ng = 16;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dg, ng, (const int*)dt, tiles, EpiNull{}));
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) CK(cudaLaunchKernelEx(&cfg, kern, ma, mb, (const GemmGroup*)dg, ng, (const int*)dt, tiles, EpiNull{}));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 16.0 * 8 * 8 * 2.0 * 256 * 256 * 1024;
    printf("[probe null epilogue] %.3f us/launch  %.1f TFLOP/s\n", ms * 1e3 / 20, flops / (ms / 20 * 1e-3) / 1e12);
}
int mma_probe_main() { mma_rate_probe<256>(); return 0; }
