// Fused epilogues of the grouped tcgen05 GEMM (grouped_gemm.cuh) and their launchers.
//
//   EpiSwiGLU   expert forward gate||up: accumulator columns [0,128) are gate,
//               [128,256) the matching up columns; writes GU (bf16, saved for
//               backward) and Hact = silu(G)*U (bf16).
//   EpiStoreF32 plain fp32 tile store (expert down-proj Y, dX, head logits / dh,
//               dWd and dHead straight into the gradient buffer).
//   EpiDSwiGLU  expert backward: dHact -> (dG, dU) using the saved GU, written as
//               dGU (bf16) for the dX and dW GEMMs.
//   EpiGradW1   dW of gate||up straight into the fp32 wg / wu gradient blocks.
// Weight-gradient GEMMs read the row-major activations directly as MN-major
// operands (grouped_gemm_kernel<..., MN=true>): no transposed copies are made.
#include "common.cuh"
#include "grouped_gemm.cuh"
#include "grouped_gemm_2cta.cuh"
#include "kernels.h"

#include <stdexcept>

namespace spes_k {

using namespace spes_dev;

__device__ __forceinline__ void store_bf16x32(bf16* dst, const float (&v)[32]) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint4 pk;
        __nv_bfloat162 a = __floats2bfloat162_rn(v[8 * i + 0], v[8 * i + 1]);
        __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * i + 2], v[8 * i + 3]);
        __nv_bfloat162 c = __floats2bfloat162_rn(v[8 * i + 4], v[8 * i + 5]);
        __nv_bfloat162 d = __floats2bfloat162_rn(v[8 * i + 6], v[8 * i + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&a);
        pk.y = *reinterpret_cast<uint32_t*>(&b);
        pk.z = *reinterpret_cast<uint32_t*>(&c);
        pk.w = *reinterpret_cast<uint32_t*>(&d);
        d4[i] = pk;
    }
}

__device__ __forceinline__ void load_bf16x32(const bf16* src, float (&v)[32]) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4 pk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) pk[i] = __ldg(s4 + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&pk[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 f = __bfloat1622float2(h[j]);
            v[8 * i + 2 * j] = f.x;
            v[8 * i + 2 * j + 1] = f.y;
        }
    }
}

struct EpiSwiGLU {
    bf16* hact;
    int64_t f;
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        bf16* gu = static_cast<bf16*>(g.out0) + row * g.ldo + static_cast<int64_t>(nt) * 256;
        bf16* ha = hact + row * f + static_cast<int64_t>(nt) * 128;
#pragma unroll 1
        for (int c = half * 64; c < half * 64 + 64; c += 32) {
            float gv[32], uv[32], hv[32];
            acc_load32(taddr + c, empty, gv);
            acc_load32(taddr + 128 + c, empty, uv);
#pragma unroll
            for (int i = 0; i < 32; ++i) hv[i] = gv[i] * sigmoid_fast(gv[i]) * uv[i];
            store_bf16x32(gu + c, gv);
            store_bf16x32(gu + 128 + c, uv);
            store_bf16x32(ha + c, hv);
        }
    }
};

template <int BN>
struct EpiDSwiGLU {
    const bf16* gu;
    int64_t f;
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half) const {
        const int64_t row = g.out_row0 + static_cast<int64_t>(mt) * GEMM_BM + r;
        const bf16* gurow = gu + row * 2 * f;
        bf16* dgurow = static_cast<bf16*>(g.out0) + row * g.ldo;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            const int64_t x0 = static_cast<int64_t>(nt) * BN + c;  // f index of column 0
            const int64_t ig = il_gate(x0), iu = il_up(x0);
            float dh[32], gv[32], uv[32], dg[32], du[32];
            load_bf16x32(gurow + ig, gv);
            load_bf16x32(gurow + iu, uv);
            acc_load32(taddr + c, empty, dh);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float s = sigmoid_fast(gv[i]);
                dg[i] = dh[i] * uv[i] * (s * (1.f + gv[i] * (1.f - s)));
                du[i] = dh[i] * (gv[i] * s);
            }
            store_bf16x32(dgurow + ig, dg);
            store_bf16x32(dgurow + iu, du);
        }
    }
};

struct EpiGradW1 {
    __device__ void operator()(const GemmGroup& g, int mt, int nt, int r, uint32_t taddr,
                               bool empty, int half) const {
        const int64_t row = static_cast<int64_t>(mt) * GEMM_BM + r;  // d index
#pragma unroll 1
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            acc_load32(taddr + c, empty, v);
            float* base = static_cast<float*>(c < 128 ? g.out0 : g.out1);
            float* dst = base + row * g.ldo + static_cast<int64_t>(nt) * 128 + (c & 127);
            float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
    }
};

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

thread_local bool g_gemm_pairs = false;
void gemm_set_pair_mode(bool on) { g_gemm_pairs = on; }

// Pair mode: cta_group::2 kernel on cluster pairs (tiles of 256 rows); otherwise the
// 1-CTA kernel (tiles of 128 rows). The group tables must match the mode.
template <int BN, bool AMN, bool BMN, class Epi>
static void launch(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const Epi& epi, cudaStream_t s) {
    if (max_tiles <= 0) return;
    if (ng > GEMM_MAX_GROUPS) throw std::invalid_argument("grouped GEMM: too many groups");
    if (g_gemm_pairs) {
        auto kern = grouped_gemm_2cta_kernel<BN, Epi, AMN, BMN>;
        static bool configured2 = false;
        if (!configured2) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Gemm2Cfg<BN>::SMEM_BYTES);
            configured2 = true;
        }
        const int pairs = max_tiles < num_sms() / 2 ? max_tiles : num_sms() / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(GEMM_THREADS);
        cfg.dynamicSmemBytes = Gemm2Cfg<BN>::SMEM_BYTES;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, a, b, g, ng, tiles, max_tiles, epi);
        count_launch();
        return;
    }
    auto kern = grouped_gemm_kernel<BN, Epi, AMN, BMN>;
    static bool configured = false;  // one per template instantiation
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             GemmCfg<BN>::SMEM_BYTES);
        configured = true;
    }
    const int grid = max_tiles < num_sms() ? max_tiles : num_sms();
    kern<<<grid, GEMM_THREADS, GemmCfg<BN>::SMEM_BYTES, s>>>(a, b, g, ng, tiles, max_tiles, epi);
    count_launch();
}

void gemm_prepare(int device) {
    (void)device;
    num_sms();
}

// expert forward gate||up: A = Xp (K-major), B = W1 [d x 2f] row-major (MN-major)
void gemm_swiglu(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                 const int32_t* tiles, int max_tiles, bf16* hact, int64_t f, cudaStream_t s) {
    launch<256, false, true>(a, b, g, ng, tiles, max_tiles, EpiSwiGLU{hact, f}, s);
}

template <int BN>
static void store_f32(GemmMajor mj, const CUtensorMap& a, const CUtensorMap& b,
                      const GemmGroup* g, int ng, const int32_t* tiles, int max_tiles,
                      cudaStream_t s) {
    switch (mj) {
        case GemmMajor::KK:
            launch<BN, false, false>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
        case GemmMajor::KMN:
            launch<BN, false, true>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
        case GemmMajor::MNMN:
            launch<BN, true, true>(a, b, g, ng, tiles, max_tiles, EpiStoreF32<BN>{}, s);
            break;
    }
}

void gemm_store_f32(int bn, GemmMajor mj, const CUtensorMap& a, const CUtensorMap& b,
                    const GemmGroup* g, int ng, const int32_t* tiles, int max_tiles,
                    cudaStream_t s) {
    if (bn == 256)
        store_f32<256>(mj, a, b, g, ng, tiles, max_tiles, s);
    else
        store_f32<128>(mj, a, b, g, ng, tiles, max_tiles, s);
}

void gemm_dswiglu(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, const bf16* gu, int64_t f,
                  cudaStream_t s) {
    if (bn == 256)
        launch<256, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLU<256>{gu, f}, s);
    else
        launch<128, false, false>(a, b, g, ng, tiles, max_tiles, EpiDSwiGLU<128>{gu, f}, s);
}

void gemm_grad_w1(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, cudaStream_t s) {
    launch<256, true, true>(a, b, g, ng, tiles, max_tiles, EpiGradW1{}, s);
}

}  // namespace spes_k
