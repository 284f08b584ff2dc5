// Epilogue store-path microbenchmark (no MMA): 148 CTAs x 8 warps, each CTA writes
// NT tiles of 128 rows x 256 fp32 columns into a [rows x 2048] fp32 buffer, the way the
// grouped GEMM epilogue does (warp = 32 rows x 128 columns, 32-column pieces per lane).
//   direct : each lane stores its row piece with 8 x STG.128
//   put    : smem transpose (EpiOut::put), 4 whole rows per STG.128
//   tma    : 128B-swizzled smem box + cp.async.bulk.tensor.2d store (one lane)
#include <cstdio>
#include <vector>

#include "../common.cuh"
#include "../grouped_gemm.cuh"
#include "../tmap.hpp"

using namespace spes_dev;

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

constexpr int COLS = 2048;

__device__ __forceinline__ void fill(float (&v)[32], int seed) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = static_cast<float>(seed + i);
}

// AdamW-epilogue pattern (no MMA): per 32-column piece fetch theta / m / v rows with
// cp.async into 3 slots, update in place, store back row-major (+ bf16 shadow)
template <int NW, int PW>
__global__ void __launch_bounds__(NW * 32, 1)
    adam_k(float* th, float* m, float* v, __nv_bfloat16* sh, int ntiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NCOL = NW / 4;           // column groups per lane quarter
    constexpr int CW = 256 / NCOL;         // columns per warp
    constexpr int N16 = PW / 4;
    const int q = warp & 3, half = warp >> 2;  // half = column group index
    EpiOut eo{smem + warp * 3 * EPI_SLOT_BYTES, lane};
    AdamScalars a{1e-3f, 0.9f, 0.95f, 0.1f, 0.05f, 1e-8f, 0.1f, 0.1f, 0.05f};
    for (int it = 0; it < ntiles; ++it) {
        const int tile = blockIdx.x * ntiles + it;
        const int mt = tile / (COLS / 256), nt = tile % (COLS / 256);
        const int64_t row = static_cast<int64_t>(mt) * 128 + q * 32 + lane;
        for (int c = half * CW; c < half * CW + CW; c += PW) {
            const int64_t off = row * COLS + nt * 256 + c;
            eo.rows_load_async<N16>(0, th + off);
            eo.rows_load_async<N16>(1, m + off);
            eo.rows_load_async<N16>(2, v + off);
            eo.rows_wait();
            float tv[32];
#pragma unroll
            for (int h2 = 0; h2 < PW / 16; ++h2) {  // 16 elements in registers: full ILP
                float4 t4[4], m4[4], v4[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    t4[j] = reinterpret_cast<float4*>(eo.my_row(0))[4 * h2 + j];
                    m4[j] = reinterpret_cast<float4*>(eo.my_row(1))[4 * h2 + j];
                    v4[j] = reinterpret_cast<float4*>(eo.my_row(2))[4 * h2 + j];
                }
                float* tt = &t4[0].x;
                float* mmv = &m4[0].x;
                float* vvv = &v4[0].x;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    tt[i] = adam_elem(tt[i], 0.001f * (16 * h2 + i), mmv[i], vvv[i], a);
                    tv[16 * h2 + i] = tt[i];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    reinterpret_cast<float4*>(eo.my_row(0))[4 * h2 + j] = t4[j];
                    reinterpret_cast<float4*>(eo.my_row(1))[4 * h2 + j] = m4[j];
                    reinterpret_cast<float4*>(eo.my_row(2))[4 * h2 + j] = v4[j];
                }
            }
            eo.rows_store<N16>(0, th + off);
            eo.rows_store<N16>(1, m + off);
            eo.rows_store<N16>(2, v + off);
            uint4 pk[4];
#pragma unroll
            for (int i = 0; i < PW / 8; ++i) {
                __nv_bfloat162 x0 = __floats2bfloat162_rn(tv[8 * i], tv[8 * i + 1]);
                __nv_bfloat162 x1 = __floats2bfloat162_rn(tv[8 * i + 2], tv[8 * i + 3]);
                __nv_bfloat162 x2 = __floats2bfloat162_rn(tv[8 * i + 4], tv[8 * i + 5]);
                __nv_bfloat162 x3 = __floats2bfloat162_rn(tv[8 * i + 6], tv[8 * i + 7]);
                pk[i] = make_uint4(*reinterpret_cast<uint32_t*>(&x0), *reinterpret_cast<uint32_t*>(&x1),
                                   *reinterpret_cast<uint32_t*>(&x2), *reinterpret_cast<uint32_t*>(&x3));
            }
            if constexpr (PW == 32) eo.put<4>(sh + off, pk, 0);
            else { reinterpret_cast<uint4*>(sh + off)[0] = pk[0]; reinterpret_cast<uint4*>(sh + off)[1] = pk[1]; }
        }
    }
}

// Same with the next piece's rows prefetched into registers (row-major loads) while the
// current piece is updated and stored; PW = piece width in columns (16 or 32).
template <int PW>
__global__ void __launch_bounds__(256, 1)
    adam_pf_k(float* th, float* m, float* v, __nv_bfloat16* sh, int ntiles) {
    constexpr int N16 = PW / 4;  // 16-byte words per row piece (4 or 8)
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    EpiOut eo{smem + warp * 3 * EPI_SLOT_BYTES, lane};
    AdamScalars a{1e-3f, 0.9f, 0.95f, 0.1f, 0.05f, 1e-8f, 0.1f, 0.1f, 0.05f};
    constexpr int PPT = 128 / PW;  // pieces per tile-half
    const int npieces = ntiles * PPT;
    auto off_of = [&](int pi) {
        const int it = pi / PPT, c = half * 128 + (pi % PPT) * PW;
        const int tile = blockIdx.x * ntiles + it;
        const int mt = tile / (COLS / 256), nt = tile % (COLS / 256);
        const int64_t row = static_cast<int64_t>(mt) * 128 + q * 32 + lane;
        return row * COLS + nt * 256 + c;
    };
    uint4 rt[N16], rm[N16], rv[N16];
    eo.load_rows<N16>(th + off_of(0), rt);
    eo.load_rows<N16>(m + off_of(0), rm);
    eo.load_rows<N16>(v + off_of(0), rv);
    for (int pi = 0; pi < npieces; ++pi) {
        const int64_t off = off_of(pi);
        // land this piece into the slots (transposed: lane = row)
        {
            constexpr int RPI = 32 / N16;
            const int sub = lane % N16, r0 = lane / N16;
#pragma unroll
            for (int i = 0; i < N16; ++i) {
                reinterpret_cast<uint4*>(eo.row_of(0, i * RPI + r0))[sub] = rt[i];
                reinterpret_cast<uint4*>(eo.row_of(1, i * RPI + r0))[sub] = rm[i];
                reinterpret_cast<uint4*>(eo.row_of(2, i * RPI + r0))[sub] = rv[i];
            }
            __syncwarp();
        }
        if (pi + 1 < npieces) {  // next piece in flight during this one
            const int64_t o2 = off_of(pi + 1);
            eo.load_rows<N16>(th + o2, rt);
            eo.load_rows<N16>(m + o2, rm);
            eo.load_rows<N16>(v + o2, rv);
        }
        float* t = reinterpret_cast<float*>(eo.my_row(0));
        float* mm = reinterpret_cast<float*>(eo.my_row(1));
        float* vv = reinterpret_cast<float*>(eo.my_row(2));
        float tv[PW];
#pragma unroll
        for (int i = 0; i < PW; ++i) {
            t[i] = adam_elem(t[i], 0.001f * i, mm[i], vv[i], a);
            tv[i] = t[i];
        }
        eo.rows_store<N16>(0, th + off);
        eo.rows_store<N16>(1, m + off);
        eo.rows_store<N16>(2, v + off);
        uint4 pk[N16 / 2];
#pragma unroll
        for (int i = 0; i < N16 / 2; ++i) {
            __nv_bfloat162 x0 = __floats2bfloat162_rn(tv[8 * i], tv[8 * i + 1]);
            __nv_bfloat162 x1 = __floats2bfloat162_rn(tv[8 * i + 2], tv[8 * i + 3]);
            __nv_bfloat162 x2 = __floats2bfloat162_rn(tv[8 * i + 4], tv[8 * i + 5]);
            __nv_bfloat162 x3 = __floats2bfloat162_rn(tv[8 * i + 6], tv[8 * i + 7]);
            pk[i] = make_uint4(*reinterpret_cast<uint32_t*>(&x0), *reinterpret_cast<uint32_t*>(&x1),
                               *reinterpret_cast<uint32_t*>(&x2), *reinterpret_cast<uint32_t*>(&x3));
        }
        if constexpr (N16 == 8) eo.put<4>(sh + off, pk, 0);
        else {  // 32-byte shadow pieces: direct
            uint4* d = reinterpret_cast<uint4*>(sh + off);
            d[0] = pk[0];
            d[1] = pk[1];
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(256, 1)
    epi_k(float* out, int ntiles, const __grid_constant__ CUtensorMap map) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    EpiOut eo{smem + warp * EPI_SLOT_BYTES, lane};
    uint8_t* tslot = smem + 8 * EPI_SLOT_BYTES + warp * 8192;  // 2 x 4 KiB swizzled boxes
    int slot = 0;
    for (int it = 0; it < ntiles; ++it) {
        const int tile = blockIdx.x * ntiles + it;
        const int mt = tile / (COLS / 256), nt = tile % (COLS / 256);
        const int64_t row = static_cast<int64_t>(mt) * 128 + q * 32 + lane;
        float* dst = out + row * COLS + nt * 256;
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
            float v[32];
            fill(v, tile + c);
            if (MODE == 0) {
                float4* d4 = reinterpret_cast<float4*>(dst + c);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else if (MODE == 1) {
                eo.put_f32x32(dst + c, v);
            } else if (MODE == 3) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + c + 8 * i),
                                 "f"(v[8 * i]), "f"(v[8 * i + 1]), "f"(v[8 * i + 2]), "f"(v[8 * i + 3]),
                                 "f"(v[8 * i + 4]), "f"(v[8 * i + 5]), "f"(v[8 * i + 6]), "f"(v[8 * i + 7])
                                 : "memory");
            } else {
                if (lane == 0)
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                uint8_t* box = tslot + slot * 4096;
                const uint4* src = reinterpret_cast<const uint4*>(v);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    reinterpret_cast<uint4*>(box + lane * 128)[j ^ (lane & 7)] = src[j];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                            reinterpret_cast<uint64_t>(&map)),
                        "r"(nt * 256 + c), "r"(static_cast<int>(mt * 128 + q * 32)), "r"(smem_u32(box))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                slot ^= 1;
            }
        }
    }
    if (MODE == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE>
float run(float* out, int ntiles, const CUtensorMap& map) {
    const int smem = 8 * EPI_SLOT_BYTES + 8 * 8192 + 1024;
    CK(cudaFuncSetAttribute(epi_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int i = 0; i < 3; ++i) epi_k<MODE><<<148, 256, smem>>>(out, ntiles, map);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) epi_k<MODE><<<148, 256, smem>>>(out, ntiles, map);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}

int main() {
    const int ntiles = 14;
    const int64_t tiles = 148LL * ntiles;
    const int64_t rows = tiles / (COLS / 256) * 128;
    float* out;
    CK(cudaMalloc(&out, rows * COLS * 4));
    CUtensorMap map;
    {
        cuuint64_t dims[2] = {COLS, static_cast<cuuint64_t>(rows)};
        cuuint64_t strides[1] = {COLS * 4};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t es[2] = {1, 1};
        CUresult r = spes_host::tmap_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims,
                                               strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                               CU_TENSOR_MAP_SWIZZLE_128B,
                                               CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("tmap failed %d\n", r);
            return 1;
        }
    }
    const double bytes = static_cast<double>(rows) * COLS * 4;
    const char* names[4] = {"direct", "put", "tma", "v8"};
    float t[4] = {run<0>(out, ntiles, map), run<1>(out, ntiles, map), run<2>(out, ntiles, map),
                  run<3>(out, ntiles, map)};
    for (int m = 0; m < 4; ++m)
        printf("[epi %-6s] %8.2f us  %7.1f GB/s  (%.2f us per tile per CTA)\n", names[m], t[m] * 1e3,
               bytes / (t[m] * 1e-3) / 1e9, t[m] * 1e3 / ntiles);
    // verify tma and put wrote identical data
    std::vector<float> h(static_cast<size_t>(rows) * COLS);
    CK(cudaMemcpy(h.data(), out, rows * COLS * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int64_t r = 0; r < rows; ++r)
        for (int c = 0; c < COLS; ++c) {
            const int mt = static_cast<int>(r / 128), nt = c / 256;
            const int tile = mt * (COLS / 256) + nt;
            const int cc = c % 256;
            const float want = static_cast<float>(tile + (cc / 32) * 32 + (cc % 32));
            if (h[r * COLS + c] != want) ++bad;
        }
    printf("verify: %ld bad\n", bad);
    {  // AdamW epilogue pattern: 26 bytes per element
        float *th, *m, *v;
        __nv_bfloat16* sh;
        CK(cudaMalloc(&th, rows * COLS * 4));
        CK(cudaMalloc(&m, rows * COLS * 4));
        CK(cudaMalloc(&v, rows * COLS * 4));
        CK(cudaMalloc(&sh, rows * COLS * 2));
        CK(cudaMemset(th, 0, rows * COLS * 4));
        CK(cudaMemset(m, 0, rows * COLS * 4));
        CK(cudaMemset(v, 0, rows * COLS * 4));
        int smem = 8 * 3 * EPI_SLOT_BYTES;
        cudaEvent_t a0, b0;
        cudaEventCreate(&a0);
        cudaEventCreate(&b0);
        const double ab = static_cast<double>(rows) * COLS * 26;
        auto runw = [&](auto kern, int nw, const char* nm) {
            const int sm = nw * 3 * EPI_SLOT_BYTES;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            for (int i = 0; i < 2; ++i) kern<<<148, nw * 32, sm>>>(th, m, v, sh, ntiles);
            cudaEventRecord(a0);
            for (int i = 0; i < 5; ++i) kern<<<148, nw * 32, sm>>>(th, m, v, sh, ntiles);
            cudaEventRecord(b0);
            CK(cudaEventSynchronize(b0));
            float ms;
            cudaEventElapsedTime(&ms, a0, b0);
            ms /= 5;
            printf("[epi %-6s] %8.2f us  %7.1f GB/s  (%.2f us per tile per CTA)\n", nm, ms * 1e3,
                   ab / (ms * 1e-3) / 1e9, ms * 1e3 / ntiles);
        };
        runw(adam_k<8, 32>, 8, "a8x32");
        runw(adam_k<16, 32>, 16, "a16x32");
        runw(adam_k<16, 16>, 16, "a16x16");
        runw(adam_k<8, 16>, 8, "a8x16");
        auto runpf = [&](auto kern, const char* nm) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            for (int i = 0; i < 2; ++i) kern<<<148, 256, smem>>>(th, m, v, sh, ntiles);
            cudaEventRecord(a0);
            for (int i = 0; i < 5; ++i) kern<<<148, 256, smem>>>(th, m, v, sh, ntiles);
            cudaEventRecord(b0);
            CK(cudaEventSynchronize(b0));
            float ms2;
            cudaEventElapsedTime(&ms2, a0, b0);
            ms2 /= 5;
            printf("[epi %-6s] %8.2f us  %7.1f GB/s\n", nm, ms2 * 1e3, ab / (ms2 * 1e-3) / 1e9);
        };
        runpf(adam_pf_k<32>, "pf32");
        runpf(adam_pf_k<16>, "pf16");
    }
    return bad != 0;
}
