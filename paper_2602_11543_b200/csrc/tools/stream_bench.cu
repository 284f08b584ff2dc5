// HBM streaming ceiling for the AdamW access pattern: 4 fp32 read streams (theta, g, m, v),
// 3 fp32 write streams (theta, m, v) and one bf16 write stream, 28 + 2 B per element,
// with the same float4 / 2-in-flight layout as adamw_k, versus a plain copy.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <int U>
__global__ void adam_like_k(float4* th, const float4* __restrict__ g, float4* m, float4* v,
                            uint2* sh, long n4) {
    const long stride = (long)gridDim.x * blockDim.x * U;
    for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n4; base += stride) {
        float4 t[U], gg[U], mm[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + (long)u * blockDim.x;
            t[u] = th[i]; gg[u] = __ldcs(g + i); mm[u] = __ldcs(m + i); vv[u] = __ldcs(v + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + (long)u * blockDim.x;
            t[u].x += gg[u].x * 1e-3f; mm[u].x += gg[u].y; vv[u].x += gg[u].z;
            th[i] = t[u]; __stcs(m + i, mm[u]); __stcs(v + i, vv[u]);
            __nv_bfloat162 a = __floats2bfloat162_rn(t[u].x, t[u].y), b = __floats2bfloat162_rn(t[u].z, t[u].w);
            sh[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
        }
    }
}

int main() {
    const long n = 51L << 20, n4 = n / 4;
    float4 *a, *b, *c, *d;
    uint2* s;
    cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&d, n * 4);
    cudaMalloc(&s, n * 2);
    cudaMemset(a, 0, n * 4); cudaMemset(b, 0, n * 4); cudaMemset(c, 0, n * 4); cudaMemset(d, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](auto f, const char* name, double bytes) {
        for (int i = 0; i < 3; ++i) f();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
        printf("[%-14s] %8.1f us  %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    time([&] { copy_k<<<148 * 8, 256>>>(a, b, n4); }, "copy", 8.0 * n);
    time([&] { adam_like_k<1><<<148 * 8, 256>>>(a, b, c, d, s, n4); }, "adam-like U1", 30.0 * n);
    time([&] { adam_like_k<2><<<148 * 8, 256>>>(a, b, c, d, s, n4); }, "adam-like U2", 30.0 * n);
    time([&] { adam_like_k<2><<<148 * 16, 256>>>(a, b, c, d, s, n4); }, "adam-like U2 2x", 30.0 * n);
    time([&] { adam_like_k<4><<<148 * 4, 256>>>(a, b, c, d, s, n4); }, "adam-like U4", 30.0 * n);
    return 0;
}
