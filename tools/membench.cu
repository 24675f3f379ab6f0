// membench.cu -- achievable HBM bandwidth of the streaming access mixes the hot path uses
// (dev tool; not part of libtqp). Each pattern runs over 60M int64 rows (the SF10 probe
// side), timed with CUDA events, best of 20:
//   r8w16 : read 8 B, write 16 B to two arrays (the PK-FK probe's direct output)
//   r8w8  : read 8 B, write 8 B (a copy)
//   w16   : write 16 B to two arrays
//   r8    : read 8 B (reduced to one word so the loads are kept)
//   r38   : read 38 B per row over 7 columns (Q1's columns: 4 + 1 + 1 + 4 x 8)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void r8w16(const long long* __restrict__ a, long long* __restrict__ l, long long* __restrict__ r, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long v = __ldcs(a + i);
        __stcs(l + i, v + 1);
        __stcs(r + i, i);
    }
}
__global__ void r8w8(const long long* __restrict__ a, long long* __restrict__ l, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(l + i, __ldcs(a + i) + 1);
}
__global__ void w16(long long* __restrict__ l, long long* __restrict__ r, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        __stcs(l + i, i);
        __stcs(r + i, i);
    }
}
__global__ void r8(const long long* __restrict__ a, long long* out, int64_t n) {
    long long s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s ^= __ldcs(a + i);
    if (s == 0x123456789) *out = s;
}
__global__ void r38(const int* __restrict__ d, const unsigned char* __restrict__ f1, const unsigned char* __restrict__ f2,
                    const long long* __restrict__ q, const long long* __restrict__ p, const long long* __restrict__ di,
                    const long long* __restrict__ t, long long* out, int64_t n) {
    long long s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += __ldcs(d + i) + __ldcs(f1 + i) + __ldcs(f2 + i) + __ldcs(q + i) + __ldcs(p + i) + __ldcs(di + i) + __ldcs(t + i);
    if (s == 0x123456789) *out = s;
}

template <typename F>
static float best(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float bestms = 1e9f;
    for (int it = 0; it < 20; it++) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 1 && ms < bestms) bestms = ms;
    }
    return bestms;
}

int main() {
    const int64_t n = 60000000;
    long long *a, *l, *r, *o, *q, *p, *di, *t;
    int* d;
    unsigned char *f1, *f2;
    cudaMalloc(&a, n * 8); cudaMalloc(&l, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&o, 8);
    cudaMalloc(&q, n * 8); cudaMalloc(&p, n * 8); cudaMalloc(&di, n * 8); cudaMalloc(&t, n * 8);
    cudaMalloc(&d, n * 4); cudaMalloc(&f1, n); cudaMalloc(&f2, n);
    cudaMemset(a, 1, n * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {4, 8, 16}) {
        const int g = sms * per;
        float ms;
        ms = best([&] { r8w16<<<g, 256>>>(a, l, r, n); });
        printf("grid %5d r8w16 %.4f ms %.0f GB/s\n", g, ms, 24.0 * n / ms / 1e6);
        ms = best([&] { r8w8<<<g, 256>>>(a, l, n); });
        printf("grid %5d r8w8  %.4f ms %.0f GB/s\n", g, ms, 16.0 * n / ms / 1e6);
        ms = best([&] { w16<<<g, 256>>>(l, r, n); });
        printf("grid %5d w16   %.4f ms %.0f GB/s\n", g, ms, 16.0 * n / ms / 1e6);
        ms = best([&] { r8<<<g, 256>>>(a, o, n); });
        printf("grid %5d r8    %.4f ms %.0f GB/s\n", g, ms, 8.0 * n / ms / 1e6);
        ms = best([&] { r38<<<g, 256>>>(d, f1, f2, q, p, di, t, o, n); });
        printf("grid %5d r38   %.4f ms %.0f GB/s\n", g, ms, 38.0 * n / ms / 1e6);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
