// Dependent-chain latency of FFMA and FFMA2 (one warp per SM, clock64 around a chain of 4096 dependent ops).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void lat_ffma(float* out, long long* cyc, float a) {
    float x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fmaf(x, a, 0.5f * a);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_ffma2(float* out, long long* cyc, float a) {
    unsigned long long x = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint((float)threadIdx.x);
    const unsigned long long aa = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x) : "l"(aa));
    long long t1 = clock64();
    out[threadIdx.x] = __uint_as_float((unsigned)x) + __uint_as_float((unsigned)(x >> 32));
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_fadd2(float* out, long long* cyc, float a) {
    unsigned long long x = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint((float)threadIdx.x);
    const unsigned long long aa = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(aa));
    long long t1 = clock64();
    out[threadIdx.x] = __uint_as_float((unsigned)x) + __uint_as_float((unsigned)(x >> 32));
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <class K> void run(const char* nm, K k) {
    float* o; long long* c; long long h;
    cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
    k<<<1, 32>>>(o, c, 0.999f);
    k<<<1, 32>>>(o, c, 0.999f);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-6s %.2f cycles per dependent op\n", nm, (double)h / N);
}
int main() { run("FFMA", lat_ffma); run("FFMA2", lat_ffma2); run("FADD2", lat_fadd2); return 0; }
