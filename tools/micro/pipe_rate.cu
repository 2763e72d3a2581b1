// Issue rate of the FP32 forms on one B200 (sm_100a): FFMA (3 registers), FFMA2 (packed f32x2), FMNMX (ALU pipe)
// and an FFMA + FMNMX mix.  8 independent chains per thread, 32 warps per SM, 148 x 8 blocks; reports warp-
// instructions per cycle per SM from clock64 and CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
    float r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = fmaf(r[i], a, r[(i + 1) & 7]);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long f2(float x, float y) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
}

__global__ void k_ffma2(float* out, float a, float b) {
    unsigned long long r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = f2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const unsigned long long aa = f2(a, b);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(r[i]) : "l"(aa), "l"(r[(i + 1) & 7]));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)r[i]) + __uint_as_float((unsigned)(r[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fmnmx(float* out, float a, float b) {
    float r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = fmaxf(r[i], r[(i + 1) & 7]);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mix(float* out, float a, float b) {
    float r[8], q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { r[i] = threadIdx.x * 1e-3f + i; q[i] = i; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { r[i] = fmaf(r[i], a, r[(i + 1) & 7]); q[i] = fmaxf(q[i], q[(i + 1) & 7]); }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += r[i] + q[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
void run(const char* name, K kern, int instr_per_iter) {
    int nsm, clk;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 256, blocks = nsm * 8;
    float* out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    kern<<<blocks, threads>>>(out, 0.999f, 0.5f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 0.999f, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = 5.0 * blocks * (threads / 32) * (double)ITERS * instr_per_iter;
    const double cycles = ms * 1e-3 * 1965e6;      // at the max SM clock (clocks are not locked: an estimate)
    printf("%-8s %.3f ms  %.2f warp-instr / cycle / SM  (%.1f T thread-instr/s)\n", name, ms, warp_instr / cycles / nsm,
           warp_instr * 32 / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    run("FFMA", k_ffma, 8);
    run("FFMA2", k_ffma2, 8);
    run("FMNMX", k_fmnmx, 8);
    run("mix", k_mix, 16);
    return 0;
}
