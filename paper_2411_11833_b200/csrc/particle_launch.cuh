// particle_launch.cuh -- launch helpers for the k_particle instantiations (one per translation unit).
#pragma once
#include "particle.cuh"

namespace tamp {
void note_launch();

template <int MODE, int LPF, int HP, int BSYNC, bool SM, int MAXT>
static cudaError_t launch_particle_t(const KProgram& P, const KArgs& A, int threads, size_t smem, cudaStream_t st) {
    auto fn = k_particle<MODE, LPF, HP, BSYNC, SM, MAXT>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int per_block = threads / (LPF * HP);
    const int64_t blocks = (A.n + per_block - 1) / per_block;
    fn<<<(unsigned)blocks, threads, smem, st>>>(P, A);
    note_launch();
    return cudaGetLastError();
}

template <int LPF, int HP, bool SM, int MAXT>
static cudaError_t launch_particle_map(int mode, int bsync, const KProgram& P, const KArgs& A, int threads, size_t smem,
                                       cudaStream_t st) {
    if (mode == MODE_EVAL) return launch_particle_t<MODE_EVAL, LPF, HP, 2, SM, MAXT>(P, A, threads, smem, st);
    if (mode == MODE_CHECK) {
        if (bsync == 0) return launch_particle_t<MODE_CHECK, LPF, HP, 0, SM, MAXT>(P, A, threads, smem, st);
        if (bsync == 1) return launch_particle_t<MODE_CHECK, LPF, HP, 1, SM, MAXT>(P, A, threads, smem, st);
        return launch_particle_t<MODE_CHECK, LPF, HP, 2, SM, MAXT>(P, A, threads, smem, st);
    }
    switch (bsync) {
        case 0: return launch_particle_t<MODE_OPT, LPF, HP, 0, SM, MAXT>(P, A, threads, smem, st);
        case 1: return launch_particle_t<MODE_OPT, LPF, HP, 1, SM, MAXT>(P, A, threads, smem, st);
        default: return launch_particle_t<MODE_OPT, LPF, HP, 2, SM, MAXT>(P, A, threads, smem, st);
    }
}

template <int LPF, int HP, bool SM, int MAXT>
static int particle_regs_t() {
    static int cached = 0;   // a property of the loaded module: queried once per process
    if (cached) return cached;
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, k_particle<MODE_OPT, LPF, HP, 1, SM, MAXT>) != cudaSuccess) {
        cudaGetLastError();
        return MAXT == 512 ? 128 : 80;
    }
    cached = a.numRegs;
    return cached;
}

}  // namespace tamp
