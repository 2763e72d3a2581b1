// tamp_particle_smooth.cu -- instantiations of k_particle with the CHOMP-smooth collision cost
// (split from tamp_kernels.cu so the instantiations compile in parallel).
#include "particle.cuh"

namespace tamp {
void note_launch();
static inline void counted() { note_launch(); }

template <int MODE, int LPF, int HP, int BSYNC, bool SM>
static cudaError_t launch_particle_t(const KProgram& P, const KArgs& A, int threads, size_t smem, cudaStream_t st) {
    auto fn = k_particle<MODE, LPF, HP, BSYNC, SM>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int per_block = threads / (LPF * HP);
    const int64_t blocks = (A.n + per_block - 1) / per_block;
    fn<<<(unsigned)blocks, threads, smem, st>>>(P, A);
    counted();
    return cudaGetLastError();
}

template <int LPF, int HP, bool SM>
static cudaError_t launch_particle_map(int mode, int bsync, const KProgram& P, const KArgs& A, int threads, size_t smem,
                                       cudaStream_t st) {
    if (mode == MODE_EVAL) return launch_particle_t<MODE_EVAL, LPF, HP, 2, SM>(P, A, threads, smem, st);
    if (mode == MODE_CHECK) {
        if (bsync == 0) return launch_particle_t<MODE_CHECK, LPF, HP, 0, SM>(P, A, threads, smem, st);
        if (bsync == 1) return launch_particle_t<MODE_CHECK, LPF, HP, 1, SM>(P, A, threads, smem, st);
        return launch_particle_t<MODE_CHECK, LPF, HP, 2, SM>(P, A, threads, smem, st);
    }
    switch (bsync) {
        case 0: return launch_particle_t<MODE_OPT, LPF, HP, 0, SM>(P, A, threads, smem, st);
        case 1: return launch_particle_t<MODE_OPT, LPF, HP, 1, SM>(P, A, threads, smem, st);
        default: return launch_particle_t<MODE_OPT, LPF, HP, 2, SM>(P, A, threads, smem, st);
    }
}


cudaError_t launch_particle_smooth(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                 size_t smem, cudaStream_t st) {
    if (gs == 16) return launch_particle_map<8, 2, true>(mode, bsync, P, A, threads, smem, st);
    if (gs == 4) return launch_particle_map<4, 1, true>(mode, bsync, P, A, threads, smem, st);
    return launch_particle_map<8, 1, true>(mode, bsync, P, A, threads, smem, st);
}

}  // namespace tamp
