// tamp_particle_hinge_wide.cu -- k_particle with the hinge collision cost, 8 lanes, blocks of more than 768 threads:
// 896-thread bound (<= 72 registers) and 1024-thread bound (<= 64 registers).  One large block per SM holds up to
// 111 / 128 particles, so a multi-wave launch needs fewer waves (config 3 at 32,768 particles: 2 waves of 111
// particles per SM instead of 3 of 74); split into its own translation unit so it compiles in parallel.
#include "particle_launch.cuh"

namespace tamp {

cudaError_t launch_particle_hinge_wide(int mode, int bsync, int threads, const KProgram& P, const KArgs& A,
                                       size_t smem, cudaStream_t st) {
    if (threads > 896) return launch_particle_map<8, 1, false, 1024>(mode, bsync, P, A, threads, smem, st);
    return launch_particle_map<8, 1, false, 896>(mode, bsync, P, A, threads, smem, st);
}

int particle_regs_hinge_wide(int threads) {
    return threads > 896 ? particle_regs_t<8, 1, false, 1024>() : particle_regs_t<8, 1, false, 896>();
}

}  // namespace tamp
