// tamp_particle_hinge_rich.cu -- k_particle with the hinge collision cost, 512-thread launch bound (<= 128
// registers): 8 lanes in blocks of <= 512 threads (single-wave launches) and the 16-lane mapping.
#include "particle_launch.cuh"

namespace tamp {

cudaError_t launch_particle_hinge_rich(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                       size_t smem, cudaStream_t st) {
    if (gs == 16) return launch_particle_map<8, 2, false, 512>(mode, bsync, P, A, threads, smem, st);
    return launch_particle_map<8, 1, false, 512>(mode, bsync, P, A, threads, smem, st);
}

int particle_regs_hinge_rich(int gs) {
    return gs == 16 ? particle_regs_t<8, 2, false, 512>() : particle_regs_t<8, 1, false, 512>();
}

}  // namespace tamp
