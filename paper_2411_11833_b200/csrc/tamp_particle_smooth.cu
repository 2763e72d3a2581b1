// tamp_particle_smooth.cu -- k_particle with the CHOMP-smooth collision cost: 8 lanes (768-thread
// bound), 16 and 4 lanes (512).  Compiled in its own translation unit, in parallel with the hinge variants.
#include "particle_launch.cuh"

namespace tamp {

cudaError_t launch_particle_smooth(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                   size_t smem, cudaStream_t st) {
    if (gs == 16) return launch_particle_map<8, 2, true, 512>(mode, bsync, P, A, threads, smem, st);
    if (gs == 4) return launch_particle_map<4, 1, true, 512>(mode, bsync, P, A, threads, smem, st);
    return launch_particle_map<8, 1, true, 768>(mode, bsync, P, A, threads, smem, st);
}

}  // namespace tamp
