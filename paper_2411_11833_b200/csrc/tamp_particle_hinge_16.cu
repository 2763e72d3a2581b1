// tamp_particle_hinge_16.cu -- k_particle with the hinge collision cost, 16 lanes (two FK instances at a time),
// blocks of more than 512 threads: the 768-thread bound (<= 80 registers, no spills), so a knot-heavy skeleton
// (config 4) keeps more resident warps per SM.  Own translation unit: compiles in parallel with the others.
#include "particle_launch.cuh"

namespace tamp {

cudaError_t launch_particle_hinge_16(int mode, int bsync, int threads, const KProgram& P, const KArgs& A, size_t smem,
                                     cudaStream_t st) {
    return launch_particle_map<8, 2, false, 768>(mode, bsync, P, A, threads, smem, st);
}

int particle_regs_hinge_16() { return particle_regs_t<8, 2, false, 768>(); }

}  // namespace tamp
