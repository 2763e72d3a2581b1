// tamp_particle_hinge.cu -- k_particle with the hinge collision cost: 8 lanes, 768-thread bound (multi-wave
// launches) and 4 lanes (split from tamp_kernels.cu so the instantiations compile in parallel).
#include "particle_launch.cuh"

namespace tamp {

cudaError_t launch_particle_hinge_rich(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                       size_t smem, cudaStream_t st);
int particle_regs_hinge_rich(int gs);
cudaError_t launch_particle_hinge_wide(int mode, int bsync, int threads, const KProgram& P, const KArgs& A,
                                       size_t smem, cudaStream_t st);
int particle_regs_hinge_wide(int threads);
cudaError_t launch_particle_hinge_16(int mode, int bsync, int threads, const KProgram& P, const KArgs& A, size_t smem,
                                     cudaStream_t st);
int particle_regs_hinge_16();

// 16 lanes, and 8 lanes in blocks of <= 512 threads: the 512-thread-bound (register-rich) instantiations
cudaError_t launch_particle_hinge(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                  size_t smem, cudaStream_t st) {
    if (gs == 16 && threads > 512) return launch_particle_hinge_16(mode, bsync, threads, P, A, smem, st);
    if (gs == 16 || (gs == 8 && threads <= 512)) return launch_particle_hinge_rich(mode, gs, bsync, threads, P, A, smem, st);
    if (gs == 4) return launch_particle_map<4, 1, false, 512>(mode, bsync, P, A, threads, smem, st);
    if (threads > 768) return launch_particle_hinge_wide(mode, bsync, threads, P, A, smem, st);
    return launch_particle_map<8, 1, false, 768>(mode, bsync, P, A, threads, smem, st);
}

// registers per thread of the variant a block of `threads` threads would run (launch-configuration policy)
int particle_kernel_regs_sm(int gs, int threads) {
    if (gs == 16 && threads > 512) return particle_regs_hinge_16();
    if (gs == 16 || (gs == 8 && threads <= 512)) return particle_regs_hinge_rich(gs);
    if (gs == 4) return particle_regs_t<4, 1, false, 512>();
    if (threads > 768) return particle_regs_hinge_wide(threads);
    return particle_regs_t<8, 1, false, 768>();
}

cudaError_t launch_particle_smooth(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                                   size_t smem, cudaStream_t st);

cudaError_t launch_particle_sm(bool smooth, int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                               size_t smem, cudaStream_t st) {
    return smooth ? launch_particle_smooth(mode, gs, bsync, threads, P, A, smem, st)
                  : launch_particle_hinge(mode, gs, bsync, threads, P, A, smem, st);
}

}  // namespace tamp
