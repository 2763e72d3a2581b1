// tamp_particle_serial.cu -- instantiations of the serial mapping (one thread per particle, particle_serial.cuh)
#include "particle_serial.cuh"

#ifndef TAMP_SERIAL_PP   // 0: the generic sweep for every program (A/B builds)
#define TAMP_SERIAL_PP 1
#endif

namespace tamp {
void note_launch();

template <int MODE, bool SM, bool PP>
static cudaError_t launch_serial_t(const KProgram& P, const KArgs& A, int threads, cudaStream_t st) {
    auto fn = k_serial<MODE, SM, PP>;
    const size_t smem = serial_smem_bytes(P, threads, MODE == MODE_OPT);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (A.n + threads - 1) / threads;
    fn<<<(unsigned)blocks, threads, smem, st>>>(P, A);
    note_launch();
    return cudaGetLastError();
}

template <bool SM, bool PP>
static cudaError_t launch_serial_m(int mode, const KProgram& P, const KArgs& A, int threads, cudaStream_t st) {
    if (mode == MODE_EVAL) return launch_serial_t<MODE_EVAL, SM, PP>(P, A, threads, st);
    if (mode == MODE_CHECK) return launch_serial_t<MODE_CHECK, SM, PP>(P, A, threads, st);
    return launch_serial_t<MODE_OPT, SM, PP>(P, A, threads, st);
}

cudaError_t launch_particle_serial(bool smooth, int mode, int threads, const KProgram& P, const KArgs& A,
                                   cudaStream_t st) {
    if (A.n <= 0) return cudaSuccess;
    // pick-place class programs (serial_program_pp): the unrolled one-box link sweep; the smooth variant keeps the
    // generic sweep
    if (TAMP_SERIAL_PP && !smooth && serial_program_pp(P)) return launch_serial_m<false, true>(mode, P, A, threads, st);
    return smooth ? launch_serial_m<true, false>(mode, P, A, threads, st) : launch_serial_m<false, false>(mode, P, A, threads, st);
}

int serial_kernel_regs(bool pp) {
    static int cached[2] = {0, 0};
    if (cached[pp]) return cached[pp];
    cudaFuncAttributes a;
    const void* fn = pp ? (const void*)k_serial<MODE_OPT, false, true> : (const void*)k_serial<MODE_OPT, false, false>;
    if (cudaFuncGetAttributes(&a, fn) != cudaSuccess) {
        cudaGetLastError();
        return 128;
    }
    cached[pp] = a.numRegs;
    return cached[pp];
}

}  // namespace tamp
