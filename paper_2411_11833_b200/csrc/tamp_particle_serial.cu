// tamp_particle_serial.cu -- instantiations of the serial mapping (one thread per particle, particle_serial.cuh)
#include "particle_serial.cuh"

namespace tamp {
void note_launch();

template <int MODE, bool SM>
static cudaError_t launch_serial_t(const KProgram& P, const KArgs& A, int threads, cudaStream_t st) {
    auto fn = k_serial<MODE, SM>;
    const size_t smem = serial_smem_bytes(P, threads, MODE == MODE_OPT);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (A.n + threads - 1) / threads;
    fn<<<(unsigned)blocks, threads, smem, st>>>(P, A);
    note_launch();
    return cudaGetLastError();
}

template <bool SM>
static cudaError_t launch_serial_m(int mode, const KProgram& P, const KArgs& A, int threads, cudaStream_t st) {
    if (mode == MODE_EVAL) return launch_serial_t<MODE_EVAL, SM>(P, A, threads, st);
    if (mode == MODE_CHECK) return launch_serial_t<MODE_CHECK, SM>(P, A, threads, st);
    return launch_serial_t<MODE_OPT, SM>(P, A, threads, st);
}

cudaError_t launch_particle_serial(bool smooth, int mode, int threads, const KProgram& P, const KArgs& A,
                                   cudaStream_t st) {
    if (A.n <= 0) return cudaSuccess;
    return smooth ? launch_serial_m<true>(mode, P, A, threads, st) : launch_serial_m<false>(mode, P, A, threads, st);
}

int serial_kernel_regs() {
    static int cached = 0;
    if (cached) return cached;
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, k_serial<MODE_OPT, false>) != cudaSuccess) { cudaGetLastError(); return 128; }
    cached = a.numRegs;
    return cached;
}

}  // namespace tamp
