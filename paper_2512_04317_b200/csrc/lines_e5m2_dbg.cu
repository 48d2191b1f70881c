// Instantiations of the line kernel for E5M2 (debug-capture variant, n <= 4096); one
// translation unit per format and variant so the build compiles them in parallel.
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_e5m2_dbg(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    return disp_cpb<F_E5M2, true>(a, cpb, smem, st);
}
}  // namespace mxfft
