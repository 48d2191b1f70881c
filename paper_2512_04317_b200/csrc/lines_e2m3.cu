// Instantiations of the line kernel for E2M3; one
// translation unit per format and variant so the build compiles them in parallel.
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_e2m3(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    return disp_cpb<F_E2M3, false>(a, cpb, smem, st);
}
}  // namespace mxfft
