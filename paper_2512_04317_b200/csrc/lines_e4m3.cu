// Instantiations of the line kernel for E4M3 (split per format so the
// build compiles formats in parallel).
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_e4m3(const MxLinesArgs& a, int cpb, int nt, size_t smem, bool dbg,
                             cudaStream_t st) {
    return dbg ? disp_cpb<F_E4M3, true>(a, cpb, nt, smem, st) : disp_cpb<F_E4M3, false>(a, cpb, nt, smem, st);
}
}  // namespace mxfft
