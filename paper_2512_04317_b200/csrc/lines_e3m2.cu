// Instantiations of the line kernel for E3M2 (split per format so the
// build compiles formats in parallel).
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_e3m2(const MxLinesArgs& a, int cpb, int nt, size_t smem, bool dbg,
                             cudaStream_t st) {
    return dbg ? disp_cpb<F_E3M2, true>(a, cpb, nt, smem, st) : disp_cpb<F_E3M2, false>(a, cpb, nt, smem, st);
}
}  // namespace mxfft
