// The statistics-folding first pass of mxfft_pipeline_folded (k_mx_lines_tma<.., ACC = true>)
// for E3M2; its own translation unit so the build compiles the formats in parallel.
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_acc_e3m2(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    return disp_acc<F_E3M2>(a, cpb, smem, st);
}
}  // namespace mxfft
