// The statistics-folding first pass of mxfft_pipeline_folded (k_mx_lines_tma<.., ACC = true>)
// for E2M1; its own translation unit so the build compiles the formats in parallel.
#include "mxfft_lines.cuh"

namespace mxfft {
cudaError_t run_mx_lines_acc_e2m1(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    return disp_acc<F_E2M1>(a, cpb, smem, st);
}
}  // namespace mxfft
