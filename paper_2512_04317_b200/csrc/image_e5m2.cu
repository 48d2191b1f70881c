// Instantiations of the fused small-image kernel (mxfft_image.cuh) for E5M2;
// one translation unit per format so the build compiles them in parallel.
#include "mxfft_image.cuh"

namespace mxfft {
cudaError_t run_mx_image_e5m2(const ImageArgs& a, int cpb, size_t smem, int grid, cudaStream_t st) {
    void (*k)(ImageArgs) = nullptr;
    switch (cpb) {
        case 8: k = k_mx_image<F_E5M2, 8>; break;
        case 16: k = k_mx_image<F_E5M2, 16>; break;
        case 32: k = k_mx_image<F_E5M2, 32>; break;
        default: return cudaErrorInvalidValue;
    }
    cudaError_t e = ensure_smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, IM_NT, smem, st>>>(a);  // (programmatic dependent launch measured +0.8 % here: off)
    note_launch();
    return cudaGetLastError();
}
}  // namespace mxfft
