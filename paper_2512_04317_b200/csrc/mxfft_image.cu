// mxfft_image.cu -- dispatch of the fused small-image pipeline (kernels in
// mxfft_image.cuh, instantiated per element format in image_<fmt>.cu).
#include "mxfft_image.cuh"

namespace mxfft {

cudaError_t run_mx_image_e4m3(const ImageArgs&, int, size_t, int, cudaStream_t);
cudaError_t run_mx_image_e5m2(const ImageArgs&, int, size_t, int, cudaStream_t);
cudaError_t run_mx_image_e2m3(const ImageArgs&, int, size_t, int, cudaStream_t);
cudaError_t run_mx_image_e3m2(const ImageArgs&, int, size_t, int, cudaStream_t);
cudaError_t run_mx_image_e2m1(const ImageArgs&, int, size_t, int, cudaStream_t);

int g_fused_image = -1;  // -1 automatic (mxfft_fft2), 0 line passes, 1 fused image kernel

bool mx_image_ok(const Plan& p) {
    return p.n == IM_N && p.fmt.id != F_GENERIC && (p.cpb == 8 || p.cpb == 16 || p.cpb == 32);
}

cudaError_t run_mx_image(const Plan& p, const void* x, void* y, int64_t nimg, int mode,
                         const mxfft_prescale_cfg& cfg, mxfft_prescale_result* res, int32_t* kvec,
                         const int32_t* kin, int k_group, cudaStream_t st) {
    if (nimg <= 0) return cudaSuccess;
    ImageArgs a{};
    a.in = reinterpret_cast<const float2*>(x);
    a.out = reinterpret_cast<float2*>(y);
    a.nimg = nimg;
    a.npass = mode == 2 ? 4 : 2;
    a.first_inverse = mode == 1;
    a.kin = kin;
    a.stats = res != nullptr;
    a.k_group = k_group > 0 ? k_group : 1;
    a.tw_fwd = p.d_tw16_fwd;
    a.tw_inv = p.d_tw16_inv;
    a.twe = p.d_twe8;
    a.trivial01 = p.trivial01;
    a.cfg = cfg;
    a.q = cfg.tau / 100.0;
    a.res = res;
    a.kvec = kvec;
    a.fmt = p.fmt;
    a.cpb = p.cpb;
    a.wcr = p.d_wcr;
    a.wci = p.d_wci;
    a.wsexp = p.d_wsexp;
    // twiddles first; the tile on a 4 KB boundary of the shared window
    // (dynamic shared memory starts after the per-block reserved area)
    const int reserved = device_attr(cudaDevAttrReservedSharedMemoryPerBlock);
    int off = 2 * IM_N * 4 + IM_N;
    off = ((reserved + off + 4095) / 4096) * 4096 - reserved;
    a.tile_off = off;
    const size_t smem = (size_t)off + (size_t)IM_EL * 8 + sizeof(ImStats);
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    const int grid = (int)(nimg < sms ? nimg : sms);
    switch (p.fmt.id) {
        case F_E4M3: return run_mx_image_e4m3(a, p.cpb, smem, grid, st);
        case F_E5M2: return run_mx_image_e5m2(a, p.cpb, smem, grid, st);
        case F_E2M3: return run_mx_image_e2m3(a, p.cpb, smem, grid, st);
        case F_E3M2: return run_mx_image_e3m2(a, p.cpb, smem, grid, st);
        case F_E2M1: return run_mx_image_e2m1(a, p.cpb, smem, grid, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mxfft
