// FFT NK2 / NK4 codelets for t in {24, 25, 27, 28, 30, 31, 32} (fft_xforms.cuh).
#include "fft_xforms.cuh"

cudaError_t fc_fft_xform_c(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s,
                           int *handled) {
    *handled = 0;
    switch (g.t) {
        case 24: *handled = 1; return fcfft::launch_fft<24>(g, src, dst, forward, s);
        case 25: *handled = 1; return fcfft::launch_fft<25>(g, src, dst, forward, s);
        case 27: *handled = 1; return fcfft::launch_fft<27>(g, src, dst, forward, s);
        case 28: *handled = 1; return fcfft::launch_fft<28>(g, src, dst, forward, s);
        case 30: *handled = 1; return fcfft::launch_fft<30>(g, src, dst, forward, s);
        case 31: *handled = 1; return fcfft::launch_fft<31>(g, src, dst, forward, s);
        case 32: *handled = 1; return fcfft::launch_fft<32>(g, src, dst, forward, s);
    }
    return cudaSuccess;
}

cudaError_t fc_fft_twiddles_c() { return fct::upload_twiddles(); }
