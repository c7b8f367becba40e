// FFT NK2 / NK4 codelets for t in {13, 14, 15, 16, 18, 20, 21} (fft_xforms.cuh).
#include "fft_xforms.cuh"

cudaError_t fc_fft_xform_b(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s,
                           int *handled) {
    *handled = 0;
    switch (g.t) {
        case 13: *handled = 1; return fcfft::launch_fft<13>(g, src, dst, forward, s);
        case 14: *handled = 1; return fcfft::launch_fft<14>(g, src, dst, forward, s);
        case 15: *handled = 1; return fcfft::launch_fft<15>(g, src, dst, forward, s);
        case 16: *handled = 1; return fcfft::launch_fft<16>(g, src, dst, forward, s);
        case 18: *handled = 1; return fcfft::launch_fft<18>(g, src, dst, forward, s);
        case 20: *handled = 1; return fcfft::launch_fft<20>(g, src, dst, forward, s);
        case 21: *handled = 1; return fcfft::launch_fft<21>(g, src, dst, forward, s);
    }
    return cudaSuccess;
}

cudaError_t fc_fft_twiddles_b() { return fct::upload_twiddles(); }
