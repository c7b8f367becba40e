// FFT NK2 / NK4 codelets for t in {4, 5, 6, 7, 8, 9, 10, 12} (fft_xforms.cuh).
#include "fft_xforms.cuh"

cudaError_t fc_fft_xform_a(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s,
                           int *handled) {
    *handled = 0;
    switch (g.t) {
        case 4: *handled = 1; return fcfft::launch_fft<4>(g, src, dst, forward, s);
        case 5: *handled = 1; return fcfft::launch_fft<5>(g, src, dst, forward, s);
        case 6: *handled = 1; return fcfft::launch_fft<6>(g, src, dst, forward, s);
        case 7: *handled = 1; return fcfft::launch_fft<7>(g, src, dst, forward, s);
        case 8: *handled = 1; return fcfft::launch_fft<8>(g, src, dst, forward, s);
        case 9: *handled = 1; return fcfft::launch_fft<9>(g, src, dst, forward, s);
        case 10: *handled = 1; return fcfft::launch_fft<10>(g, src, dst, forward, s);
        case 12: *handled = 1; return fcfft::launch_fft<12>(g, src, dst, forward, s);
    }
    return cudaSuccess;
}

cudaError_t fc_fft_twiddles_a() { return fct::upload_twiddles(); }
