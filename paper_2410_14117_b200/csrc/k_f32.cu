// fp32 instantiation of the engine kernels (the product path).
#define UUV_F32_TU 1   // defines launch_band (the band kernel's FMA-formulation instantiations)
#include "uuv_kernels.cuh"
#include "uuv_common_kernels.cuh"

UUV_INSTANTIATE(float)

#ifdef UUV_BAND_CLOCK
// A/B builds only: copy the timeline table out (and clear it)
extern "C" int uuvsim_debug_timeline(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, g_uuv_tl, sizeof(g_uuv_tl)) != cudaSuccess) return -1;
    static unsigned long long zero[TL_ROWS][TL_BLOCKS];
    cudaMemcpyToSymbol(g_uuv_tl, zero, sizeof(g_uuv_tl));
    return TL_ROWS * TL_BLOCKS;
}
#endif
