// The fp64 band kernel's reference-operation-order instantiations (uuv_kernels.cuh
// k_band<..., REFOP = true>, EngineP::band_refop, DESIGN.md §4a / §6) in their own
// translation unit, compiled with -fmad=false: substep_ref then rounds exactly
// like the reference's scalar fp64 code.  The FMA-formulation band kernel (the
// default) is instantiated in k_f32.cu.
#define UUV_BAND_TU 1
#include "uuv_kernels.cuh"
