// fp64 instantiation (parity / precision mode). Compiled with -fmad=false so
// every expression rounds exactly as the reference's scalar fp64 code.
#include "uuv_kernels.cuh"

UUV_INSTANTIATE(double)
