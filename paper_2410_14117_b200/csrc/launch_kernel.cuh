// launch_kernel.cuh -- one launch helper for every .cu translation unit:
// <<<>>> launch, or cudaLaunchKernelEx with programmatic stream serialisation
// (the kernel then starts while its predecessor on the stream finishes and
// waits in griddepcontrol.wait before touching anything that predecessor writes).
#pragma once

#include <cuda_runtime.h>

namespace uuv {

template <class... KArgs, class... Args>
static cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, bool pdl, Args... args) {
    if (!pdl) {
        k<<<grid, block, smem, st>>>(args...);
        return cudaSuccess;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

}  // namespace uuv
