// Kernel launch with programmatic dependent launch (PDL) on sm_100a.
//
// Every stage kernel starts with pdl_begin(): griddepcontrol.wait (block until
// the previous kernel in the stream has completed and its writes are visible)
// followed by griddepcontrol.launch_dependents (let the next kernel launch).
// The next kernel's CTAs are therefore scheduled as soon as every CTA of this
// one is resident, run their prologue (barrier init, TMEM alloc, tensor-map
// prefetch) on SMs freed by this kernel's tail, and wait for completion before
// touching memory — the kernel-boundary drain/launch gap disappears without
// changing any ordering.  PTK_PDL=0 disables the attribute (plain stream order).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace ptk {

__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PTK_PDL");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}

// cluster_x > 1: thread-block cluster of that many CTAs along x.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    unsigned n = 0;
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace ptk
