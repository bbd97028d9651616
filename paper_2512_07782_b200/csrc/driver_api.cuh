// driver_api.cuh -- CUDA driver entry points resolved at run time through the
// runtime (cudaGetDriverEntryPoint), so libgfwa.so has no link-time dependency
// on libcuda.so.1 and loads on machines without a driver (the CPU test suite
// checks its exported symbols there).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace gfwa {
namespace drv {

template <typename Fn>
inline Fn resolve(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<Fn>(fn);
}

inline CUresult tensorMapEncodeTiled(CUtensorMap* map, CUtensorMapDataType dt, cuuint32_t rank, void* addr,
                                     const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                                     const cuuint32_t* estr, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                                     CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = resolve<Fn>("cuTensorMapEncodeTiled");
    if (!fn) return CUDA_ERROR_NOT_FOUND;
    return fn(map, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
}

inline CUresult ctxGetCurrent(CUcontext* c) {
    using Fn = CUresult (*)(CUcontext*);
    static Fn fn = resolve<Fn>("cuCtxGetCurrent");
    return fn ? fn(c) : CUDA_ERROR_NOT_FOUND;
}

inline CUresult ctxSetCurrent(CUcontext c) {
    using Fn = CUresult (*)(CUcontext);
    static Fn fn = resolve<Fn>("cuCtxSetCurrent");
    return fn ? fn(c) : CUDA_ERROR_NOT_FOUND;
}

inline CUresult pointerGetAttribute(void* data, CUpointer_attribute attr, CUdeviceptr ptr) {
    using Fn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
    static Fn fn = resolve<Fn>("cuPointerGetAttribute");
    return fn ? fn(data, attr, ptr) : CUDA_ERROR_NOT_FOUND;
}

}  // namespace drv
}  // namespace gfwa
