// tma.cpp -- CUtensorMap encoding through the runtime-resolved driver entry point.
#include "tma.hpp"

#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

namespace spx {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 resolve_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        }
    });
    return fn;
}

}  // namespace

bool make_tma_map_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, char* err,
                       size_t err_len) {
    return make_tma_map_bf16_swizzle(map, base, rank, dims, strides_bytes, box, 128, err, err_len);
}

bool make_tma_map_bf16_swizzle(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                               const uint64_t* strides_bytes, const uint32_t* box, int swizzle_bytes,
                               char* err, size_t err_len) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = resolve_encode();
    if (!encode) {
        std::snprintf(err, err_len, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
        return false;
    }
    cuuint64_t gdim[5];
    cuuint64_t gstride[4];
    cuuint32_t bdim[5];
    cuuint32_t estride[5];
    for (int i = 0; i < rank; ++i) {
        gdim[i] = dims[i];
        bdim[i] = box[i];
        estride[i] = 1;
        if (i + 1 < rank) gstride[i] = strides_bytes[i];
    }
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<cuuint32_t>(rank),
                        const_cast<void*>(base), gdim, gstride, bdim, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::snprintf(err, err_len,
                      "cuTensorMapEncodeTiled failed (%d): rank %d dims [%llu %llu %llu] box "
                      "[%u %u %u] base %p",
                      static_cast<int>(r), rank, (unsigned long long)dims[0],
                      (unsigned long long)(rank > 1 ? dims[1] : 0),
                      (unsigned long long)(rank > 2 ? dims[2] : 0), box[0],
                      rank > 1 ? box[1] : 0, rank > 2 ? box[2] : 0, base);
        return false;
    }
    return true;
}

}  // namespace spx
