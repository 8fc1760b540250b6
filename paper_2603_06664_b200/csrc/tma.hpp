// tma.hpp -- host-side construction of TMA tensor maps (CUtensorMap) without linking libcuda:
// the driver entry point is resolved through the runtime (cudaGetDriverEntryPoint).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace spx {

// Tiled bf16 tensor map, SWIZZLE_128B, OOB elements read as zero.
//   dims[0] is the contiguous dimension; strides_bytes[i] is the byte stride of dims[i+1].
// Returns false (and fills err) when the driver rejects the map.
bool make_tma_map_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, char* err,
                       size_t err_len);
// the same with SWIZZLE_64B (swizzle_bytes = 64: 32-element boxes) or SWIZZLE_128B (128)
bool make_tma_map_bf16_swizzle(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                               const uint64_t* strides_bytes, const uint32_t* box, int swizzle_bytes,
                               char* err, size_t err_len);

}  // namespace spx
