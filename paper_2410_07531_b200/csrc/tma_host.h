#pragma once
#include <cuda.h>

#include <cstdint>

namespace rgo {

// rank-N tiled tensor map; dims[0] is the contiguous dimension, strides_bytes
// has rank-1 entries (stride of dims[1..]).
bool make_tmap(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint32_t rank,
               const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
               CUtensorMapSwizzle swizzle);

}  // namespace rgo
