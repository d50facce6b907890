// tma_host.h -- encode TMA tensor maps of complex64 (8-byte element) arrays.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace dc {
// rank <= 5; dims innermost first; strides_bytes has rank-1 entries (multiples of 16); box <= 256 each.
bool encode_tile_map(CUtensorMap *m, const void *base, int rank, const uint64_t *dims, const uint64_t *strides_bytes,
                     const uint32_t *box, CUtensorMapSwizzle swizzle);
}  // namespace dc
