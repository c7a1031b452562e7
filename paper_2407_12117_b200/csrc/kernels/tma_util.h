// tma_util.h — host-side TMA tensor-map construction (driver entry point is
// resolved at run time through the runtime, so libmemo does not link libcuda).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace memo {

// 2-D bf16 map over a row-major matrix: `inner` contiguous elements per row,
// `outer` rows, row pitch `ld_elems`; 128-byte swizzle, OOB reads are zero.
bool make_tma_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                      uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer);

int num_sms();

}  // namespace memo
