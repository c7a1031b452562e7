// tma_util.h — host-side TMA tensor-map construction (driver entry point is
// resolved at run time through the runtime, so libmemo does not link libcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace memo {

// 2-D bf16 map over a row-major matrix: `inner` contiguous elements per row,
// `outer` rows, row pitch `ld_elems`; 128-byte swizzle, OOB reads are zero.
bool make_tma_2d_bf16(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                      uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer);

int num_sms();

// Timing events: a plain record on an eager stream; while the stream is being
// captured into a CUDA graph, an external record node, so the graph replays
// the record and cudaEventElapsedTime keeps working on it.
inline cudaError_t record_timing_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}

}  // namespace memo
