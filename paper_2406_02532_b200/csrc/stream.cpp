// KS: stage 3, the offloaded-weight path. Per-layer weights live in pinned host
// memory and are streamed into device staging buffers on a dedicated copy
// stream (copy engines, PCIe), double-buffered against the compute stream:
//
//   copy stream : wait(buffer b free) -> memcpyAsync(layer l -> buffer b) -> record(l ready)
//   compute     : wait(l ready) -> layer l kernels -> record(buffer b free)
//
// No reference counterpart exists: the reference only models this analytically
// (costsim.forward_time, pkg/src/speckit/costsim.py:59-65); bench.py reports the
// achieved host-link GB/s against that model and the measured pinned-H2D peak.
#include "capi_util.h"
#include "specexec_b200.h"

extern "C" int sx_stream_copy(void* dst, const void* src, long long bytes, int to_device, cudaStream_t stream,
                              cudaEvent_t wait_event, cudaEvent_t done_event) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return sx::arg_error("sx_stream_copy: bad buffer");
  cudaError_t e;
  if (wait_event) {
    e = cudaStreamWaitEvent(stream, wait_event, 0);
    if (e != cudaSuccess) return sx::cuda_status(e, "sx_stream_copy: wait");
  }
  if (bytes > 0) {
    e = cudaMemcpyAsync(dst, src, (size_t)bytes, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                        stream);
    if (e != cudaSuccess) return sx::cuda_status(e, "sx_stream_copy: memcpy");
  }
  if (done_event) {
    e = cudaEventRecord(done_event, stream);
    if (e != cudaSuccess) return sx::cuda_status(e, "sx_stream_copy: record");
  }
  return sx::SX_OK;
}
