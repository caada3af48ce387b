// Host-side helpers shared by the C-ABI entry points: error reporting
// (thread-local last error, the `int` status convention of include/specexec_b200.h)
// and TMA tensor-map creation through the driver entry point (no -lcuda link).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

namespace sx {

// status codes: 0 ok, <0 argument error (Python raises ValueError),
// >0 a cudaError_t (Python raises RuntimeError).
constexpr int SX_OK = 0;
constexpr int SX_EARG = -1;
constexpr int SX_ECAP = -2;  // capacity exceeded (workspace too small)

void set_last_error(const std::string& msg);
const char* get_last_error();

int arg_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

// 2D row-major bf16 matrix [rows, cols] (cols contiguous, row pitch `ld`
// elements) -> tensor map with a {64, box_rows} box and 128B swizzle.
// Cached by (ptr, rows, cols, ld, box_rows).
// Raise a kernel's dynamic shared-memory limit to `bytes` on the CURRENT device
// (the attribute is per device: one process may drive several GPUs, e.g.
// tensor-parallel thread-ranks). Thread-safe; a no-op once set at >= bytes.
int ensure_smem_attr(const void* fn, int bytes);

int make_tmap_bf16_kmajor(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                          int box_rows);

}  // namespace sx

namespace sx {
// kernels launched through the C ABI since load (bench.py reports it as gpu_launches)
void count_launch();
}  // namespace sx

#define SX_CHECK_LAUNCH(where)                                  \
  do {                                                          \
    ::sx::count_launch();                                       \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::sx::cuda_status(_e, where); \
  } while (0)
