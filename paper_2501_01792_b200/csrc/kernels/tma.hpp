// Host-side TMA descriptor encoding shared by the tcgen05 kernels (gemm.cu).
#pragma once
#include <cuda.h>

namespace hc {

// 2-D f16 tensor [rows x cols], row stride ld elements, box = box_rows x 64
// columns (one 128-byte row segment), 128B swizzle, OOB rows zero-filled.
CUtensorMap make_map(const void* ptr, long long rows, long long cols, long long ld, int box_rows);

}  // namespace hc
