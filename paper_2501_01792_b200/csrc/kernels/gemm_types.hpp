// Host-visible constants of the tcgen05 GEMM (gemm.cuh).
#pragma once

namespace hc::gemm {

// kSplitF32: split-K partials (fp32, [splits][M][N]) reduced by splitk_reduce
// kAttnPart: recompute fused with decode attention (gemm.cuh, attn_part_tile)
enum Epi : int { kStore = 0, kRelu = 1, kKvPaged = 2, kF32 = 3, kSplitF32 = 4, kAttnPart = 5 };

constexpr int BM = 128;  // rows per M tile (UMMA M)
constexpr int BK = 64;   // K per pipeline stage (one 128-byte swizzle atom of f16)

}  // namespace hc::gemm
