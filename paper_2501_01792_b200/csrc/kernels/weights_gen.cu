// DecoderWeights::generate on the GPU (model.cpp:82-117 + the rescale +
// fp64 -> fp32 -> f16 rounding of csrc/host/model.cpp), bit-exact with the
// host generator: SplitMix64 is counter based (draw i of stream s is
// mix(s + (i+1)*golden)), so every output element is computed independently.
// Each thread produces one element of the TRANSPOSED matrix ([cols][rows]),
// which keeps the stores coalesced. fp64 arithmetic uses explicit _rn
// intrinsics so no FMA contraction changes the rounding vs the host.
#include "kernels.hpp"

namespace hc {

namespace {

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t f16_bits_rn(double v) {
    return __half_as_ushort(__float2half_rn(__double2float_rn(v)));
}

__device__ __forceinline__ double draw_u(uint64_t seed, uint64_t i) {
    const uint64_t z = splitmix_mix(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
    const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    // lo + (hi - lo) * u with lo = -0.1, hi = 0.1 (rng.hpp:23)
    return __dadd_rn(-0.1, __dmul_rn(__dadd_rn(0.1, 0.1), u));
}

// dst[c * rows + r] = f16(scale * U_{r*cols + c})
__global__ void gen_transposed_kernel(uint16_t* __restrict__ dst, int rows, int cols, uint64_t seed, double scale,
                                      int apply_scale) {
    const size_t n = static_cast<size_t>(rows) * cols;
    for (size_t o = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; o < n;
         o += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t c = o / rows, r = o - c * rows;
        double v = draw_u(seed, r * static_cast<size_t>(cols) + c);
        if (apply_scale) v = __dmul_rn(v, scale);
        dst[o] = f16_bits_rn(v);
    }
}

__global__ void gen_plain_kernel(uint16_t* __restrict__ dst, size_t n, uint64_t seed) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] = f16_bits_rn(draw_u(seed, i));
}

}  // namespace

void gen_weights_transposed(uint16_t* dst, int rows, int cols, uint64_t seed, double scale, bool apply_scale,
                            cudaStream_t st) {
    if (rows > 0 && cols > 0)
        gen_transposed_kernel<<<8 * num_sms(), 256, 0, st>>>(dst, rows, cols, seed, scale, apply_scale ? 1 : 0);
}

void gen_weights_plain(uint16_t* dst, size_t n, uint64_t seed, cudaStream_t st) {
    if (n) gen_plain_kernel<<<8 * num_sms(), 256, 0, st>>>(dst, n, seed);
}

}  // namespace hc
