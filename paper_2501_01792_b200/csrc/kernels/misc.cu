// Small HBM-bound kernels of the path: embedding gather, the activation-cache
// writer / KV append for decode tokens, prefill block scatter, argmax.
// All move 16-byte vectors; one CTA per row / block.
#include <algorithm>
#include <cfloat>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"

namespace hc {

namespace {

__global__ void embed_kernel(const f16* __restrict__ E, const f16* __restrict__ Pos, const int* __restrict__ ids,
                             const int* __restrict__ pos, int d, f16* __restrict__ X, long long ldx) {
    const int r = blockIdx.x;
    const f16* e = E + static_cast<long long>(ids[r]) * d;
    const f16* p = Pos + static_cast<long long>(pos[r]) * d;
    f16* x = X + r * ldx;
    for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
        const uint4 a = *reinterpret_cast<const uint4*>(e + c);
        const uint4 b = *reinterpret_cast<const uint4*>(p + c);
        const __half2* ha = reinterpret_cast<const __half2*>(&a);
        const __half2* hb = reinterpret_cast<const __half2*>(&b);
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 fa = __half22float2(ha[i]), fb = __half22float2(hb[i]);
            o[i] = ptx::pack_f16x2(fa.x + fb.x, fa.y + fb.y);
        }
        *reinterpret_cast<uint4*>(x + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__device__ __forceinline__ f16* ref_ptr(f16* const* region, int ref, long long block_elems) {
    return region[ref >> 28] + static_cast<long long>(ref & 0x0FFFFFFF) * block_elems;
}

// one CTA per request: X row -> ACT block row (device and/or host pool)
__global__ void act_append_kernel(const AppendCall c) {
    const int b = blockIdx.x;
    const int refs[2] = {c.dev_ref ? c.dev_ref[b] : -1, c.host_ref ? c.host_ref[b] : -1};
    const int t = c.tok[b];
    const long long block_elems = static_cast<long long>(c.tpb) * c.d;
    const f16* src = c.src + b * c.ld;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (refs[k] < 0) continue;
        f16* dst = ref_ptr(c.region, refs[k], block_elems) + static_cast<long long>(t) * c.d;
        for (int x = threadIdx.x * 8; x < c.d; x += blockDim.x * 8)
            *reinterpret_cast<uint4*>(dst + x) = *reinterpret_cast<const uint4*>(src + x);
    }
}

// one CTA per request: K|V of the new token -> its KV block slot
__global__ void kv_append_kernel(const AppendCall c) {
    const int b = blockIdx.x;
    const int refs[2] = {c.dev_ref ? c.dev_ref[b] : -1, c.host_ref ? c.host_ref[b] : -1};
    const int t = c.tok[b];
    const long long block_elems = 2LL * c.tpb * c.d;
    const f16* src = c.src + b * c.ld + c.d;  // K at +d, V at +2d
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (refs[k] < 0) continue;
        f16* blk = ref_ptr(c.region, refs[k], block_elems);
        for (int x = threadIdx.x * 8; x < 2 * c.d; x += blockDim.x * 8) {
            const int part = x / c.d;
            const int rem = x - part * c.d;
            const int h = rem / c.hd;
            const int cc = rem - h * c.hd;
            f16* dst = blk + static_cast<long long>(part) * c.d * c.tpb + static_cast<long long>(h) * c.tpb * c.hd +
                        t * c.hd + cc;
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src + x);
        }
    }
}

// one CTA per block
__global__ void scatter_act_kernel(const BlockScatter c) {
    const int i = blockIdx.x;
    const int n = c.n_tok[i];
    const long long block_elems = static_cast<long long>(c.tpb) * c.d;
    f16* blk = ref_ptr(c.region, c.dst_ref[i], block_elems);
    const f16* src = c.src + static_cast<long long>(c.src_row[i]) * c.ld;
    const int per_row = c.d / 8;
    // rows past n_tok (a partial last block) are zeroed: the block's bytes
    // are deterministic wherever they are copied (HBM staging -> pinned host)
    for (int idx = threadIdx.x; idx < c.tpb * per_row; idx += blockDim.x) {
        const int t = idx / per_row, x = (idx - t * per_row) * 8;
        *reinterpret_cast<uint4*>(blk + static_cast<long long>(t) * c.d + x) =
            t < n ? *reinterpret_cast<const uint4*>(src + t * c.ld + x) : make_uint4(0, 0, 0, 0);
    }
}

__global__ void scatter_kv_kernel(const BlockScatter c) {
    const int i = blockIdx.x;
    const int n = c.n_tok[i];
    const long long block_elems = 2LL * c.tpb * c.d;
    f16* blk = ref_ptr(c.region, c.dst_ref[i], block_elems);
    const f16* src = c.src + static_cast<long long>(c.src_row[i]) * c.ld + c.d;
    // destination-major walk: consecutive threads write consecutive 16 B of a
    // head's [tpb][hd] run
    const int chunks_per_head = c.tpb * c.hd / 8;
    const int total = 2 * (c.d / c.hd) * chunks_per_head;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int ph = idx / chunks_per_head;     // part*H + head
        const int w = idx - ph * chunks_per_head;
        const int t = (w * 8) / c.hd;
        const int cc = (w * 8) - t * c.hd;
        const int part = ph / (c.d / c.hd);
        const int h = ph - part * (c.d / c.hd);
        const uint4 v = t < n ? *reinterpret_cast<const uint4*>(src + t * c.ld + part * c.d + h * c.hd + cc)
                              : make_uint4(0, 0, 0, 0);  // unfilled slots of a partial block
        *reinterpret_cast<uint4*>(blk + static_cast<long long>(ph) * c.tpb * c.hd + t * c.hd + cc) = v;
    }
}

__global__ void argmax_kernel(const float* __restrict__ logits, int V, int* __restrict__ out) {
    const int b = blockIdx.x;
    const float* row = logits + static_cast<long long>(b) * V;
    float best = -FLT_MAX;
    int arg = 0;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const float v = row[i];
        if (v > best) {
            best = v;
            arg = i;
        }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    for (int o = 16; o >= 1; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ov > best || (ov == best && oi < arg)) {
            best = ov;
            arg = oi;
        }
    }
    const int w = threadIdx.x / 32;
    if (threadIdx.x % 32 == 0) {
        sv[w] = best;
        si[w] = arg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x / 32); ++k)
            if (sv[k] > best || (sv[k] == best && si[k] < arg)) {
                best = sv[k];
                arg = si[k];
            }
        out[b] = arg;
    }
}

// 8 columns per thread; partial s of element (m, n) at ws[(s*M + m)*N + n]
// acc[0..8) += 8 consecutive f16 at src (16-byte aligned)
__device__ __forceinline__ void add8(float (&acc)[8], const f16* src) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(src));
    const __half2* h2 = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(h2[i]);
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
    }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, f16* __restrict__ out,
                                     int relu, const f16* __restrict__ bias, const f16* __restrict__ res,
                                     long long ldr) {
    const size_t n8 = static_cast<size_t>(M) * N / 8;
    const size_t plane = static_cast<size_t>(M) * N;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int s = 0; s < splits; ++s) {
            const float4* src = reinterpret_cast<const float4*>(ws + s * plane + i * 8);
            const float4 a = __ldg(src), b = __ldg(src + 1);
            acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
            acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
        }
        const size_t e0 = i * 8;
        const int col = static_cast<int>(e0 % N);
        if (bias) add8(acc, bias + col);
        if (res) add8(acc, res + static_cast<long long>(e0 / N) * ldr + col);
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float x = acc[2 * j], y = acc[2 * j + 1];
            if (relu) {
                x = fmaxf(x, 0.f);
                y = fmaxf(y, 0.f);
            }
            o[j] = ptx::pack_f16x2(x, y);
        }
        *reinterpret_cast<uint4*>(out + i * 8) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__global__ void fill_pattern_kernel(f16* dst, size_t n, uint64_t seed, float amp) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f);
        dst[i] = __float2half_rn(amp * (2.f * u - 1.f));
    }
}

// LayerNorm of one row per CTA (256 threads): the row stays in registers
// (8 f16 per 16-byte chunk, <= kLnChunks chunks per thread), two-pass fp32
// mean / variance with warp-shuffle + smem block reductions.
constexpr int kLnThreads = 256, kLnChunks = 8;  // d <= 16384

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();  // red[] reuse across calls
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = lane < kLnThreads / 32 ? red[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // every lane gets the total
    return t;
}

__global__ void __launch_bounds__(kLnThreads)
    layernorm_kernel(const f16* __restrict__ x, long long ldx, const f16* __restrict__ g,
                     const f16* __restrict__ b, f16* __restrict__ y, long long ldy, int d, float eps) {
    ptx::pdl_trigger();  // the FFN1 GEMM after LN2 may start streaming its weights
    __shared__ float red[kLnThreads / 32];
    const f16* xr = x + blockIdx.x * ldx;
    const int nch = d / 8;
    float v[kLnChunks][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kLnChunks; ++k) {
        const int ch = threadIdx.x + k * kLnThreads;
        if (ch < nch) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(xr) + ch);
            const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h[i]);
                v[k][2 * i] = f.x;
                v[k][2 * i + 1] = f.y;
                s += f.x + f.y;
            }
        }
    }
    const float mean = block_sum(s, red) / d;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kLnChunks; ++k)
        if (threadIdx.x + k * kLnThreads < nch)
#pragma unroll
            for (int i = 0; i < 8; ++i) q += (v[k][i] - mean) * (v[k][i] - mean);
    const float rstd = rsqrtf(block_sum(q, red) / d + eps);
    f16* yr = y + blockIdx.x * ldy;
#pragma unroll
    for (int k = 0; k < kLnChunks; ++k) {
        const int ch = threadIdx.x + k * kLnThreads;
        if (ch < nch) {
            const uint4 gu = __ldg(reinterpret_cast<const uint4*>(g) + ch);
            const uint4 bu = __ldg(reinterpret_cast<const uint4*>(b) + ch);
            const __half2* gh = reinterpret_cast<const __half2*>(&gu);
            const __half2* bh = reinterpret_cast<const __half2*>(&bu);
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 gf = __half22float2(gh[i]), bf = __half22float2(bh[i]);
                o[i] = ptx::pack_f16x2((v[k][2 * i] - mean) * rstd * gf.x + bf.x,
                                        (v[k][2 * i + 1] - mean) * rstd * gf.y + bf.y);
            }
            reinterpret_cast<uint4*>(yr)[ch] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

__global__ void sum_rows_kernel(const float* __restrict__ src, int parts, size_t n, float* __restrict__ out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int j = 0; j < parts; ++j) acc += src[j * n + i];
        out[i] = acc;
    }
}

// 8 columns per thread: 2 x float4 of the sum, 16 B of bias and residual
__global__ void add_bias_residual_kernel(const float* __restrict__ sum, const f16* __restrict__ bias,
                                         const f16* __restrict__ res, long long ldr, int M, int N,
                                         f16* __restrict__ out) {
    ptx::pdl_trigger();
    const size_t n8 = static_cast<size_t>(M) * N / 8;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t e0 = i * 8;
        const int row = static_cast<int>(e0 / N), col = static_cast<int>(e0 % N);
        const float4 a = __ldg(reinterpret_cast<const float4*>(sum + e0));
        const float4 b = __ldg(reinterpret_cast<const float4*>(sum + e0) + 1);
        float acc[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        if (bias) add8(acc, bias + col);
        if (res) add8(acc, res + static_cast<long long>(row) * ldr + col);
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = ptx::pack_f16x2(acc[2 * j], acc[2 * j + 1]);
        *reinterpret_cast<uint4*>(out + e0) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__global__ void splitk_reduce_f32_kernel(const float* __restrict__ ws, int splits, size_t n4, size_t plane,
                                         float* __restrict__ out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < splits; ++s) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(ws + s * plane) + i);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        reinterpret_cast<float4*>(out)[i] = acc;
    }
}

}  // namespace

static int grid_for(size_t work) {
    return static_cast<int>(std::min<size_t>((work + 255) / 256, 4 * static_cast<size_t>(num_sms())));
}

void sum_rows_f32(const float* src, int parts, size_t n, float* out, cudaStream_t st) {
    if (n) sum_rows_kernel<<<grid_for(n), 256, 0, st>>>(src, parts, n, out);
}

void add_bias_residual(const float* sum, const f16* bias, const f16* res, long long ldr, int M, int N, f16* out,
                       cudaStream_t st) {
    if (N % 8) throw std::invalid_argument("add_bias_residual: N must be a multiple of 8");
    const size_t n8 = static_cast<size_t>(M) * N / 8;
    if (n8) add_bias_residual_kernel<<<grid_for(n8), 256, 0, st>>>(sum, bias, res, ldr, M, N, out);
}

void splitk_reduce_f32(const float* ws, int splits, int M, int N, float* out, cudaStream_t st) {
    if (N % 4) throw std::invalid_argument("splitk_reduce_f32: N must be a multiple of 4");
    const size_t plane = static_cast<size_t>(M) * N;
    if (plane) splitk_reduce_f32_kernel<<<grid_for(plane / 4), 256, 0, st>>>(ws, splits, plane / 4, plane, out);
}

void layernorm_rows(const f16* x, long long ldx, const f16* gamma, const f16* beta, f16* y, long long ldy, int n,
                    int d, float eps, cudaStream_t st) {
    if (d % 8 || d > kLnThreads * kLnChunks * 8) throw std::invalid_argument("layernorm: d must be a multiple of 8, <= 16384");
    if (n > 0) layernorm_kernel<<<n, kLnThreads, 0, st>>>(x, ldx, gamma, beta, y, ldy, d, eps);
}

void embed(const f16* E, const f16* Pos, const int* ids, const int* pos, int n, int d, f16* X,
           long long ldx, cudaStream_t st) {
    if (n <= 0) return;
    if (d % 8) throw std::invalid_argument("embed: hidden_dim must be a multiple of 8");
    embed_kernel<<<n, 128, 0, st>>>(E, Pos, ids, pos, d, X, ldx);
}

void act_append(const AppendCall& c, cudaStream_t st) {
    if (c.B > 0) act_append_kernel<<<c.B, 128, 0, st>>>(c);
}

void kv_append(const AppendCall& c, cudaStream_t st) {
    if (c.B > 0) kv_append_kernel<<<c.B, 256, 0, st>>>(c);
}

void scatter_act_blocks(const BlockScatter& c, cudaStream_t st) {
    if (c.n_blocks > 0) scatter_act_kernel<<<c.n_blocks, 256, 0, st>>>(c);
}

void scatter_kv_blocks(const BlockScatter& c, cudaStream_t st) {
    if (c.n_blocks > 0) scatter_kv_kernel<<<c.n_blocks, 256, 0, st>>>(c);
}

void argmax_rows(const float* logits, int B, int V, int* out, cudaStream_t st) {
    if (B > 0) argmax_kernel<<<B, 256, 0, st>>>(logits, V, out);
}

void splitk_reduce(const float* ws, int splits, int M, int N, f16* out, bool relu, cudaStream_t st,
                   const f16* bias, const f16* res, long long ldr) {
    if (N % 8) throw std::invalid_argument("splitk_reduce: N must be a multiple of 8");
    const size_t n8 = static_cast<size_t>(M) * N / 8;
    const int blocks = static_cast<int>(std::min<size_t>((n8 + 255) / 256, 4 * static_cast<size_t>(num_sms())));
    if (n8) splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, splits, M, N, out, relu ? 1 : 0, bias, res, ldr);
}

void fill_pattern(f16* dst, size_t n, uint64_t seed, float amp, cudaStream_t st) {
    if (n) fill_pattern_kernel<<<4 * num_sms(), 256, 0, st>>>(dst, n, seed, amp);
}

}  // namespace hc
