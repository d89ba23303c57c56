// Decode attention over the hybrid block table (north-star (3)) and causal
// prefill attention.
//
// Semantics: attention_row, decoder.cpp:15-43 — per head h,
//   out_h = softmax(q_h . K_h^T * s) . V_h,  s = 1/sqrt(hd) (scaled=true),
// max-subtracted. Here the softmax is computed online (flash-decoding) over
// the request's logical blocks, which may live in different regions
// (streamed KV staging, GPU-resident KV, or the buffer the recompute GEMM just
// filled from ACT blocks): the context is never concatenated
// (decoder.cpp:167 / verify.cpp:71-72 copies are eliminated).
//
// Memory path: one warp walks one block at a time; every lane issues 16-byte
// loads of K and V rows (head-major block layout makes each head's K and V a
// contiguous tpb*hd*2-byte run), all loads of a block are in flight before
// any math; softmax and the P.V reduction use warp shuffles only.
#include <cfloat>
#include <stdexcept>

#include "kernels.hpp"
#include "ptx.cuh"

namespace hc {

namespace {

constexpr int kWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void load8(const bf16* p, float (&f)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(h[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}

__device__ __forceinline__ uint4 ldg16(const bf16* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(h[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}

// grid: (B*H, splits); block: 128 threads (4 warps)
template <int HD, int TPB>
__global__ void __launch_bounds__(kWarps * 32)
    decode_attn_kernel(const AttnCall c) {
    constexpr int LPT = HD / 8;        // lanes per token row
    constexpr int TPW = 32 / LPT;      // token rows per warp-wide load
    constexpr int ITERS = TPB / TPW;   // loads per block per lane (K and V each)
    static_assert(TPB % TPW == 0, "tokens per block must be a multiple of rows per load");

    const int bh = blockIdx.x;
    const int b = bh / c.H;
    const int h = bh - b * c.H;
    const int split = blockIdx.y;
    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int grp = lane / LPT;         // which token row of a load
    const int col = (lane % LPT) * 8;   // 8 columns of the head

    const int nb = c.n_blocks[b];
    const int ctx = c.ctx_len[b];
    const int per = (nb + c.splits - 1) / c.splits;
    const int blk_begin = split * per;
    const int blk_end = min(nb, blk_begin + per);

    const int d = c.H * HD;
    const long long block_elems = 2LL * d * TPB;
    const long long head_off = static_cast<long long>(h) * TPB * HD;
    const long long v_off = static_cast<long long>(d) * TPB;

    float q[8];
    load8(c.q + static_cast<long long>(b) * c.ldq + h * HD + col, q);
    const float qs = c.scale * kLog2e;
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] *= qs;

    float m = -FLT_MAX;  // running max (log2 domain)
    float l = 0.f;       // running denominator, this lane's token group
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};

    const int* refs = c.blk_ref + static_cast<long long>(b) * c.max_blocks;
    for (int blk = blk_begin + warp; blk < blk_end; blk += kWarps) {
        const int ref = refs[blk];
        const bf16* base = c.region[ref >> 28] + static_cast<long long>(ref & 0x0FFFFFFF) * block_elems + head_off;
        const int valid = (blk == nb - 1) ? ctx - (nb - 1) * TPB : TPB;
        uint4 kr[ITERS], vr[ITERS];
#pragma unroll
        for (int i = 0; i < ITERS; ++i) {
            const int t = i * TPW + grp;
            kr[i] = ldg16(base + t * HD + col);
            vr[i] = ldg16(base + v_off + t * HD + col);
        }
        float s[ITERS];
        float bmax = -FLT_MAX;
#pragma unroll
        for (int i = 0; i < ITERS; ++i) {
            float kf[8];
            unpack8(kr[i], kf);
            float dot = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) dot = fmaf(q[j], kf[j], dot);
#pragma unroll
            for (int o = LPT / 2; o >= 1; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const int t = i * TPW + grp;
            s[i] = t < valid ? dot : -FLT_MAX;
            bmax = fmaxf(bmax, s[i]);
        }
#pragma unroll
        for (int o = LPT; o < 32; o <<= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
        const float m_new = fmaxf(m, bmax);
        const float corr = exp2f(m - m_new);
        l *= corr;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= corr;
        m = m_new;
#pragma unroll
        for (int i = 0; i < ITERS; ++i) {
            const int t = i * TPW + grp;
            const float pr = t < valid ? exp2f(s[i] - m) : 0.f;
            l += pr;
            float vf[8];
            unpack8(vr[i], vf);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = fmaf(pr, vf[j], acc[j]);
        }
    }
    // fold token groups of the warp (all share m)
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    }

    __shared__ float sm_m[kWarps], sm_l[kWarps];
    __shared__ float sm_acc[kWarps][HD];
    if (lane < LPT) {
#pragma unroll
        for (int j = 0; j < 8; ++j) sm_acc[warp][col + j] = acc[j];
    }
    if (lane == 0) {
        sm_m[warp] = m;
        sm_l[warp] = l;
    }
    __syncthreads();
    if (threadIdx.x < HD) {
        float M = -FLT_MAX;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float f = sm_l[w] > 0.f ? exp2f(sm_m[w] - M) : 0.f;
            L += sm_l[w] * f;
            O += sm_acc[w][threadIdx.x] * f;
        }
        if (c.splits == 1) {
            c.out[static_cast<long long>(b) * d + h * HD + threadIdx.x] = __float2bfloat16(L > 0.f ? O / L : 0.f);
        } else {
            float* w = c.work + (static_cast<long long>(bh) * c.splits + split) * (HD + 2);
            w[threadIdx.x] = O;
            if (threadIdx.x == 0) {
                w[HD] = M;
                w[HD + 1] = L;
            }
        }
    }
}

template <int HD>
__global__ void attn_combine_kernel(const AttnCall c) {
    const int bh = blockIdx.x;
    const int b = bh / c.H;
    const int h = bh - b * c.H;
    const int d = c.H * HD;
    const float* w = c.work + static_cast<long long>(bh) * c.splits * (HD + 2);
    float M = -FLT_MAX;
    for (int s = 0; s < c.splits; ++s)
        if (w[s * (HD + 2) + HD + 1] > 0.f) M = fmaxf(M, w[s * (HD + 2) + HD]);
    for (int col = threadIdx.x; col < HD; col += blockDim.x) {
        float L = 0.f, O = 0.f;
        for (int s = 0; s < c.splits; ++s) {
            const float* ws = w + s * (HD + 2);
            if (ws[HD + 1] <= 0.f) continue;
            const float f = exp2f(ws[HD] - M);
            L += ws[HD + 1] * f;
            O += ws[col] * f;
        }
        c.out[static_cast<long long>(b) * d + h * HD + col] = __float2bfloat16(L > 0.f ? O / L : 0.f);
    }
}

// ---------------------------------------------------------------------------
// Causal prefill attention (attention_causal, decoder.cpp:55-63): CUDA cores,
// one CTA per (request, head, 64-query tile); 2 threads per query each own
// half of the head dims; K/V tiles of 32 keys staged in shared memory.
template <int HD>
__global__ void __launch_bounds__(128)
    prefill_attn_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ out, const int* __restrict__ cu, int H,
                        float scale) {
    constexpr int QT = 64, KT = 32, HALF = HD / 2;
    const int d = H * HD;
    const int ld = 3 * d;
    const int req = blockIdx.z;
    const int h = blockIdx.y;
    const int q0 = blockIdx.x * QT;
    const int row0 = cu[req];
    const int P = cu[req + 1] - row0;
    if (q0 >= P) return;
    const int tq = threadIdx.x / 2;
    const int half = threadIdx.x % 2;
    const int t = q0 + tq;
    const bool active = t < P;

    __shared__ __align__(16) bf16 sk[KT][HD];
    __shared__ __align__(16) bf16 sv[KT][HD];

    const bf16* rowbase = qkv + static_cast<long long>(row0) * ld;
    float q[HALF];
    {
        const bf16* qp = rowbase + static_cast<long long>(active ? t : 0) * ld + h * HD + half * HALF;
#pragma unroll
        for (int j = 0; j < HALF; j += 8) {
            float f[8];
            load8(qp + j, f);
#pragma unroll
            for (int i = 0; i < 8; ++i) q[j + i] = f[i] * scale * kLog2e;
        }
    }
    float m = -FLT_MAX, l = 0.f;
    float acc[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc[j] = 0.f;

    const int kmax = min(P, q0 + QT);  // keys needed by this tile
    for (int k0 = 0; k0 < kmax; k0 += KT) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < KT * HD / 8; idx += blockDim.x) {
            const int r = idx / (HD / 8), cc = (idx % (HD / 8)) * 8;
            const int key = k0 + r;
            uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
            if (key < P) {
                const bf16* kp = rowbase + static_cast<long long>(key) * ld + d + h * HD + cc;
                kv = *reinterpret_cast<const uint4*>(kp);
                vv = *reinterpret_cast<const uint4*>(kp + d);
            }
            *reinterpret_cast<uint4*>(&sk[r][cc]) = kv;
            *reinterpret_cast<uint4*>(&sv[r][cc]) = vv;
        }
        __syncthreads();
        const int kend = min(KT, kmax - k0);
        for (int r = 0; r < kend; ++r) {
            const int key = k0 + r;
            float dot = 0.f;
#pragma unroll
            for (int j = 0; j < HALF; j += 2) {
                const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sk[r][half * HALF + j]));
                dot = fmaf(q[j], kf.x, dot);
                dot = fmaf(q[j + 1], kf.y, dot);
            }
            dot += __shfl_xor_sync(0xffffffffu, dot, 1);
            if (key > t) continue;  // causal mask (uniform within the thread pair)
            const float m_new = fmaxf(m, dot);
            const float corr = exp2f(m - m_new);
            const float pr = exp2f(dot - m_new);
            l = l * corr + pr;
#pragma unroll
            for (int j = 0; j < HALF; j += 2) {
                const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sv[r][half * HALF + j]));
                acc[j] = fmaf(pr, vf.x, acc[j] * corr);
                acc[j + 1] = fmaf(pr, vf.y, acc[j + 1] * corr);
            }
            m = m_new;
        }
    }
    if (!active) return;
    bf16* op = out + static_cast<long long>(row0 + t) * d + h * HD + half * HALF;
    const float inv = 1.f / l;
#pragma unroll
    for (int j = 0; j < HALF; j += 8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = ptx::pack_bf16x2(acc[j + 2 * i] * inv, acc[j + 2 * i + 1] * inv);
        *reinterpret_cast<uint4*>(op + j) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace

int attention_splits(int B, int H, int max_ctx, int tpb) {
    // enough CTAs for ~4 waves; never split below 8 blocks per split
    const int pairs = B * H;
    const int blocks = (max_ctx + tpb - 1) / tpb;
    int splits = 1;
    while (pairs * splits < 4 * num_sms() && blocks / (splits * 2) >= 8) splits *= 2;
    return splits;
}

void decode_attention(const AttnCall& c, cudaStream_t st) {
    if (c.B <= 0) return;
    const dim3 grid(c.B * c.H, c.splits);
#define HC_ATTN(HD_, TPB_)                                                       \
    if (c.hd == HD_ && c.tpb == TPB_) {                                          \
        decode_attn_kernel<HD_, TPB_><<<grid, kWarps * 32, 0, st>>>(c);          \
        if (c.splits > 1) attn_combine_kernel<HD_><<<c.B * c.H, HD_, 0, st>>>(c); \
        return;                                                                  \
    }
    HC_ATTN(128, 16)
    HC_ATTN(64, 16)
    HC_ATTN(128, 8)
    HC_ATTN(64, 8)
    HC_ATTN(128, 32)
    HC_ATTN(64, 32)
#undef HC_ATTN
    throw std::invalid_argument("decode_attention: unsupported (head_dim, tokens_per_block)");
}

void prefill_attention(const bf16* qkv, bf16* out, const int* cu, int n_req, int max_len, int H, int hd,
                       float scale, cudaStream_t st) {
    if (n_req <= 0 || max_len <= 0) return;
    const dim3 grid((max_len + 63) / 64, H, n_req);
    if (hd == 128)
        prefill_attn_kernel<128><<<grid, 128, 0, st>>>(qkv, out, cu, H, scale);
    else if (hd == 64)
        prefill_attn_kernel<64><<<grid, 128, 0, st>>>(qkv, out, cu, H, scale);
    else
        throw std::invalid_argument("prefill_attention: head_dim must be 64 or 128");
}

}  // namespace hc
