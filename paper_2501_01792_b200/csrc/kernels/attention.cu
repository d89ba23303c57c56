// Decode attention over the hybrid block table (north-star (3)). The causal
// prefill attention lives in prefill_attention.cu.
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

__device__ __forceinline__ void load8(const f16* p, float (&f)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 v = __half22float2(h[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}

__device__ __forceinline__ uint4 ldg16(const f16* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 v = __half22float2(h[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}

// grid: (B*H, splits); block: 128 threads (4 warps)
// REC: every block of the call is a fused-recompute block (c.records_only):
// the K|V path compiles out, so the kernel holds few registers, runs more CTAs
// per SM and keeps 8 records per warp in flight
template <int HD, int TPB, bool REC = false>
__global__ void __launch_bounds__(kWarps * 32)
    decode_attn_kernel(const AttnCall c) {
    ptx::pdl_trigger();  // the projection GEMM after it may start streaming its weights
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
    constexpr int SEG = TPB < 32 ? TPB : 32;  // rows per partial record (gemm.cuh attn_part_tile)
    // the next block's ref is loaded one iteration ahead, so a block's K|V (or
    // partial record) loads never wait on its ref
    int ref_next = blk_begin + warp < blk_end ? __ldg(refs + blk_begin + warp) : 0;
    constexpr int SEGS = TPB / SEG;
    constexpr int G = 32 / LPT;  // token groups per warp: each takes its own record
    constexpr int RB = REC ? (SEGS >= 2 ? 2 : 4) : (SEGS >= 2 ? 1 : 2);  // records per group in flight (the mixed kernel keeps its registers for K|V)
    for (int blk = blk_begin + warp; blk < blk_end;) {
        const int ref = ref_next;
        if (REC || (ref >> 28) == c.part_region) {
            // partials of recomputed blocks: o, m (log2 domain, scale folded in), l.
            // The next n <= RB x G blocks of this warp that are recomputed ones go
            // together, one per token group and slot (a record is 0.5 KB: one per
            // warp would leave the loads latency-bound); every record load is issued
            // before any math. Each lane keeps its own running (m, l, acc); the fold
            // after the loop rescales the groups to a common max.
            constexpr int NC = RB * G;
            int rk[NC];
            rk[0] = ref;
#pragma unroll
            for (int k = 1; k < NC; ++k) {
                const int bk = blk + k * kWarps;
                rk[k] = bk < blk_end ? __ldg(refs + bk) : -1;  // same address on every lane
            }
            int n = 1;
#pragma unroll
            for (int k = 1; k < NC; ++k)
                if (n == k && rk[k] >= 0 && (REC || (rk[k] >> 28) == c.part_region)) ++n;
            float4 o0[RB][SEGS], o1[RB][SEGS];
            float mp[RB][SEGS], lp[RB][SEGS];
#pragma unroll
            for (int kk = 0; kk < RB; ++kk) {
                int mine = rk[kk * G];
#pragma unroll
                for (int g = 1; g < G; ++g)
                    if (grp == g) mine = rk[kk * G + g];
                if (kk * G + grp < n) {
#pragma unroll
                    for (int sg = 0; sg < SEGS; ++sg) {
                        const float* rec =
                            c.part + ((static_cast<long long>(mine & 0x0FFFFFFF) * SEGS + sg) * c.H + h) * (HD + 4);
                        o0[kk][sg] = __ldg(reinterpret_cast<const float4*>(rec + col));
                        o1[kk][sg] = __ldg(reinterpret_cast<const float4*>(rec + col + 4));
                        mp[kk][sg] = __ldg(rec + HD);
                        lp[kk][sg] = __ldg(rec + HD + 1);
                    }
                }
            }
            blk += n * kWarps;
            if (blk < blk_end) ref_next = __ldg(refs + blk);
#pragma unroll
            for (int kk = 0; kk < RB; ++kk) {
                if (kk * G + grp < n) {
#pragma unroll
                    for (int sg = 0; sg < SEGS; ++sg) {
                        const float m_new = fmaxf(m, mp[kk][sg]);
                        const float corr = exp2f(m - m_new);
                        const float f = exp2f(mp[kk][sg] - m_new);
                        l = l * corr + lp[kk][sg] * f;
                        acc[0] = acc[0] * corr + o0[kk][sg].x * f;
                        acc[1] = acc[1] * corr + o0[kk][sg].y * f;
                        acc[2] = acc[2] * corr + o0[kk][sg].z * f;
                        acc[3] = acc[3] * corr + o0[kk][sg].w * f;
                        acc[4] = acc[4] * corr + o1[kk][sg].x * f;
                        acc[5] = acc[5] * corr + o1[kk][sg].y * f;
                        acc[6] = acc[6] * corr + o1[kk][sg].z * f;
                        acc[7] = acc[7] * corr + o1[kk][sg].w * f;
                        m = m_new;
                    }
                }
            }
            continue;
        }
        if constexpr (!REC) {
            blk += kWarps;
            if (blk < blk_end) ref_next = __ldg(refs + blk);
            const int blk_cur = blk - kWarps;
            const f16* base = c.region[ref >> 28] + static_cast<long long>(ref & 0x0FFFFFFF) * block_elems + head_off;
            const int valid = (blk_cur == nb - 1) ? ctx - (nb - 1) * TPB : TPB;
            uint4 kr[ITERS], vr[ITERS];
#pragma unroll
            for (int i = 0; i < ITERS; ++i) {
                const int t = i * TPW + grp;
                kr[i] = ldg16(base + t * HD + col);
                vr[i] = ldg16(base + v_off + t * HD + col);
            }
            if (valid < TPB) {  // unfilled slots of the last block may hold any bits (even NaN): 0 * NaN != 0
#pragma unroll
                for (int i = 0; i < ITERS; ++i)
                    if (i * TPW + grp >= valid) vr[i] = make_uint4(0, 0, 0, 0);
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
    }

    // fold the token groups of the warp: each lane's (m, l, acc) is self-consistent
    // (records give the groups different maxima), so rescale to the warp max first
    {
        float M = m;
#pragma unroll
        for (int o = LPT; o < 32; o <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float f = exp2f(m - M);  // m = -FLT_MAX (nothing merged) -> 0, or 1 when M is too
        l *= f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= f;
        m = M;
    }
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
            c.out[static_cast<long long>(b) * d + h * HD + threadIdx.x] = __float2half_rn(L > 0.f ? O / L : 0.f);
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
    ptx::pdl_trigger();
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
        c.out[static_cast<long long>(b) * d + h * HD + col] = __float2half_rn(L > 0.f ? O / L : 0.f);
    }
}

// ---------------------------------------------------------------------------
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
        if (c.records_only && c.part)                                            \
            decode_attn_kernel<HD_, TPB_, true><<<grid, kWarps * 32, 0, st>>>(c);  \
        else                                                                     \
            decode_attn_kernel<HD_, TPB_><<<grid, kWarps * 32, 0, st>>>(c);      \
        if (c.splits > 1) attn_combine_kernel<HD_><<<c.B * c.H, HD_, 0, st>>>(c); \
        return;                                                                  \
    }
    HC_ATTN(128, 16)
    HC_ATTN(64, 16)
    HC_ATTN(128, 8)
    HC_ATTN(64, 8)
    HC_ATTN(128, 32)
    HC_ATTN(64, 32)
    HC_ATTN(128, 4)
    HC_ATTN(64, 4)
    HC_ATTN(128, 64)
    HC_ATTN(64, 64)
#undef HC_ATTN
    throw std::invalid_argument("decode_attention: unsupported (head_dim, tokens_per_block)");
}

bool decode_attention_supported(int hd, int tpb) {
    return (hd == 64 || hd == 128) && (tpb == 4 || tpb == 8 || tpb == 16 || tpb == 32 || tpb == 64);
}

}  // namespace hc
