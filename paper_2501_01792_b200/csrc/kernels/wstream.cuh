// Weight-streaming decode GEMM for sm_100a (tcgen05, swap-AB, stream-K).
//
//   C[M x N] = A[M x K] . W[N x K]^T      M = the decode batch (<= 256)
//
// The decode projections (qkv_generate / project_ffn, decoder.cpp:97-121) and
// the LM head run at M = batch rows against weight matrices of N x K with
// N, K in the thousands: every weight byte is used M times, so the GEMM is
// bound by streaming W from HBM once. The generic tile kernel (gemm.cuh)
// puts the batch on the UMMA M side (128 rows, half empty at M = 64) and
// splits K into whole-tile ranges reduced by a second kernel; here
//
//   * the roles swap: W rows are the UMMA A operand (M = 128 per MMA, two
//     MMAs per k-block = 256 weight rows per unit) and the batch is the UMMA
//     N operand (MP = M rounded up to 16..256 columns of TMEM), so every smem
//     byte of W feeds a full-height MMA and the batch operand is 1/4-1/2 of
//     the W bytes per stage;
//   * the k-block iterations of all units (256 weight rows x all of K) are cut
//     into gridDim.x equal contiguous ranges (stream-K): every SM streams the
//     same number of weight bytes whatever N / 256 is against 148;
//   * a unit cut between CTAs leaves one fp32 partial per segment; a small
//     reduce kernel (launched programmatically dependent, so its launch hides
//     under the GEMM's tail) sums them in a fixed order — deterministic, and
//     spread over every SM instead of serialised on one contributor;
//   * launched with programmatic stream serialisation (GemmCall::pdl) the GEMM
//     requests its first S stages of W before griddepcontrol.wait — weights
//     never depend on the predecessor — so the weight stream starts under the
//     previous kernel's tail; the batch operand, residual and stores wait.
//
// Roles (192 threads) as in gemm.cuh: warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer, warps 2..5 epilogue (TMEM lane quarter = warp % 4,
// one weight row = one output column n per thread).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm_types.hpp"
#include "ptx.cuh"

namespace hc::wstream {

using gemm::BK;

struct Params {
    int M, N, K;
    int NK;         // k-blocks per unit (ceil(K / BK))
    int units;      // ceil(N / WT)
    long long T;    // units * NK (stream-K iterations)
    int G;          // CTAs (gridDim.x)
    void* out;      // f16 or fp32 [M x ldc]
    long long ldc;
    const __half* bias;  // [N] or null (f16 epilogues)
    const __half* res;   // [M x ldr] or null (f16 epilogues)
    long long ldr;
    float* part;    // [2G][MP][WT] fp32 partial slots (slot 2c: CTA c's first segment, 2c+1: its last)
};

template <int MP>
struct Cfg {
    static_assert(MP == 16 || MP == 32 || MP == 64 || MP == 128 || MP == 256, "MP: batch columns of TMEM");
    static constexpr int NMMA = MP == 256 ? 1 : 2;  // 128-row weight MMAs per k-block
    static constexpr int WT = 128 * NMMA;           // weight rows (output columns) per unit
    static constexpr int kWBytes = 128 * BK * 2;    // one 128-row W box
    static constexpr int kXBytes = MP * BK * 2;     // the batch box
    static constexpr int kStageBytes = NMMA * kWBytes + kXBytes;
    static constexpr int kStages = (216 * 1024) / kStageBytes > 8 ? 8 : (216 * 1024) / kStageBytes;
    static constexpr int kTmemCols = 2 * NMMA * MP < 32 ? 32 : 2 * NMMA * MP;
    static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
    static constexpr int kSmemBytes = kStages * kStageBytes + kBarBytes + 1024;
};

__device__ __forceinline__ long long seg_begin(int c, const Params& p) {
    return static_cast<long long>(c) * p.T / p.G;
}

// the CTA whose range holds iteration `it`
__device__ __forceinline__ int seg_owner(long long it, const Params& p) {
    int c = static_cast<int>(it * p.G / p.T);
    while (c + 1 < p.G && seg_begin(c + 1, p) <= it) ++c;
    while (c > 0 && seg_begin(c, p) > it) --c;
    return c;
}

template <int MP, int EPI>
__global__ void __launch_bounds__(192, 1)
    wstream_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const Params p) {
    using C = Cfg<MP>;
    constexpr int S = C::kStages;
    constexpr int NMMA = C::NMMA;
    constexpr int WT = C::WT;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_w = smem;                                 // [S][NMMA][128 x 64]
    uint8_t* smem_x = smem + S * NMMA * C::kWBytes;         // [S][MP x 64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int cta = blockIdx.x;
    const long long it_begin = seg_begin(cta, p), it_end = seg_begin(cta + 1, p);

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmW);
        ptx::tma_prefetch(&tmX);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();  // the reduce kernel may launch now (its wait holds it until this grid is done)

    if (warp == 0) {
        if (lane == 0) {
            // W is read once (evict first); the batch operand is re-read by every CTA (keep)
            const uint64_t pol_w = ptx::policy_evict_first(), pol_x = ptx::policy_evict_last();
            const int n = static_cast<int>(it_end - it_begin);
            auto load_w = [&](int i, int stage) {
                const long long it = it_begin + i;
                const int unit = static_cast<int>(it / p.NK);
                const int kb = static_cast<int>(it - static_cast<long long>(unit) * p.NK);
#pragma unroll
                for (int j = 0; j < NMMA; ++j)
                    ptx::tma_load_2d_hint(smem_w + (stage * NMMA + j) * C::kWBytes, &tmW, &full[stage], kb * BK,
                                          unit * WT + j * 128, pol_w);
            };
            auto load_x = [&](int i, int stage) {
                const long long it = it_begin + i;
                const int kb = static_cast<int>(it % p.NK);
                ptx::tma_load_2d_hint(smem_x + stage * C::kXBytes, &tmX, &full[stage], kb * BK, 0, pol_x);
            };
            // the first S stages' weights do not depend on the previous kernel:
            // issue them before griddepcontrol.wait (a programmatic launch overlaps
            // them with the predecessor's tail), the batch operand after it
            const int npre = n < S ? n : S;
            for (int i = 0; i < npre; ++i) {
                ptx::mbar_arrive_expect_tx(&full[i], C::kStageBytes);
                load_w(i, i);
            }
            ptx::pdl_wait();
            for (int i = 0; i < npre; ++i) load_x(i, i);
            int stage = npre % S;
            uint32_t phase = npre == S ? 1 : 0;
            for (int i = npre; i < n; ++i) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                load_w(i, stage);
                load_x(i, stage);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(128, MP);
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            for (long long it = it_begin; it < it_end;) {
                const int unit = static_cast<int>(it / p.NK);
                const int k0 = static_cast<int>(it - static_cast<long long>(unit) * p.NK);
                const int k1 = static_cast<int>(min(static_cast<long long>(p.NK), k0 + (it_end - it)));
                ptx::mbar_wait(&tempty[as], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + as * NMMA * MP;
                for (int kb = k0; kb < k1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t x_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_x + stage * C::kXBytes));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
                        for (int j = 0; j < NMMA; ++j) {
                            const uint64_t w_desc =
                                ptx::sw128_kmajor_desc(ptx::smem_u32(smem_w + (stage * NMMA + j) * C::kWBytes));
                            ptx::mma_f16_ss(d_tmem + j * MP, w_desc + 2 * k, x_desc + 2 * k, idesc,
                                            ((kb - k0) | k) != 0);
                        }
                    }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(&tfull[as]);
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1;
                }
                it += k1 - k0;
            }
        }
    } else {
        ptx::pdl_wait();  // res / out / partial slots belong to the predecessor until it ends
        const int q = warp % 4;
        const int r = q * 32 + lane;  // weight row within a 128-row MMA = output column offset
        int as = 0;
        uint32_t aphase = 0;
        for (long long it = it_begin; it < it_end;) {
            const int unit = static_cast<int>(it / p.NK);
            const int k0 = static_cast<int>(it - static_cast<long long>(unit) * p.NK);
            const int k1 = static_cast<int>(min(static_cast<long long>(p.NK), k0 + (it_end - it)));
            const bool first = it == it_begin;
            it += k1 - k0;
            ptx::mbar_wait(&tfull[as], aphase);
            ptx::tc_fence_after();
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * NMMA * MP;
            if (!(k0 == 0 && k1 == p.NK)) {
                // a cut unit: this segment's partial -> its slot ([m][WT], coalesced
                // along the weight rows); wstream_reduce_kernel finishes the unit
                float* slot = p.part + static_cast<size_t>(2 * cta + (first ? 0 : 1)) * MP * WT + r;
#pragma unroll 1
                for (int j = 0; j < NMMA; ++j) {
#pragma unroll 1
                    for (int c0 = 0; c0 < p.M; c0 += 16) {  // warp-uniform: tcgen05.ld is .sync.aligned
                        uint32_t v[16];
                        ptx::tmem_ld_x16(t_row + j * MP + c0, v);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c0 + i < p.M) __stcg(slot + (c0 + i) * WT + j * 128, __uint_as_float(v[i]));
                    }
                }
            } else {
#pragma unroll 1
                for (int j = 0; j < NMMA; ++j) {
                    const int n = unit * WT + j * 128 + r;
                    const bool nvalid = n < p.N;
                    float b = 0.f;
                    if constexpr (EPI != gemm::kF32)
                        if (p.bias && nvalid) b = __half2float(p.bias[n]);
#pragma unroll 1
                    for (int c0 = 0; c0 < p.M; c0 += 16) {
                        uint32_t v[16];
                        ptx::tmem_ld_x16(t_row + j * MP + c0, v);
                        ptx::tmem_ld_wait();
                        if (!nvalid) continue;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int m = c0 + i;
                            if (m >= p.M) break;
                            const float acc = __uint_as_float(v[i]);
                            if constexpr (EPI == gemm::kF32) {
                                static_cast<float*>(p.out)[m * p.ldc + n] = acc;
                            } else {
                                float x = acc + b;
                                if (p.res) x += __half2float(p.res[m * p.ldr + n]);
                                if constexpr (EPI == gemm::kRelu) x = fmaxf(x, 0.f);
                                static_cast<__half*>(p.out)[m * p.ldc + n] = __float2half_rn(x);
                            }
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[as]);
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
        }
    }

    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// Finish of the cut units: out[m][n] = epi(sum over the unit's segments, in
// CTA order, + bias[n] + res[m][n]). Work item (unit, 4-row slice): warp 0
// resolves the unit's segments into shared memory (whole units are skipped),
// then each thread owns 4 consecutive n of one row and issues its segments'
// float4 loads 8 at a time before summing — the partials are L2-resident.
// Launched with programmatic stream serialisation: the launch overlaps the
// GEMM, and griddepcontrol.wait holds the reads until the GEMM has finished.
constexpr int kMaxCut = 64;  // segments one unit may be cut into (the launcher caps G accordingly)

template <int MP, int EPI>
__global__ void __launch_bounds__(256) wstream_reduce_kernel(const Params p) {
    ptx::pdl_trigger();  // the next GEMM may start its weight prefetch
    constexpr int WT = Cfg<MP>::WT;
    constexpr int quads = WT / 4;
    constexpr int RB = 256 / quads;  // rows per work item
    __shared__ int s_slot[kMaxCut];
    __shared__ int s_n;
    const int slices = (p.M + RB - 1) / RB;
    bool waited = false;
    // grid-stride over (unit, 4-row slice) items: the grid stays small enough to
    // be resident at once, so its launch_dependents lets the next GEMM start early
    for (int item = blockIdx.x; item < p.units * slices; item += gridDim.x) {
        const int unit = item / slices;
        const long long u0 = static_cast<long long>(unit) * p.NK;
        __syncthreads();  // s_slot / s_n of the previous item are consumed
        if (threadIdx.x < 32) {
            const int c_lo = seg_owner(u0, p), c_hi = seg_owner(u0 + p.NK - 1, p);
            for (int c = c_lo + static_cast<int>(threadIdx.x); c <= c_hi && c - c_lo < kMaxCut; c += 32)
                s_slot[c - c_lo] = 2 * c + (seg_begin(c, p) >= u0 ? 0 : 1);
            if (threadIdx.x == 0) s_n = c_hi - c_lo + 1;
        }
        __syncthreads();
        const int nseg = s_n;
        if (nseg < 2) continue;  // a whole unit: wstream_kernel stored it
        const int m = (item - unit * slices) * RB + static_cast<int>(threadIdx.x) / quads;
        const int nl = (threadIdx.x % quads) * 4;
        const int n = unit * WT + nl;
        if (m >= p.M || n >= p.N) continue;
        if (!waited) {
            ptx::pdl_wait();
            waited = true;
        }
        const float* base = p.part + static_cast<size_t>(m) * WT + nl;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s0 = 0; s0 < nseg; s0 += 8) {
            float4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                v[k] = s0 + k < nseg ? __ldcg(reinterpret_cast<const float4*>(
                                           base + static_cast<size_t>(s_slot[s0 + k]) * MP * WT))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // fixed order: segment s0 + k
                acc.x += v[k].x;
                acc.y += v[k].y;
                acc.z += v[k].z;
                acc.w += v[k].w;
            }
        }
        if constexpr (EPI == gemm::kF32) {
            *reinterpret_cast<float4*>(static_cast<float*>(p.out) + m * p.ldc + n) = acc;
        } else {
            float x[4] = {acc.x, acc.y, acc.z, acc.w};
            if (p.bias) {
                const uint2 b = *reinterpret_cast<const uint2*>(p.bias + n);
                const float2 b0 = __half22float2(*reinterpret_cast<const __half2*>(&b.x));
                const float2 b1 = __half22float2(*reinterpret_cast<const __half2*>(&b.y));
                x[0] += b0.x;
                x[1] += b0.y;
                x[2] += b1.x;
                x[3] += b1.y;
            }
            if (p.res) {
                const uint2 r = *reinterpret_cast<const uint2*>(p.res + m * p.ldr + n);
                const float2 r0 = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
                const float2 r1 = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
                x[0] += r0.x;
                x[1] += r0.y;
                x[2] += r1.x;
                x[3] += r1.y;
            }
            if constexpr (EPI == gemm::kRelu)
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = fmaxf(x[i], 0.f);
            uint2 h;
            h.x = ptx::pack_f16x2(x[0], x[1]);
            h.y = ptx::pack_f16x2(x[2], x[3]);
            *reinterpret_cast<uint2*>(static_cast<__half*>(p.out) + m * p.ldc + n) = h;
        }
    }
}

}  // namespace hc::wstream
