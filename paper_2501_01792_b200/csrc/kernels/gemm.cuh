// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M x N] = A[M x K] * B[N x K]^T     (f16 in, fp32 accumulate in TMEM)
//
// A: activations, row-major (K contiguous). B: weights stored transposed
// ([out][in], K contiguous), so both operands are K-major and TMA loads
// 128-row x 64-col (128 B) boxes with the 128B swizzle UMMA expects.
//
// Roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2..5 = epilogue (TMEM lane quarter
// = warp % 4). Two TMEM accumulator stages let the epilogue of tile i overlap
// the MMAs of tile i+1; an S-stage smem ring overlaps TMA with MMA.
//
// Epilogues (one template instance each):
//   kStore      f16 row-major C
//   kRelu       f16 relu(C)                       (FFN1, decoder.cpp:118-119)
//   kKvPaged    recompute K|V written straight into the paged KV block layout
//               [blk][K|V][head][tok][hd]  (north-star (2), decoder.cpp:123-129)
//   kF32        fp32 row-major (logits)
//   kAttnPart   recompute fused with decode attention: the N tile is [K_h | V_h]
//               of 128/hd heads, and instead of storing K|V the epilogue turns
//               each segment of tokens into a flash-decoding partial (m, l, o)
//               for its request's query (decoder.cpp:15-43 over the recomputed
//               rows), which decode_attention merges with the KV-cached blocks
#pragma once
#include <cuda.h>
#include <cfloat>
#include <cuda_runtime.h>

#include "gemm_types.hpp"
#include "ptx.cuh"

namespace hc::gemm {

constexpr int kThreads = 192;

struct Params {
    int M, N, K;
    int num_m_tiles, num_n_tiles;
    const int* m_tile_rows;  // optional explicit first-row of each M tile
    void* out;
    long long ldc;
    // kKvPaged: row r -> block r / tpb + blk_off, token r % tpb
    int tpb, d, hd, blk_off;
    int group_m;  // M tiles per rasterisation group (A tiles kept in L2 while N is swept)
    int group_n;  // > 0: N tiles per group instead (B tiles kept in L2 while M is swept)
    // split-K (kSplitF32): work unit = (tile, split); split s covers k-blocks
    // [s*kb_per_split, (s+1)*kb_per_split) and writes fp32 partials to
    // out + (s*M + row)*ldc
    int splits, kb_per_split;
    // optional epilogue operands (f16; applied before relu, not to fp32 outputs):
    // C[m][n] += bias[n] + res[m * ldr + n]
    const __half* bias;
    const __half* res;
    long long ldr;
    // L2 policy bits (kL2*): which operand the raster wants kept in L2
    int l2_hint;
    // kAttnPart: N tile ni = heads [ni*128/hd, (ni+1)*128/hd); B rows of the V
    // half start at v_row (= d); blk_info[mi * (BM/tpb) + slot] = request << 8 |
    // valid tokens of the block at that slot of M tile mi (-1: not in this
    // step); q rows by request (f16, ld ldq, own heads from column 0), scaled
    // by qscale (= softmax scale * log2 e); partial records (fp32, hd + 4 for
    // 16-byte rows: o[hd], m, l, pad) at part[((blk * (tpb/seg) + seg) * heads + h) * (hd + 4)]
    int v_row;
    const int* blk_info;
    const __half* q;
    long long ldq;
    float qscale;
    int heads;
    float* part;
};

// L2 policy bits (Params::l2_hint)
constexpr int kL2KeepA = 1;    // A tiles evict_last (the group's A slab is reused across the N sweep),
                               // evict_first on an A tile's last use (its last N tile)
constexpr int kL2StreamB = 2;  // B tiles evict_first
constexpr int kL2StreamC = 4;  // C stores streaming (st.global.cs: the output is not re-read from L2)

template <int BN>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
    static constexpr int kSmemBytes = kStages * kStageBytes + kBarBytes + 1024;  // + align slack
};

__device__ __forceinline__ void tile_coords(int tile, const Params& p, int& m_idx, int& n_idx) {
    // grouped rasterisation: group_m M-tiles share each sweep over N so
    // concurrently running CTAs reuse A and B tiles from L2
    tile %= p.num_m_tiles * p.num_n_tiles;  // split-K units repeat the tile grid
    if (p.group_n > 0) {  // weight-stationary: a group of N tiles sweeps all of M
        const int G = p.num_n_tiles < p.group_n ? p.num_n_tiles : p.group_n;
        const int group = G * p.num_m_tiles;
        const int g = tile / group;
        const int first_n = g * G;
        const int gn = (p.num_n_tiles - first_n) < G ? (p.num_n_tiles - first_n) : G;
        const int within = tile - g * group;
        n_idx = first_n + within % gn;
        m_idx = within / gn;
        return;
    }
    const int G = p.num_m_tiles < p.group_m ? p.num_m_tiles : p.group_m;
    const int group = G * p.num_n_tiles;
    const int g = tile / group;
    const int first_m = g * G;
    const int gm = (p.num_m_tiles - first_m) < G ? (p.num_m_tiles - first_m) : G;
    const int within = tile - g * group;
    m_idx = first_m + within % gm;
    n_idx = within / gm;
}

// acc[0..16) += 16 consecutive f16 at src (32-byte aligned run)
__device__ __forceinline__ void add16(float (&acc)[16], const __half* src) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const uint4 u = __ldg(s4 + q);
        const __half2* h2 = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h2[i]);
            acc[8 * q + 2 * i] += f.x;
            acc[8 * q + 2 * i + 1] += f.y;
        }
    }
}

// ---- kAttnPart epilogue ----------------------------------------------------
// 16 consecutive f16 at src -> fp32 (32-byte aligned run)
__device__ __forceinline__ void load16(float (&f)[16], const __half* src) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const uint4 u = __ldg(s4 + q);
        const __half2* h2 = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 v = __half22float2(h2[i]);
            f[8 * q + 2 * i] = v.x;
            f[8 * q + 2 * i + 1] = v.y;
        }
    }
}

// the f16 value the unfused path would have stored (K|V are cached as f16)
__device__ __forceinline__ float round_f16(float x) { return __half2float(__float2half_rn(x)); }

// Sum v[0..16) over the SEG lanes of a segment (lanes that differ in their
// low log2(SEG) bits) and scatter the sums: on return this lane holds
// n = max(1, 16/SEG) column sums in v[0..n), for columns [*col0, *col0 + n)
// of the 16 (lanes whose low bits differ only above bit log2(16)... hold copies
// when SEG = 32: lane pairs (i, i^1) agree).
template <int SEG>
__device__ __forceinline__ void seg_reduce_scatter16(float (&v)[16], int lane, int* col0) {
    int base = 0;
    int n = 16;
#pragma unroll
    for (int off = SEG / 2; off >= 1; off >>= 1) {
        if (n > 1) {
            const bool up = (lane & off) != 0;
            const int half = n / 2;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k < half) {
                    const float send = up ? v[k] : v[k + half];
                    const float keep = up ? v[k + half] : v[k];
                    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
            }
            if (up) base += half;
            n = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        }
    }
    *col0 = base;
}

// One TMEM lane (= one recomputed token row) of a finished [K_h | V_h] tile:
// s = q_b,h . K_row (K rounded to f16 as the cache stores it), then per
// segment of SEG rows (one block, one request) m = max s, p = 2^(s - m),
// l = sum p, o = sum p V_row -> partial record. Rows outside the step
// (blk_info -1) and unfilled slots of a request's last block get p = 0.
template <int HD, int SEG>
__device__ __forceinline__ void attn_part_tile(const Params& p, uint32_t t_row, int mi, int r_in_tile, int row,
                                               int ni, int lane) {
    constexpr int HPT = 128 / HD;  // heads per tile
    const int bpt = BM / p.tpb;
    const int slot = r_in_tile / p.tpb;
    const int info = row < p.M ? __ldg(p.blk_info + mi * bpt + slot) : -1;
    const int tok = r_in_tile - slot * p.tpb;
    const bool valid = info >= 0 && tok < (info & 0xFF);
    const int req = info >= 0 ? (info >> 8) : 0;
    const int nseg = p.tpb / SEG;
    const int seg = tok / SEG;
    const long long blk = row / p.tpb + p.blk_off;
#pragma unroll 1
    for (int j = 0; j < HPT; ++j) {
        const int h = ni * HPT + j;
        const __half* qp = p.q + static_cast<long long>(req) * p.ldq + h * HD;
        float sc = 0.f;
#pragma unroll 1
        for (int c = 0; c < HD; c += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(t_row + j * HD + c, v);
            float qf[16], bk[16];
            load16(qf, qp + c);
#pragma unroll
            for (int i = 0; i < 16; ++i) bk[i] = 0.f;
            if (p.bias) add16(bk, p.bias + h * HD + c);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) sc = fmaf(qf[i] * p.qscale, round_f16(__uint_as_float(v[i]) + bk[i]), sc);
        }
        if (!valid) sc = -FLT_MAX;
        float m = sc;
#pragma unroll
        for (int off = SEG / 2; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        const float pr = valid ? exp2f(sc - m) : 0.f;
        float l = pr;
#pragma unroll
        for (int off = SEG / 2; off >= 1; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        float* rec = p.part + ((blk * nseg + seg) * p.heads + h) * (HD + 4);
        const bool write = info >= 0 && row < p.M;
        constexpr int NV = 16 / SEG > 1 ? 16 / SEG : 1;
        const bool writer = SEG <= 16 || (lane & (SEG / 16 - 1)) == 0;
#pragma unroll 1
        for (int c = 0; c < HD; c += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(t_row + 128 + j * HD + c, v);
            float bv[16], o[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) bv[i] = 0.f;
            if (p.bias) add16(bv, p.bias + p.d + h * HD + c);
            ptx::tmem_ld_wait();
#pragma unroll
            // rows outside the step / unfilled slots may hold any bits (even NaN): 0 * NaN != 0
            for (int i = 0; i < 16; ++i) o[i] = valid ? pr * round_f16(__uint_as_float(v[i]) + bv[i]) : 0.f;
            int col0;
            seg_reduce_scatter16<SEG>(o, lane, &col0);
            if (write && writer) {
#pragma unroll
                for (int i = 0; i < NV; ++i) rec[c + col0 + i] = o[i];
            }
        }
        if (write && (lane & (SEG - 1)) == 0) {
            rec[HD] = m;
            rec[HD + 1] = l;
        }
    }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_chunk(const Params& p, int row, int col, int split, const uint32_t (&v)[16]) {
    if (row >= p.M || col >= p.N) return;
    if constexpr (EPI == kF32 || EPI == kSplitF32) {
        float* dst = static_cast<float*>(p.out) + static_cast<long long>(row + split * p.M) * p.ldc + col;
#pragma unroll
        for (int j = 0; j < 16; j += 4) ptx::st_global_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
        return;
    } else {
        float add[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) add[j] = 0.f;
        if (p.bias) add16(add, p.bias + col);
        if (p.res) add16(add, p.res + static_cast<long long>(row) * p.ldr + col);
        uint32_t h[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float a = __uint_as_float(v[2 * j]) + add[2 * j], b = __uint_as_float(v[2 * j + 1]) + add[2 * j + 1];
            if constexpr (EPI == kRelu) {
                a = fmaxf(a, 0.f);
                b = fmaxf(b, 0.f);
            }
            h[j] = ptx::pack_f16x2(a, b);
        }
        __half* dst;
        if constexpr (EPI == kKvPaged) {
            const int blk = row / p.tpb + p.blk_off;
            const int t = row - (row / p.tpb) * p.tpb;
            const int part = col / p.d;           // 0 = K, 1 = V
            const int rem = col - part * p.d;
            const int head = rem / p.hd;
            const int c = rem - head * p.hd;
            const long long block_elems = 2LL * p.d * p.tpb;
            dst = static_cast<__half*>(p.out) + blk * block_elems +
                  static_cast<long long>(part) * p.d * p.tpb + static_cast<long long>(head) * p.tpb * p.hd +
                  t * p.hd + c;
        } else {
            dst = static_cast<__half*>(p.out) + static_cast<long long>(row) * p.ldc + col;
        }
        if (p.l2_hint & kL2StreamC) {
            ptx::st_global_cs_v4(dst, h[0], h[1], h[2], h[3]);
            ptx::st_global_cs_v4(dst + 8, h[4], h[5], h[6], h[7]);
        } else {
            ptx::st_global_v4(dst, h[0], h[1], h[2], h[3]);
            ptx::st_global_v4(dst + 8, h[4], h[5], h[6], h[7]);
        }
    }
}

template <int BN, int EPI, int HD = 0, int SEG = 0>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
    using C = Cfg<BN>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * C::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
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

    const int grid_tiles = p.num_m_tiles * p.num_n_tiles;
    const int num_tiles = grid_tiles * p.splits;
    const int num_kb = (p.K + BK - 1) / BK;
    // k-block range of work unit `tile` (whole K unless split-K)
    auto kb_range = [&](int tile, int& kb0, int& kb1) {
        const int s = tile / grid_tiles;
        kb0 = s * p.kb_per_split;
        kb1 = kb0 + p.kb_per_split < num_kb ? kb0 + p.kb_per_split : num_kb;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol_last = ptx::policy_evict_last(), pol_first = ptx::policy_evict_first();
            // operands without a policy bit take plain loads (no cache hint at all)
            auto load_a = [&](void* dst, uint64_t* bar, int k, int row, uint64_t pol) {
                if (p.l2_hint & kL2KeepA)
                    ptx::tma_load_2d_hint(dst, &tmA, bar, k, row, pol);
                else
                    ptx::tma_load_2d(dst, &tmA, bar, k, row);
            };
            auto load_b = [&](void* dst, uint64_t* bar, int k, int row) {
                if (p.l2_hint & kL2StreamB)
                    ptx::tma_load_2d_hint(dst, &tmB, bar, k, row, pol_first);
                else
                    ptx::tma_load_2d(dst, &tmB, bar, k, row);
            };
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int mi, ni, kb0, kb1;
                tile_coords(tile, p, mi, ni);
                kb_range(tile, kb0, kb1);
                const int m_row = p.m_tile_rows ? p.m_tile_rows[mi] : mi * BM;
                const int n_row = ni * BN;
                const uint64_t pol_a = ni == p.num_n_tiles - 1 ? pol_first : pol_last;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    load_a(smem_a + stage * C::kABytes, &full[stage], kb * BK, m_row, pol_a);
                    if constexpr (EPI == kAttnPart) {  // [K_h | V_h]: two 128-row boxes
                        load_b(smem_b + stage * C::kBBytes, &full[stage], kb * BK, ni * 128);
                        load_b(smem_b + stage * C::kBBytes + 128 * BK * 2, &full[stage], kb * BK, p.v_row + ni * 128);
                    } else {
                        load_b(smem_b + stage * C::kBBytes, &full[stage], kb * BK, n_row);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int kb0, kb1;
                kb_range(tile, kb0, kb1);
                ptx::mbar_wait(&tempty[as], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + as * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t a_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_a + stage * C::kABytes));
                    const uint64_t b_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // +32 B per 16-element K step inside the 128 B swizzle atom
                        ptx::mma_f16_ss(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, ((kb - kb0) | k) != 0);
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
            }
        }
    } else {
        const int q = warp % 4;  // TMEM lane quarter this warp may access
        const int r_in_tile = q * 32 + lane;
        int as = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int mi, ni;
            tile_coords(tile, p, mi, ni);
            const int m_row = p.m_tile_rows ? p.m_tile_rows[mi] : mi * BM;
            const int row = m_row + r_in_tile;
            const int n0 = ni * BN;
            const int split = tile / grid_tiles;
            ptx::mbar_wait(&tfull[as], aphase);
            ptx::tc_fence_after();
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN;
            if constexpr (EPI == kAttnPart) {
                static_assert(BN == 256, "kAttnPart tiles are [K_h | V_h], 128 + 128 columns");
                attn_part_tile<HD, SEG>(p, t_row, mi, r_in_tile, row, ni, lane);
            } else {
#pragma unroll 1
                for (int c = 0; c < BN; c += 16) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(t_row + c, v);
                    ptx::tmem_ld_wait();
                    epilogue_chunk<BN, EPI>(p, row, n0 + c, split, v);
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

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for large M: a 2-CTA cluster computes a
// 256 x 256 tile with one UMMA M=256 stream issued by the leader CTA. Each CTA
// TMA-loads its own 128 rows of A and 128 rows (N) of B per stage, so the
// smem/L2 traffic per MAC drops by a third vs the 1-SM 128 x 256 tile — the
// large-M GEMMs (ACT recompute, prefill) are L2-feed bound otherwise.
// M tiles are counted in 128-row units (m_tile_rows lists pair up
// consecutively; an odd tail repeats the last tile, writing identical values).
struct Cfg2 {
    static constexpr int BN = 256;
    static constexpr int kABytes = BM * BK * 2;          // 128 rows of A per CTA
    static constexpr int kBBytes = (BN / 2) * BK * 2;    // 128 rows of B per CTA
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = 6;
    static constexpr int kTmemCols = 512;                // 2 x 256 accumulator columns
    static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 16;
    static constexpr int kSmemBytes = kStages * kStageBytes + kBarBytes + 1024;
};

__device__ __forceinline__ void pair_tile_coords(int tile, int num_pm, int num_n, int group, int group_n, int& pm,
                                                 int& ni) {
    if (group_n > 0) {  // weight-stationary raster (see tile_coords)
        const int G = num_n < group_n ? num_n : group_n;
        const int per = G * num_pm;
        const int g = tile / per;
        const int first = g * G;
        const int gn = (num_n - first) < G ? (num_n - first) : G;
        const int within = tile - g * per;
        ni = first + within % gn;
        pm = within / gn;
        return;
    }
    const int G = num_pm < group ? num_pm : group;
    const int per = G * num_n;
    const int g = tile / per;
    const int first = g * G;
    const int gm = (num_pm - first) < G ? (num_pm - first) : G;
    const int within = tile - g * per;
    pm = first + within % gm;
    ni = within / gm;
}

template <int EPI, int HD = 0, int SEG = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const Params p) {
    using C = Cfg2;
    constexpr int S = C::kStages;
    constexpr int BN = C::BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * C::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const int pair = blockIdx.x / 2;
    const int num_pairs = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], 256);  // both CTAs' epilogues arrive on the leader's
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_pair<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_pm = (p.num_m_tiles + 1) / 2;
    const int num_tiles = num_pm * p.num_n_tiles;
    const int num_kb = (p.K + BK - 1) / BK;
    auto m_row_of = [&](int pm, uint32_t r) {
        int t = 2 * pm + static_cast<int>(r);
        if (p.m_tile_rows) {
            if (t >= p.num_m_tiles) t = p.num_m_tiles - 1;
            return p.m_tile_rows[t];
        }
        return t * BM;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol_last = ptx::policy_evict_last(), pol_first = ptx::policy_evict_first();
            for (int tile = pair; tile < num_tiles; tile += num_pairs) {
                int pm, ni;
                pair_tile_coords(tile, num_pm, p.num_n_tiles, p.group_m, p.group_n, pm, ni);
                const int m_row = m_row_of(pm, rank);
                // kAttnPart: rank 0 loads K_h rows, rank 1 the V_h rows of the heads
                const int n_row = EPI == kAttnPart ? (rank ? p.v_row : 0) + ni * 128
                                                   : ni * BN + static_cast<int>(rank) * (BN / 2);
                const uint64_t pol_a = ni == p.num_n_tiles - 1 ? pol_first : pol_last;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
                    if (p.l2_hint & kL2KeepA)
                        ptx::tma_load_2d_pair_hint(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * BK, m_row,
                                                   pol_a);
                    else
                        ptx::tma_load_2d_pair(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * BK, m_row);
                    if (p.l2_hint & kL2StreamB)
                        ptx::tma_load_2d_pair_hint(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n_row,
                                                   pol_first);
                    else
                        ptx::tma_load_2d_pair(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n_row);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            for (int tile = pair; tile < num_tiles; tile += num_pairs) {
                ptx::mbar_wait(&tempty[as], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + as * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t a_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_a + stage * C::kABytes));
                    const uint64_t b_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        ptx::mma_f16_ss_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
                    ptx::mma_commit_pair_mc(&empty[stage], 0x3);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_pair_mc(&tfull[as], 0x3);
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1;
                }
            }
        }
    } else {
        const int q = warp % 4;
        int as = 0;
        uint32_t aphase = 0;
        for (int tile = pair; tile < num_tiles; tile += num_pairs) {
            int pm, ni;
            pair_tile_coords(tile, num_pm, p.num_n_tiles, p.group_m, p.group_n, pm, ni);
            const int row = m_row_of(pm, rank) + q * 32 + lane;
            const int n0 = ni * BN;
            ptx::mbar_wait(&tfull[as], aphase);
            ptx::tc_fence_after();
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN;
            if constexpr (EPI == kAttnPart) {
                int mt = 2 * pm + static_cast<int>(rank);  // this CTA's 128-row M tile (odd tail repeats the last)
                if (mt >= p.num_m_tiles) mt = p.num_m_tiles - 1;
                const bool dup = 2 * pm + static_cast<int>(rank) >= p.num_m_tiles;
                if (!dup) attn_part_tile<HD, SEG>(p, t_row, mt, q * 32 + lane, row, ni, lane);
            } else {
#pragma unroll 1
                for (int c = 0; c < BN; c += 16) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(t_row + c, v);
                    ptx::tmem_ld_wait();
                    epilogue_chunk<BN, EPI>(p, row, n0 + c, 0, v);
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive_cluster(&tempty[as], 0);
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
        }
    }

    __syncthreads();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<C::kTmemCols>(tmem_base);
    }
}

}  // namespace hc::gemm
