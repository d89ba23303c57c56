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
#pragma once
#include <cuda.h>
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
};

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
        ptx::st_global_v4(dst, h[0], h[1], h[2], h[3]);
        ptx::st_global_v4(dst + 8, h[4], h[5], h[6], h[7]);
    }
}

template <int BN, int EPI>
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
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int mi, ni, kb0, kb1;
                tile_coords(tile, p, mi, ni);
                kb_range(tile, kb0, kb1);
                const int m_row = p.m_tile_rows ? p.m_tile_rows[mi] : mi * BM;
                const int n_row = ni * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                    ptx::tma_load_2d(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * BK, m_row);
                    ptx::tma_load_2d(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n_row);
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
#pragma unroll 1
            for (int c = 0; c < BN; c += 16) {
                uint32_t v[16];
                ptx::tmem_ld_x16(t_row + c, v);
                ptx::tmem_ld_wait();
                epilogue_chunk<BN, EPI>(p, row, n0 + c, split, v);
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

template <int EPI>
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
            for (int tile = pair; tile < num_tiles; tile += num_pairs) {
                int pm, ni;
                pair_tile_coords(tile, num_pm, p.num_n_tiles, p.group_m, p.group_n, pm, ni);
                const int m_row = m_row_of(pm, rank);
                const int n_row = ni * BN + static_cast<int>(rank) * (BN / 2);
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
                    ptx::tma_load_2d_pair(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * BK, m_row);
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
#pragma unroll 1
            for (int c = 0; c < BN; c += 16) {
                uint32_t v[16];
                ptx::tmem_ld_x16(t_row + c, v);
                ptx::tmem_ld_wait();
                epilogue_chunk<BN, EPI>(p, row, n0 + c, 0, v);
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
