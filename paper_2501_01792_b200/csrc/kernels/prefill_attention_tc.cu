// Causal prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA),
// head_dim 128 (attention_causal, decoder.cpp:55-63). Two kernels:
//   prefill_tc2_kernel (default) — persistent, pairs of query tiles, two
//                                  softmax warpgroups (see its header below)
//   prefill_tc_kernel  (HC_PREFILL_TC=1) — one query tile per CTA:
//
// One CTA per (128-query tile, head, request); 192 threads:
//   warp 0      TMA producer: Q once, then K|V tiles of 128 keys into a
//               2-stage ring (one tensor map over the packed Q|K|V rows)
//   warp 1      TMEM owner + single-thread MMA issuer:
//                 S[j%2] = Q . K_j^T        (M=128, N=128 keys, K=hd)
//                 O     += P_j . V_j        (M=128, N=hd, K=128 keys; V read
//                                            MN-major straight from its tile)
//               S_{j+1} is issued before P_j arrives, so the QK^T of the next
//               tile overlaps the softmax of this one (two S buffers in TMEM)
//   warps 2..5  softmax: thread = query row = TMEM lane; S row via tcgen05.ld,
//               causal / ragged mask, online max in the exp2 domain with a
//               lazy O correction (only when the max grows by > 2^8, so P
//               stays <= 256 and O is rescaled in TMEM rarely), P (f16) into
//               a 128B-swizzled K-major smem tile for the P.V MMA; finally
//               O / l from TMEM to HBM.
// TMEM: S0 | S1 | O = 384 of 512 columns. smem: Q 32 KB, 2 x (K 32 + V 32) KB,
// 2 x P 32 KB = 224 KB -> one CTA per SM; with two P buffers the softmax of
// tile j writes P while P.V(j-1) still runs. Heavy (late) query tiles first.
#include <cuda.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"
#include "launch.hpp"
#include "ptx.cuh"
#include "tma.hpp"

namespace hc {

namespace {

constexpr int kT = 128;        // queries per CTA = keys per tile
constexpr int kHD = 128;       // head dim
constexpr int kBox = kT * 64 * 2;           // one [128 rows][64 cols] f16 box = 16 KB
constexpr int kTile = 2 * kBox;             // [128][128] = 32 KB
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;            // lazy correction threshold (log2 units)

struct Smem {
    static constexpr int q = 0;
    static constexpr int k = kTile;                       // stage s at k + s * 2 * kTile
    static constexpr int v = 2 * kTile;                   // stage s at v + s * 2 * kTile
    static constexpr int p = (1 + 2 * kStages) * kTile;    // P buffer b at p + b * kTile
    static constexpr int bars = p + 2 * kTile;
    static constexpr int bytes = bars + 256 + 1024;       // + barrier block + 1 KB alignment slack
};

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// exp2 on the MUFU (ex2.approx.ftz; arguments are <= 8 by the lazy correction, masked ones -> 0)
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// packed fp32x2 FMA / add (FFMA2 / FADD2 on sm_100): half the issue slots of
// the softmax's per-element scale-and-subtract and row-sum work
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 %0, ra, rb, rc;\n\t}"
        : "=l"(d)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("{\n\t.reg .b64 ra, rb;\n\t"
        "mov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
        "add.rn.f32x2 %0, ra, rb;\n\t}"
        : "=l"(d)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// MN-major, 128B-swizzled operand (V: rows = K (keys), 64 N (hd) per 128 B row):
// SBO = 1024 B between 8-row (K) groups, LBO = 16 KB between 64-wide N boxes.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

__global__ void __launch_bounds__(kThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm, f16* __restrict__ out, const int* __restrict__ cu,
                      int H, float scale, uint32_t v_lbo, uint32_t v_sbo) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;      // [kStages]
    uint64_t* kv_empty = bars + 3;     // [kStages]
    uint64_t* s_full = bars + 5;       // [2]
    uint64_t* s_free = bars + 7;       // [2]
    uint64_t* p_full = bars + 9;       // [2] (per P buffer)
    uint64_t* pv_done = bars + 11;     // [2] (per P buffer)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const int req = blockIdx.z, h = blockIdx.y;
    const int row0 = cu[req];
    const int P = cu[req + 1] - row0;
    const int n_qt = (P + kT - 1) / kT;
    const int qt = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);
    if (qt >= n_qt) return;
    const int q0 = qt * kT;
    const int n_kt = qt + 1;  // causal: key tiles 0..qt (q and key tiles aligned)
    const int d = H * kHD;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tm);
        ptx::mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&kv_full[s], 1);
            ptx::mbar_init(&kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&s_full[b], 1);
            ptx::mbar_init(&s_free[b], 128);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&p_full[b], 128);
            ptx::mbar_init(&pv_done[b], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    auto t_s = [&](int b) { return tmem + 128u * static_cast<uint32_t>(b); };  // S double buffer
    const uint32_t t_o = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------------- TMA producer
            const int qc = h * kHD, kc = d + h * kHD, vc = 2 * d + h * kHD;
            ptx::mbar_arrive_expect_tx(q_full, kTile);
            ptx::tma_load_2d(smem + Smem::q, &tm, q_full, qc, row0 + q0);
            ptx::tma_load_2d(smem + Smem::q + kBox, &tm, q_full, qc + 64, row0 + q0);
            for (int j = 0; j < n_kt; ++j) {
                const int s = j % kStages;
                ptx::mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
                uint8_t* kb = smem + Smem::k + s * 2 * kTile;
                uint8_t* vb = smem + Smem::v + s * 2 * kTile;
                ptx::mbar_arrive_expect_tx(&kv_full[s], 2 * kTile);
                const int r = row0 + j * kT;
                ptx::tma_load_2d(kb, &tm, &kv_full[s], kc, r);
                ptx::tma_load_2d(kb + kBox, &tm, &kv_full[s], kc + 64, r);
                ptx::tma_load_2d(vb, &tm, &kv_full[s], vc, r);
                ptx::tma_load_2d(vb + kBox, &tm, &kv_full[s], vc + 64, r);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ------------------------------------------ MMA issuer
            constexpr uint32_t id_s = ptx::idesc_f16_f32(kT, kT);               // A, B K-major
            constexpr uint32_t id_o = ptx::idesc_f16_f32(kT, kHD) | (1u << 16);  // B MN-major (V)
            const uint32_t qa = ptx::smem_u32(smem + Smem::q);
            const uint32_t pa = ptx::smem_u32(smem + Smem::p);
            auto issue_s = [&](int j) {
                const int s = j % kStages, b = j & 1;
                ptx::mbar_wait(&kv_full[s], (j / kStages) & 1);
                if (j >= 2) ptx::mbar_wait(&s_free[b], ((j - 2) / 2) & 1);
                ptx::tc_fence_after();
                const uint32_t kb = ptx::smem_u32(smem + Smem::k + s * 2 * kTile);
#pragma unroll
                for (int k = 0; k < kHD / 16; ++k) {  // hd in two 64-wide boxes, 4 k-steps each
                    const uint32_t off = (k / 4) * kBox;
                    ptx::mma_f16_ss(t_s(b), ptx::sw128_kmajor_desc(qa + off) + 2 * (k % 4),
                                     ptx::sw128_kmajor_desc(kb + off) + 2 * (k % 4), id_s, k > 0);
                }
                ptx::mma_commit(&s_full[b]);
            };
            ptx::mbar_wait(q_full, 0);
            issue_s(0);
            for (int j = 0; j < n_kt; ++j) {
                if (j + 1 < n_kt) issue_s(j + 1);
                const int pb = j & 1;
                ptx::mbar_wait(&p_full[pb], (j / 2) & 1);
                ptx::tc_fence_after();
                const int s = j % kStages;
                const uint32_t vb = ptx::smem_u32(smem + Smem::v + s * 2 * kTile);
                const uint32_t pbuf = pa + pb * kTile;
#pragma unroll
                for (int k = 0; k < kT / 16; ++k) {  // keys: P in two 64-wide boxes; V rows 16 per step
                    const uint64_t a = ptx::sw128_kmajor_desc(pbuf + (k / 4) * kBox) + 2 * (k % 4);
                    const uint64_t bdesc = sw128_mnmajor_desc(vb + k * 16 * 128, v_lbo, v_sbo);
                    ptx::mma_f16_ss(t_o, a, bdesc, id_o, (j > 0 || k > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&pv_done[pb]);
                ptx::mma_commit(&kv_empty[s]);
            }
        }
    } else {  // ----------------------------------------------------- softmax
        const int q = warp % 4;
        const int r = q * 32 + lane;            // query row within the tile = TMEM lane
        const int qrow = q0 + r;                // row within the request
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const float sl = scale * kLog2e;
        float m = -FLT_MAX, l = 0.f;
        const uint32_t prow = ptx::smem_u32(smem + Smem::p);
        for (int j = 0; j < n_kt; ++j) {
            const int b = j & 1;
            ptx::mbar_wait(&s_full[b], (j / 2) & 1);
            ptx::tc_fence_after();
            // the whole S row in one batch of TMEM loads, one wait
            uint32_t sraw[kT];
#pragma unroll
            for (int c = 0; c < kT; c += 16)
                ptx::tmem_ld_x16(t_s(b) + lane_off + c, *reinterpret_cast<uint32_t(*)[16]>(&sraw[c]));
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&s_free[b]);
            const int k0 = j * kT;
            const bool diag = j == n_kt - 1 || k0 + kT > P;
            // 8 independent max / sum chains (a single chain is 128 dependent ops)
            float mx8[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) mx8[t] = -FLT_MAX;
#pragma unroll
            for (int i = 0; i < kT; ++i) {
                float x = __uint_as_float(sraw[i]) * sl;
                if (diag && (k0 + i > qrow || k0 + i >= P)) x = -FLT_MAX;
                sraw[i] = __float_as_uint(x);
                mx8[i % 8] = fmaxf(mx8[i % 8], x);
            }
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
            // lazy correction: keep the reference max unless it grows by > 2^8
            float alpha = 1.f;
            bool rescale = false;
            if (mx > m + kRescale || j == 0) {
                alpha = ex2(m - mx);
                rescale = j > 0;
                m = mx;
                l *= alpha;
            }
            // P = exp2(s - m) as packed f16, computed while P.V(j-1) still runs
            uint32_t pw[kT / 2];
            float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < kT / 2; ++i) {
                const float p0 = ex2(__uint_as_float(sraw[2 * i]) - m), p1 = ex2(__uint_as_float(sraw[2 * i + 1]) - m);
                l8[i % 8] += p0 + p1;
                pw[i] = ptx::pack_f16x2(p0, p1);
            }
            l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
            // P buffer j%2 is free once P.V(j-2) has completed; O may be
            // rescaled only after P.V(j-1) (the rare lazy correction)
            const int pb = j & 1;
            if (j >= 2) {
                ptx::mbar_wait(&pv_done[pb], ((j - 2) / 2) & 1);
                ptx::tc_fence_after();
            }
            if (rescale) {
                ptx::mbar_wait(&pv_done[pb ^ 1], ((j - 1) / 2) & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < kHD; c += 16) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(t_o + lane_off + c, v);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                    tmem_st_x16(t_o + lane_off + c, v);
                }
                tmem_st_wait();
            }
            // P row -> two 64-key 128B-swizzled K-major boxes of buffer pb
            const uint32_t pbase = prow + pb * kTile + (r / 8) * 1024 + (r % 8) * 128;
#pragma unroll
            for (int c = 0; c < kT / 8; ++c) {  // 16-byte chunks of 8 keys
                const int box = c / 8, ch = c % 8;
                sts128(pbase + box * kBox + ((ch ^ (r % 8)) * 16), pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
            }
            fence_async_smem();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&p_full[pb]);
        }
        // O / l -> HBM
        ptx::mbar_wait(&pv_done[(n_kt - 1) & 1], ((n_kt - 1) / 2) & 1);
        ptx::tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        f16* orow = out + static_cast<long long>(row0 + qrow) * d + h * kHD;
#pragma unroll 1
        for (int c = 0; c < kHD; c += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(t_o + lane_off + c, v);
            ptx::tmem_ld_wait();
            uint32_t o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                o[i] = ptx::pack_f16x2(__uint_as_float(v[2 * i]) * inv, __uint_as_float(v[2 * i + 1]) * inv);
            if (qrow < P) {
                ptx::st_global_v4(orow + c, o[0], o[1], o[2], o[3]);
                ptx::st_global_v4(orow + c + 8, o[4], o[5], o[6], o[7]);
            }
        }
        ptx::tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------------------
// Two-tile persistent variant (default). A work item is a PAIR of 128-query
// tiles of one (request, head); one CTA per SM walks the items heaviest pair
// first (static stride). 320 threads:
//   warps 0..3  softmax of query tile 0 of the item (rows q0 .. q0+127)
//   warps 4..7  softmax of query tile 1 (rows q0+128 .. q0+255)
//   warp 8      TMA producer: Q0|Q1, then K_j, V_j into a 3-slot ring; the
//               next item's Q and K/V load while this item finishes
//   warp 9      TMEM owner + MMA issuer, ping-pong between the tiles:
//                 PV0(j), S0(j+1), PV1(j), S1(j+1)
//               so the tensor core runs tile 1's MMAs while tile 0's softmax
//               works and vice versa (one softmax group alone leaves the
//               tensor pipe idle ~80 % of the time); the next item's first
//               QK^T runs while the softmax warps write this item's O.
// TMEM: S0 | S1 | O0 | O1 = 512 columns. smem: Q0, Q1, P0, P1, 3 K/V slots of
// 32 KB = 224 KB. With one S and one P buffer per tile no free barriers are
// needed inside an item: the commit that signals S_t(j) also covers PV_t(j-1)
// (tcgen05 operations of one thread complete in issue order), so when the
// softmax sees S_t(j) both P_t and O_t are free to write. Across items: Q is
// reloaded after the item's last QK^T (q_empty), O_t is overwritten only after
// the softmax has read it out (o_free). Barrier phases run on per-role
// counters that continue across items.
constexpr int kSlots2 = 3;
constexpr int kThreads2 = 320;

// head_dim 64 has the smem for a second P buffer per tile: P = P_hi + P_lo (both
// f16, P_lo = f16(p - P_hi)) and O += P_hi V + P_lo V keeps P to ~16 mantissa
// bits, as the mma.sync kernel's hi/lo split does — halving the head dim
// doubles the weight of the P rounding per output (12-layer OPT-125M traces).
template <int HD>
struct Smem2 {
    static constexpr bool lo = HD == 64;
    static constexpr int qkv = kT * HD * 2;     // one Q / K / V tile: HD / 64 boxes of [128 rows][64 cols]
    static constexpr int q = 0;                 // tile t at q + t * qkv
    static constexpr int p = 2 * qkv;           // tile t at p + t * kTile (P is [128 queries][128 keys])
    static constexpr int kv = p + 2 * kTile;    // slot s at kv + s * qkv
    static constexpr int plo = kv + kSlots2 * qkv;  // P_lo of tile t at plo + t * kTile (head_dim 64)
    static constexpr int bars = plo + (lo ? 2 * kTile : 0);
    static constexpr int bytes = bars + 256 + 1024;
};
static_assert(Smem2<64>::bytes <= 232448, "prefill_tc2<64>: shared memory over the per-CTA limit");
static_assert(Smem2<128>::bytes <= 232448, "prefill_tc2: shared memory over the per-CTA limit");

struct Item {  // one (request, head, query-tile pair)
    int row0, P, h, qt0, n0, n1, n_kt;
    bool has1;
};
// heaviest pairs first: item w -> pair n_pairs-1 - w / (H n_req); false if the
// pair lies beyond its request (every role skips it identically)
__device__ __forceinline__ bool item_of(int w, int n_pairs, int H, int n_req, const int* cu, Item& it) {
    const int per = H * n_req;
    const int pair = n_pairs - 1 - w / per, rem = w % per;
    it.h = rem % H;
    const int req = rem / H;
    it.row0 = cu[req];
    it.P = cu[req + 1] - it.row0;
    const int n_qt = (it.P + kT - 1) / kT;
    it.qt0 = 2 * pair;
    if (it.qt0 >= n_qt) return false;
    it.has1 = it.qt0 + 1 < n_qt;
    it.n0 = it.qt0 + 1;  // causal key tiles per query tile
    it.n1 = it.has1 ? it.qt0 + 2 : 0;
    it.n_kt = it.has1 ? it.n1 : it.n0;
    return true;
}

// PT: P_t is written into TMEM over S_t's first columns (packed f16 pairs;
// P_lo after it at head_dim 64) and O += P V reads it from there (tcgen05.mma
// with A in TMEM) instead of a swizzled smem tile: no smem stores, no async-proxy
// fence, no smem reads of P by the tensor core. S_t is in registers by then, and
// S_t(j+1) is issued after PV_t(j) by the same thread (in-order completion).
template <int HD, bool PT = false>  // head_dim 64 or 128
__global__ void __launch_bounds__(kThreads2, 1)
    prefill_tc2_kernel(const __grid_constant__ CUtensorMap tm, f16* __restrict__ out, const int* __restrict__ cu,
                       int n_req, int n_pairs, int H, float scale, uint32_t v_lbo, uint32_t v_sbo) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem2<HD>::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;   // [kSlots2]
    uint64_t* kv_empty = bars + 5;  // [kSlots2]
    uint64_t* s_full = bars + 8;    // [2] per tile
    uint64_t* p_full = bars + 10;   // [2] per tile
    uint64_t* o_done = bars + 12;   // [2] per tile
    uint64_t* o_free = bars + 14;   // [2] per tile
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

    const int n_items = n_pairs * H * n_req;
    const int d = H * HD;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tm);
        ptx::mbar_init(q_full, 1);
        ptx::mbar_init(q_empty, 1);
        for (int s = 0; s < kSlots2; ++s) {
            ptx::mbar_init(&kv_full[s], 1);
            ptx::mbar_init(&kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            ptx::mbar_init(&s_full[t], 1);
            ptx::mbar_init(&p_full[t], 128);
            ptx::mbar_init(&o_done[t], 1);
            ptx::mbar_init(&o_free[t], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 9) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 8) {
        if (lane == 0) {  // ---------------------------------------- TMA producer
            uint32_t ring = 0, n_it = 0;
            for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
                Item it;
                if (!item_of(w, n_pairs, H, n_req, cu, it)) continue;
                const int qc = it.h * HD, kc = d + it.h * HD, vc = 2 * d + it.h * HD;
                if (n_it > 0) ptx::mbar_wait(q_empty, (n_it - 1) & 1);  // last QK^T of the previous item done
                ptx::mbar_arrive_expect_tx(q_full, it.has1 ? 2 * Smem2<HD>::qkv : Smem2<HD>::qkv);
                for (int t = 0; t < (it.has1 ? 2 : 1); ++t) {
                    uint8_t* qb = smem + Smem2<HD>::q + t * Smem2<HD>::qkv;
                    for (int bx = 0; bx < HD / 64; ++bx)
                        ptx::tma_load_2d(qb + bx * kBox, &tm, q_full, qc + 64 * bx, it.row0 + (it.qt0 + t) * kT);
                }
                for (int i = 0; i < 2 * it.n_kt; ++i) {  // K_0, V_0, K_1, V_1, ...
                    const uint32_t g = ring + i, s = g % kSlots2;
                    ptx::mbar_wait(&kv_empty[s], ((g / kSlots2) & 1) ^ 1);
                    uint8_t* b = smem + Smem2<HD>::kv + s * Smem2<HD>::qkv;
                    ptx::mbar_arrive_expect_tx(&kv_full[s], Smem2<HD>::qkv);
                    const int c = (i & 1) ? vc : kc, r = it.row0 + (i / 2) * kT;
                    for (int bx = 0; bx < HD / 64; ++bx)
                        ptx::tma_load_2d(b + bx * kBox, &tm, &kv_full[s], c + 64 * bx, r);
                }
                ring += 2 * it.n_kt;
                ++n_it;
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {  // ------------------------------------------ MMA issuer
            constexpr uint32_t id_s = ptx::idesc_f16_f32(kT, kT);               // A, B K-major
            constexpr uint32_t id_o = ptx::idesc_f16_f32(kT, HD) | (1u << 16);  // B MN-major (V)
            uint32_t ring = 0, n_it = 0, pc[2] = {0, 0}, oc[2] = {0, 0};
            auto slot_addr = [&](uint32_t g) { return ptx::smem_u32(smem + Smem2<HD>::kv + (g % kSlots2) * Smem2<HD>::qkv); };
            auto s_mma = [&](int t, uint32_t g) {  // S_t = Q_t . K^T, K at ring entry g
                ptx::mbar_wait(&kv_full[g % kSlots2], (g / kSlots2) & 1);
                ptx::tc_fence_after();
                const uint32_t qa = ptx::smem_u32(smem + Smem2<HD>::q + t * Smem2<HD>::qkv), kb = slot_addr(g);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint32_t off = (k / 4) * kBox;
                    ptx::mma_f16_ss(tmem + 128u * t, ptx::sw128_kmajor_desc(qa + off) + 2 * (k % 4),
                                     ptx::sw128_kmajor_desc(kb + off) + 2 * (k % 4), id_s, k > 0);
                }
                ptx::mma_commit(&s_full[t]);
            };
            auto pv_mma = [&](int t, uint32_t g, bool first) {  // O_t += P_t . V, V at ring entry g
                ptx::mbar_wait(&kv_full[g % kSlots2], (g / kSlots2) & 1);
                if (first && oc[t] > 0) ptx::mbar_wait(&o_free[t], (oc[t] - 1) & 1);  // previous O_t read out
                ptx::mbar_wait(&p_full[t], pc[t] & 1);
                ++pc[t];
                ptx::tc_fence_after();
                const uint32_t pa = ptx::smem_u32(smem + Smem2<HD>::p + t * kTile), vb = slot_addr(g);
                const uint32_t d_o = tmem + 256u + static_cast<uint32_t>(HD) * t;
#pragma unroll
                for (int k = 0; k < kT / 16; ++k) {
                    const uint64_t bdesc = sw128_mnmajor_desc(vb + k * 16 * 128, v_lbo, v_sbo);
                    if constexpr (PT) {
                        ptx::mma_f16_ts(d_o, tmem + 128u * t + 8u * k, bdesc, id_o, (!first || k > 0) ? 1u : 0u);
                    } else {
                        const uint64_t a = ptx::sw128_kmajor_desc(pa + (k / 4) * kBox) + 2 * (k % 4);
                        ptx::mma_f16_ss(d_o, a, bdesc, id_o, (!first || k > 0) ? 1u : 0u);
                    }
                }
                if constexpr (Smem2<HD>::lo) {  // + P_lo . V
                    const uint32_t pl = ptx::smem_u32(smem + Smem2<HD>::plo + t * kTile);
#pragma unroll
                    for (int k = 0; k < kT / 16; ++k) {
                        const uint64_t bdesc = sw128_mnmajor_desc(vb + k * 16 * 128, v_lbo, v_sbo);
                        if constexpr (PT) {
                            ptx::mma_f16_ts(d_o, tmem + 128u * t + 64u + 8u * k, bdesc, id_o, 1u);
                        } else {
                            const uint64_t a = ptx::sw128_kmajor_desc(pl + (k / 4) * kBox) + 2 * (k % 4);
                            ptx::mma_f16_ss(d_o, a, bdesc, id_o, 1u);
                        }
                    }
                }
            };
            for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
                Item it;
                if (!item_of(w, n_pairs, H, n_req, cu, it)) continue;
                const int n0 = it.n0, n1 = it.n1, n_kt = it.n_kt;
                ptx::mbar_wait(q_full, n_it & 1);
                s_mma(0, ring);
                if (n1) s_mma(1, ring);
                ptx::mma_commit(&kv_empty[ring % kSlots2]);  // K_0 consumed
                if (n_kt == 1) ptx::mma_commit(q_empty);       // last QK^T of the item issued
                for (int j = 0; j < n_kt; ++j) {
                    const uint32_t gk = ring + 2 * j + 2, gv = ring + 2 * j + 1;  // K_{j+1}, V_j
                    if (j < n0) {
                        pv_mma(0, gv, j == 0);
                        if (j + 1 == n0) ptx::mma_commit(&o_done[0]);
                    }
                    if (j + 1 < n0) s_mma(0, gk);
                    if (j < n1) {
                        pv_mma(1, gv, j == 0);
                        if (j + 1 == n1) ptx::mma_commit(&o_done[1]);
                    }
                    ptx::mma_commit(&kv_empty[gv % kSlots2]);  // V_j consumed
                    if (j + 1 < n1) s_mma(1, gk);
                    if (j + 1 < n_kt) {
                        ptx::mma_commit(&kv_empty[gk % kSlots2]);  // K_{j+1} consumed
                        if (j + 2 == n_kt) ptx::mma_commit(q_empty);
                    }
                }
                ++oc[0];
                if (n1) ++oc[1];
                ring += 2 * n_kt;
                ++n_it;
            }
        }
    } else {  // ------------------------------------------------------------- softmax
        const int t = warp / 4;
        const int q = warp % 4;
        const int r = q * 32 + lane;  // query row within the tile = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t t_s = tmem + 128u * t, t_o = tmem + 256u + static_cast<uint32_t>(HD) * t;
        const float sl = scale * kLog2e;
        const uint32_t pbase = ptx::smem_u32(smem + Smem2<HD>::p + t * kTile) + (r / 8) * 1024 + (r % 8) * 128;
        uint32_t sc = 0, oc = 0;
        for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
            Item it;
            if (!item_of(w, n_pairs, H, n_req, cu, it)) continue;
            if (t == 1 && !it.has1) continue;
            const int P = it.P, n = t ? it.n1 : it.n0;
            const int qrow = (it.qt0 + t) * kT + r;  // row within the request
            float m = -FLT_MAX, l = 0.f;              // running max (scaled log2 domain) and sum
            for (int j = 0; j < n; ++j) {
                ptx::mbar_wait(&s_full[t], sc & 1);
                ++sc;
                ptx::tc_fence_after();
                uint32_t sraw[kT];
#pragma unroll
                for (int c = 0; c < kT; c += 16)
                    ptx::tmem_ld_x16(t_s + lane_off + c, *reinterpret_cast<uint32_t(*)[16]>(&sraw[c]));
                ptx::tmem_ld_wait();
                const int k0 = j * kT;
                if (j == n - 1 || k0 + kT > P) {
#pragma unroll
                    for (int i = 0; i < kT; ++i)
                        if (k0 + i > qrow || k0 + i >= P) sraw[i] = __float_as_uint(-FLT_MAX);
                }
                float mx8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) mx8[u] = -FLT_MAX;
#pragma unroll
                for (int i = 0; i < kT; ++i) mx8[i % 8] = fmaxf(mx8[i % 8], __uint_as_float(sraw[i]));
                const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                const float mx = mraw == -FLT_MAX ? -FLT_MAX : mraw * sl;
                float alpha = 1.f;
                bool rescale = false;
                if (mx > m + kRescale || j == 0) {  // lazy correction (see prefill_tc_kernel)
                    alpha = ex2(m - mx);
                    rescale = j > 0;
                    m = mx;
                    l *= alpha;
                }
                // p = 2^(s * sl - m) in one FFMA + MUFU; masked entries (-FLT_MAX * sl) underflow to 0.
                // Each 8-key chunk goes to the 128B-swizzled P tile as soon as it is packed
                // (P_t is free: S_t(j) completing implies PV_t(j-1) did), so only one chunk
                // of packed words is live at a time.
                float2 l4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                const float2 sl2 = make_float2(sl, sl), nm2 = make_float2(-m, -m);
                uint32_t pt16[16], plt16[16];  // PT: 32 keys of packed P (and P_lo) per tcgen05.st
#pragma unroll
                for (int c = 0; c < kT / 8; ++c) {
                    uint32_t pw[4], plw[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = 4 * c + u;
                        const float2 y = ffma2(make_float2(__uint_as_float(sraw[2 * i]), __uint_as_float(sraw[2 * i + 1])),
                                               sl2, nm2);
                        const float2 pp = make_float2(ex2(y.x), ex2(y.y));
                        l4[u] = fadd2(l4[u], pp);
                        pw[u] = ptx::pack_f16x2(pp.x, pp.y);
                        if constexpr (Smem2<HD>::lo) {  // the f16 residual of each P entry
                            const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&pw[u]));
                            plw[u] = ptx::pack_f16x2(pp.x - h.x, pp.y - h.y);
                        }
                    }
                    if constexpr (PT) {  // P over S_t's columns [0, 64), P_lo over [64, 128)
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            pt16[(c % 4) * 4 + u] = pw[u];
                            if constexpr (Smem2<HD>::lo) plt16[(c % 4) * 4 + u] = plw[u];
                        }
                        if (c % 4 == 3) {
                            tmem_st_x16(t_s + lane_off + 16u * (c / 4), pt16);
                            if constexpr (Smem2<HD>::lo) tmem_st_x16(t_s + lane_off + 64u + 16u * (c / 4), plt16);
                        }
                    } else {
                        const int box = c / 8, ch = c % 8;
                        const uint32_t dst = pbase + box * kBox + ((ch ^ (r % 8)) * 16);
                        sts128(dst, pw[0], pw[1], pw[2], pw[3]);
                        if constexpr (Smem2<HD>::lo)
                            sts128(dst + (Smem2<HD>::plo - Smem2<HD>::p), plw[0], plw[1], plw[2], plw[3]);
                    }
                }
                const float2 ls = fadd2(fadd2(l4[0], l4[1]), fadd2(l4[2], l4[3]));
                l += ls.x + ls.y;
                if (rescale) {  // PV_t(j-1) completed before S_t(j) was signalled
#pragma unroll 1
                    for (int c = 0; c < HD; c += 16) {
                        uint32_t v[16];
                        ptx::tmem_ld_x16(t_o + lane_off + c, v);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                        tmem_st_x16(t_o + lane_off + c, v);
                    }
                    tmem_st_wait();
                }
                if constexpr (PT)
                    tmem_st_wait();  // P is in TMEM before the MMA lane is told
                else
                    fence_async_smem();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&p_full[t]);
            }
            ptx::mbar_wait(&o_done[t], oc & 1);
            ++oc;
            ptx::tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            f16* orow = out + static_cast<long long>(it.row0 + qrow) * d + it.h * HD;
#pragma unroll 1
            for (int c = 0; c < HD; c += 16) {
                uint32_t v[16];
                ptx::tmem_ld_x16(t_o + lane_off + c, v);
                ptx::tmem_ld_wait();
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    o[i] = ptx::pack_f16x2(__uint_as_float(v[2 * i]) * inv, __uint_as_float(v[2 * i + 1]) * inv);
                if (qrow < P) {
                    ptx::st_global_v4(orow + c, o[0], o[1], o[2], o[3]);
                    ptx::st_global_v4(orow + c + 8, o[4], o[5], o[6], o[7]);
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&o_free[t]);  // O_t may be overwritten by the next item's first PV
        }
    }
    __syncthreads();
    if (warp == 9) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace

// Tensor-core path for head_dim 128 (prefill_attention.cu dispatches here);
// rows = total rows of qkv (the TMA map bounds).
bool prefill_attention_tc(const f16* qkv, long long rows, f16* out, const int* cu, int n_req, int max_len, int H,
                          int hd, float scale, cudaStream_t st) {
    static const int enabled = [] {
        const char* e = std::getenv("HC_PREFILL_TC");  // 0 mma.sync, 1 one tile per CTA, 2 tile pairs
        return e ? std::atoi(e) : 2;
    }();
    if (!enabled || rows <= 0 || (hd != 128 && (hd != 64 || enabled == 1))) return false;
    static std::atomic<uint64_t> configured1{0}, configured2{0};
    max_dynamic_smem_once(prefill_tc_kernel, Smem::bytes, configured1);
    static std::atomic<uint64_t> configured3{0};
    static std::atomic<uint64_t> configured4{0}, configured5{0};
    max_dynamic_smem_once(prefill_tc2_kernel<128>, Smem2<128>::bytes, configured2);
    max_dynamic_smem_once(prefill_tc2_kernel<64>, Smem2<64>::bytes, configured3);
    max_dynamic_smem_once(prefill_tc2_kernel<128, true>, Smem2<128>::bytes, configured4);
    max_dynamic_smem_once(prefill_tc2_kernel<64, true>, Smem2<64>::bytes, configured5);
    const long long d3 = 3LL * H * hd;
    const CUtensorMap tm = make_map(qkv, rows, d3, d3, kT);
    static const uint32_t lbo = [] {
        const char* e = std::getenv("HC_PREFILL_TC_LBO");
        return e ? static_cast<uint32_t>(std::atoi(e)) : static_cast<uint32_t>(kBox);
    }();
    static const uint32_t sbo = [] {
        const char* e = std::getenv("HC_PREFILL_TC_SBO");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 1024u;
    }();
    const int n_qt = (max_len + kT - 1) / kT;
    if (enabled == 1) {  // one query tile per CTA (single softmax group)
        prefill_tc_kernel<<<dim3(n_qt, H, n_req), kThreads, Smem::bytes, st>>>(tm, out, cu, H, scale, lbo, sbo);
    } else {  // pairs of query tiles, two softmax groups (default)
        static const int sms = [] {
            int dev = 0, n = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
            return n;
        }();
        const int n_pairs = (n_qt + 1) / 2;
        const long long items = static_cast<long long>(n_pairs) * H * n_req;
        const int grid = static_cast<int>(std::min<long long>(items, sms));
        // P kept in TMEM (TS-form P.V MMA): 1.4-2.2 % faster at head_dim 128 (P = 1024 / 2048),
        // 6 % slower at 64 (its hi/lo split doubles the tcgen05.st traffic) — so 128 only by default
        static const int p_tmem = [] {
            const char* e = std::getenv("HC_PREFILL_PTMEM");  // 0: never, 1: head_dim 128 (default), 2: both
            return e ? std::atoi(e) : 1;
        }();
        if (hd == 128 && p_tmem >= 1)
            prefill_tc2_kernel<128, true><<<grid, kThreads2, Smem2<128>::bytes, st>>>(tm, out, cu, n_req, n_pairs, H,
                                                                                       scale, lbo, sbo);
        else if (hd == 128)
            prefill_tc2_kernel<128><<<grid, kThreads2, Smem2<128>::bytes, st>>>(tm, out, cu, n_req, n_pairs, H, scale,
                                                                                 lbo, sbo);
        else if (p_tmem >= 2)
            prefill_tc2_kernel<64, true><<<grid, kThreads2, Smem2<64>::bytes, st>>>(tm, out, cu, n_req, n_pairs, H,
                                                                                     scale, lbo, sbo);
        else
            prefill_tc2_kernel<64><<<grid, kThreads2, Smem2<64>::bytes, st>>>(tm, out, cu, n_req, n_pairs, H, scale,
                                                                               lbo, sbo);
    }
    return true;
}

}  // namespace hc
