// Causal prefill attention (attention_causal, decoder.cpp:55-63: row t of
// request r attends to keys [0, t] of the same request; softmax(q.K^T*s).V,
// s = 1/sqrt(hd), max-subtracted) over ragged requests packed end to end.
//
// prefill_attention() dispatches to the tcgen05 kernels (prefill_attention_tc.cu,
// head_dim 64 and 128); the mma.sync kernel below is the comparison path kept
// behind HC_PREFILL_TC=0 (and the fallback for other head dims):
//
// Tensor-core flash attention: one CTA (4 warps) per (64-query tile, head,
// request); each warp owns 16 query rows. S = Q.K^T and O += P.V run on
// mma.sync m16n8k16 f16 (fp32 accumulate; P.V as hi+lo f16 halves of P);
// the online softmax lives in the
// accumulator registers (a thread owns 2 rows, quad shuffles reduce them) and
// P is re-packed register-to-register as the A operand of P.V. K and V tiles
// of 64 keys are double-buffered in XOR-swizzled shared memory with cp.async
// (16-byte chunks, conflict-free ldmatrix), so tile j+1 streams in while
// tile j is multiplied. Causality skips every key tile right of the
// diagonal; heavier (later) query tiles launch first.
//
// Q shares buffer 1's K slot (64 KB of smem per CTA at HD 128) and registers
// are capped for 3 resident CTAs per SM.
// Prefill is <2% of an offloaded decode run, so this kernel
// uses the warp-level MMA path rather than a TMEM-resident tcgen05 pipeline.
#include <cfloat>
#include <stdexcept>

#include "kernels.hpp"
#include "launch.hpp"
#include "ptx.cuh"

namespace hc {

namespace {

constexpr int kQT = 64;   // query rows per CTA
constexpr int kKT = 64;   // keys per tile
static_assert(kQT == kKT, "Q is staged in a K tile slot");
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    const int n = pred ? 16 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (a, b) -> f16x2 hi = rn(a, b) and lo = rn((a, b) - hi)
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// byte offset of 16-B chunk `ch` of row `row` in a [rows][HD] f16 tile
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int ch) {
    constexpr int CH = HD / 8;  // chunks per row (16 or 8)
    return static_cast<uint32_t>((row * CH + (ch ^ (row & 7))) * 16);
}

// rows [0, min(n, 64)) of a 64 x HD tile at g (row stride ld elements) into
// swizzled smem; rows >= n are zero-filled
template <int HD>
__device__ __forceinline__ void load_tile(uint32_t sbase, const f16* g, long long ld, int n) {
    constexpr int CH = HD / 8;
    for (int i = threadIdx.x; i < kKT * CH; i += blockDim.x) {
        const int r = i / CH, ch = i % CH;
        const bool ok = r < n;
        cp_async16(sbase + swz<HD>(r, ch), g + (ok ? static_cast<long long>(r) * ld + ch * 8 : 0), ok);
    }
}

template <int HD>
__global__ void __launch_bounds__(128, 3)
    prefill_flash_kernel(const f16* __restrict__ qkv, f16* __restrict__ out, const int* __restrict__ cu, int H,
                         float scale) {
    constexpr int NK = HD / 16;  // k16 steps over the head dim
    constexpr int NO = HD / 8;   // n8 tiles of O
    const int req = blockIdx.z, h = blockIdx.y;
    const int row0 = cu[req];
    const int P = cu[req + 1] - row0;
    const int n_qt = (P + kQT - 1) / kQT;
    const int qt = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);  // heavy tiles first
    if (qt >= n_qt) return;
    const int q0 = qt * kQT;
    const int d = H * HD;
    const long long ld = 3LL * d;
    const f16* base = qkv + static_cast<long long>(row0) * ld + h * HD;

    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t s0 = smem_u32(smem);
    // buffer c: K at s0 + 2 kKT HD 2 c bytes, V right after it. Q is staged in
    // buffer 1's K slot: it moves to registers before tile 1 is prefetched, so
    // the CTA needs 4 tiles of smem (64 KB at HD 128) and 3 CTAs fit an SM
    auto sK = [&](int c) { return s0 + static_cast<uint32_t>(2 * kKT * c * HD * 2); };
    auto sV = [&](int c) { return sK(c) + static_cast<uint32_t>(kKT * HD * 2); };
    const uint32_t sQ = sK(1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int kend = min(P, q0 + kQT);           // keys this tile needs (causal)
    const int n_kt = (kend + kKT - 1) / kKT;

    load_tile<HD>(sQ, base + static_cast<long long>(q0) * ld, ld, P - q0);
    load_tile<HD>(sK(0), base + d, ld, kend);
    load_tile<HD>(sV(0), base + 2 * d, ld, kend);
    cp_async_commit();

    float o[NO][4];
#pragma unroll
    for (int j = 0; j < NO; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
    uint32_t qa[NK][4];
    const float sl = scale * kLog2e;
    const int qrow = q0 + warp * 16 + lane / 4;  // rows qrow and qrow + 8
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
        const int r = warp * 16 + (lane % 16), ch = kk * 2 + lane / 16;
        ldsm_x4(sQ + swz<HD>(r, ch), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
    }
    __syncthreads();  // the Q slot is buffer 1's K: free it before the first prefetch

    for (int kt = 0; kt < n_kt; ++kt) {
        const int cur = kt & 1;
        if (kt + 1 < n_kt) {
            const int k1 = (kt + 1) * kKT;
            load_tile<HD>(sK(cur ^ 1), base + static_cast<long long>(k1) * ld + d, ld, kend - k1);
            load_tile<HD>(sV(cur ^ 1), base + static_cast<long long>(k1) * ld + 2 * d, ld, kend - k1);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        // S = Q.K^T : 16 x 64 per warp
        float s[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {  // key n-tiles 2jp, 2jp+1
                const int key = jp * 16 + (lane / 16) * 8 + (lane % 8);
                const int ch = kk * 2 + ((lane / 8) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sK(cur) + swz<HD>(key, ch), b0, b1, b2, b3);
                mma16816(s[2 * jp], qa[kk], b0, b1);
                mma16816(s[2 * jp + 1], qa[kk], b2, b3);
            }
        }
        // mask (causal + request end), online softmax in the exp2 domain
        const int k0 = kt * kKT;
        const bool need_mask = k0 + kKT > q0 || k0 + kKT > P;
        float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = s[j][e] * sl;
                if (need_mask) {
                    const int key = k0 + j * 8 + (lane % 4) * 2 + (e & 1);
                    const int row = qrow + (e >> 1) * 8;
                    if (key > row || key >= P) v = -FLT_MAX;
                }
                s[j][e] = v;
                mx[e >> 1] = fmaxf(mx[e >> 1], v);
            }
        }
        float alpha[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
            alpha[i] = exp2f(m_r[i] - mx[i]);
            m_r[i] = mx[i];
            l_r[i] *= alpha[i];
        }
#pragma unroll
        for (int j = 0; j < NO; ++j) {
            o[j][0] *= alpha[0];
            o[j][1] *= alpha[0];
            o[j][2] *= alpha[1];
            o[j][3] *= alpha[1];
        }
        // P as the A operand (k16 chunk = keys 16kk..16kk+15), split into
        // f16 hi + lo parts: P.V = P_hi.V + P_lo.V keeps P to ~16 bits, so
        // the prefill matches fp32 softmax weights (a single f16 P costs ~2^-9
        // relative per weight, visible after a dozen layers)
        uint32_t pa[4][4], pl[4][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float p0 = exp2f(s[j][0] - m_r[0]), p1 = exp2f(s[j][1] - m_r[0]);
            const float p2 = exp2f(s[j][2] - m_r[1]), p3 = exp2f(s[j][3] - m_r[1]);
            l_r[0] += p0 + p1;
            l_r[1] += p2 + p3;
            split_f16x2(p0, p1, pa[j / 2][(j & 1) * 2 + 0], pl[j / 2][(j & 1) * 2 + 0]);
            split_f16x2(p2, p3, pa[j / 2][(j & 1) * 2 + 1], pl[j / 2][(j & 1) * 2 + 1]);
        }
        // O += P.V : V tile [key][hd] read transposed as the col-major B operand
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int jp = 0; jp < NO / 2; ++jp) {  // hd n-tiles 2jp, 2jp+1
                const int key = kk * 16 + ((lane / 8) & 1) * 8 + (lane % 8);
                const int ch = jp * 2 + lane / 16;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sV(cur) + swz<HD>(key, ch), b0, b1, b2, b3);
                mma16816(o[2 * jp], pa[kk], b0, b1);
                mma16816(o[2 * jp + 1], pa[kk], b2, b3);
                mma16816(o[2 * jp], pl[kk], b0, b1);
                mma16816(o[2 * jp + 1], pl[kk], b2, b3);
            }
        }
        __syncthreads();  // tile `cur` is overwritten by the load issued next iteration
    }
    // finish: full row sums across the quad, normalise, store f16
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        l_r[i] += __shfl_xor_sync(0xffffffffu, l_r[i], 1);
        l_r[i] += __shfl_xor_sync(0xffffffffu, l_r[i], 2);
        l_r[i] = l_r[i] > 0.f ? 1.f / l_r[i] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = qrow + i * 8;
        if (row >= P) continue;
        f16* op = out + static_cast<long long>(row0 + row) * d + h * HD + (lane % 4) * 2;
#pragma unroll
        for (int j = 0; j < NO; ++j)
            *reinterpret_cast<uint32_t*>(op + j * 8) = ptx::pack_f16x2(o[j][2 * i] * l_r[i], o[j][2 * i + 1] * l_r[i]);
    }
}

template <int HD>
void launch_prefill(const f16* qkv, f16* out, const int* cu, int n_req, int max_len, int H, float scale,
                    cudaStream_t st) {
    constexpr size_t smem = static_cast<size_t>(4 * kKT) * HD * 2;
    static std::atomic<uint64_t> configured{0};
    max_dynamic_smem_once(prefill_flash_kernel<HD>, static_cast<int>(smem), configured);
    const dim3 grid((max_len + kQT - 1) / kQT, H, n_req);
    prefill_flash_kernel<HD><<<grid, 128, smem, st>>>(qkv, out, cu, H, scale);
}

}  // namespace

bool prefill_attention_tc(const f16* qkv, long long rows, f16* out, const int* cu, int n_req, int max_len, int H,
                          int hd, float scale, cudaStream_t st);

void prefill_attention(const f16* qkv, f16* out, const int* cu, int n_req, int max_len, int H, int hd,
                       float scale, cudaStream_t st, long long rows) {
    if (n_req <= 0 || max_len <= 0) return;
    if (prefill_attention_tc(qkv, rows, out, cu, n_req, max_len, H, hd, scale, st)) return;
    if (hd == 128)
        launch_prefill<128>(qkv, out, cu, n_req, max_len, H, scale, st);
    else if (hd == 64)
        launch_prefill<64>(qkv, out, cu, n_req, max_len, H, scale, st);
    else
        throw std::invalid_argument("prefill_attention: head_dim must be 64 or 128");
}

}  // namespace hc
