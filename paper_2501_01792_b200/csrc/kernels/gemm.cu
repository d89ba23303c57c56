// Host launcher for the tcgen05 GEMM (gemm.cuh): tensor-map encoding,
// tile-shape heuristic and template dispatch.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm.cuh"
#include "kernels.hpp"
#include "launch.hpp"
#include "tma.hpp"

namespace hc {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

// 2-D f16 tensor [rows x cols] with row stride ld (elements); box = box_rows x 64.
CUtensorMap make_map(const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(gemm::BK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) +
                                 "): rows=" + std::to_string(rows) + " cols=" + std::to_string(cols) +
                                 " ld=" + std::to_string(ld));
    return m;
}

namespace {

template <int BN, int EPI, int HD = 0, int SEG = 0>
void launch(const GemmCall& c, const gemm::Params& p, cudaStream_t st) {
    using Cf = gemm::Cfg<BN>;
    auto kern = gemm::gemm_tn_kernel<BN, EPI, HD, SEG>;
    static std::atomic<uint64_t> attr_set{0};  // per instantiation, per device
    max_dynamic_smem_once(kern, Cf::kSmemBytes, attr_set);
    const CUtensorMap ta = make_map(c.A, c.a_rows, c.K, c.lda, gemm::BM);
    const CUtensorMap tb = make_map(c.B, c.N, c.K, c.ldb, EPI == gemm::kAttnPart ? 128 : BN);
    const int tiles = p.num_m_tiles * p.num_n_tiles * p.splits;
    int grid = tiles < num_sms() ? tiles : num_sms();
    if (c.max_ctas > 0 && grid > c.max_ctas) grid = c.max_ctas;
    kern<<<grid, gemm::kThreads, Cf::kSmemBytes, st>>>(ta, tb, p);
}

template <int EPI, int HD = 0, int SEG = 0>
void launch_pair(const GemmCall& c, const gemm::Params& p, cudaStream_t st) {
    using Cf = gemm::Cfg2;
    auto kern = gemm::gemm2_tn_kernel<EPI, HD, SEG>;
    static std::atomic<uint64_t> attr_set{0};
    max_dynamic_smem_once(kern, Cf::kSmemBytes, attr_set);
    const CUtensorMap ta = make_map(c.A, c.a_rows, c.K, c.lda, gemm::BM);
    const CUtensorMap tb = make_map(c.B, c.N, c.K, c.ldb, Cf::BN / 2);
    const int tiles = ((p.num_m_tiles + 1) / 2) * p.num_n_tiles;
    const int pairs = std::min(tiles, num_sms() / 2);
    kern<<<2 * pairs, gemm::kThreads, Cf::kSmemBytes, st>>>(ta, tb, p);
}

template <int BN>
void dispatch_epi(const GemmCall& c, const gemm::Params& p, cudaStream_t st) {
    switch (c.epi) {
        case gemm::kStore: return launch<BN, gemm::kStore>(c, p, st);
        case gemm::kRelu: return launch<BN, gemm::kRelu>(c, p, st);
        case gemm::kKvPaged: return launch<BN, gemm::kKvPaged>(c, p, st);
        case gemm::kF32: return launch<BN, gemm::kF32>(c, p, st);
        case gemm::kSplitF32: return launch<BN, gemm::kSplitF32>(c, p, st);
    }
    throw std::invalid_argument("gemm: unknown epilogue");
}

// recompute fused with decode attention: template on (head_dim, segment rows)
template <bool kPair, int HD>
void dispatch_attn_seg(const GemmCall& c, const gemm::Params& p, cudaStream_t st) {
    const int seg = c.tpb < 32 ? c.tpb : 32;
#define HC_SEG(S_)                                                           \
    if (seg == S_) {                                                         \
        if constexpr (kPair)                                                 \
            launch_pair<gemm::kAttnPart, HD, S_>(c, p, st);                  \
        else                                                                 \
            launch<256, gemm::kAttnPart, HD, S_>(c, p, st);                  \
        return;                                                              \
    }
    HC_SEG(4)
    HC_SEG(8)
    HC_SEG(16)
    HC_SEG(32)
#undef HC_SEG
    throw std::invalid_argument("gemm: kAttnPart needs tokens_per_block 4..64");
}

template <bool kPair>
void dispatch_attn(const GemmCall& c, const gemm::Params& p, cudaStream_t st) {
    if (c.hd == 128) return dispatch_attn_seg<kPair, 128>(c, p, st);
    if (c.hd == 64) return dispatch_attn_seg<kPair, 64>(c, p, st);
    throw std::invalid_argument("gemm: kAttnPart needs head_dim 64 or 128");
}

int pick_bn(int num_m_tiles, int N) {
    if (num_m_tiles >= 8) return 256;
    // weight-streaming regime: minimise the per-CTA (A + B) tile bytes
    const int sms = num_sms();
    int best = 256;
    long best_cost = -1;
    for (int bn : {256, 128, 64, 32}) {
        const long tiles = static_cast<long>(num_m_tiles) * ((N + bn - 1) / bn);
        const long per_cta = (tiles + sms - 1) / sms;
        const long cost = per_cta * (gemm::BM + bn);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = bn;
        }
    }
    return best;
}

// split-K planner for the weight-streaming regime (M <= 2 tiles): choose
// (BN, splits) so every SM streams weights; per-CTA cost ~ units/SM x
// (A + B tile bytes of one split) + the fp32 partial round trip.
void pick_split(int num_m_tiles, int M, int N, int K, size_t ws_floats, int& bn_out, int& splits_out) {
    const int sms = num_sms();
    const int num_kb = (K + gemm::BK - 1) / gemm::BK;
    double best = -1;
    bn_out = pick_bn(num_m_tiles, N);
    splits_out = 1;
    for (int bn : {256, 128, 64}) {
        for (int s = 1; s <= 16; ++s) {
            const int kps = (num_kb + s - 1) / s;
            if (s > 1 && kps < 4) break;
            if (s > 1 && static_cast<size_t>(s) * M * N > ws_floats) break;
            const long units = static_cast<long>(num_m_tiles) * ((N + bn - 1) / bn) * s;
            const long per_cta = (units + sms - 1) / sms;
            double cost = static_cast<double>(per_cta) * (gemm::BM + bn) * kps * gemm::BK * 2.0;
            // fp32 partial write + reduce read per SM, plus ~5 us of extra launch
            if (s > 1) cost += 2.0 * s * M * N * 4.0 / sms + 2.2e5;
            if (best < 0 || cost < best) {
                best = cost;
                bn_out = bn;
                splits_out = s;
            }
        }
    }
}

}  // namespace

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

namespace {
bool validate(const GemmCall& c) {  // false: an empty problem
    if (c.M <= 0 || c.N <= 0 || c.K <= 0) return false;
    if (c.N % 16 != 0) throw std::invalid_argument("gemm: N must be a multiple of 16");
    if ((c.lda * 2) % 16 || (c.ldb * 2) % 16 || (c.K * 2) % 16)
        throw std::invalid_argument("gemm: row strides must be 16-byte multiples");
    if (reinterpret_cast<uintptr_t>(c.A) % 16 || reinterpret_cast<uintptr_t>(c.B) % 16)
        throw std::invalid_argument("gemm: operands must be 16-byte aligned");
    return true;
}
}  // namespace

void run_gemm(const GemmCall& c, cudaStream_t st) {
    if (!validate(c)) return;
    if (run_wstream(c, st)) return;  // decode-batch GEMMs: swap-AB stream-K weight streaming (wstream.cuh)
    run_gemm_tiled(c, st);
}

void run_gemm_tiled(const GemmCall& c, cudaStream_t st) {
    if (!validate(c)) return;
    gemm::Params p{};
    p.M = c.M;
    p.N = c.N;
    p.K = c.K;
    p.m_tile_rows = c.m_tile_rows;
    p.num_m_tiles = c.m_tile_rows ? c.num_m_tiles : (c.M + gemm::BM - 1) / gemm::BM;
    if (p.num_m_tiles <= 0) return;
    p.out = c.out;
    p.ldc = c.ldc;
    p.tpb = c.tpb;
    p.d = c.d;
    p.hd = c.hd;
    p.blk_off = c.blk_off;
    if ((c.bias || c.res) && (c.epi == gemm::kF32 || c.epi == gemm::kSplitF32))
        throw std::invalid_argument("gemm: bias / residual apply to f16 epilogues only");
    if ((c.bias && reinterpret_cast<uintptr_t>(c.bias) % 16) ||
        (c.res && (reinterpret_cast<uintptr_t>(c.res) % 16 || (c.ldr * 2) % 16)))
        throw std::invalid_argument("gemm: bias / residual must be 16-byte aligned");
    p.bias = c.bias;
    p.res = c.res;
    p.ldr = c.ldr;
    if (c.epi == gemm::kAttnPart) {
        if (c.d % 128 || c.N != 2 * c.d || !c.blk_info || !c.q || !c.part || c.res || !c.m_tile_rows ||
            c.tpb <= 0 || gemm::BM % c.tpb || (c.ldq * 2) % 16 || reinterpret_cast<uintptr_t>(c.q) % 16)
            throw std::invalid_argument("gemm: kAttnPart needs d % 128 == 0, N = 2d, tile rows, blk_info, q, part");
        p.v_row = c.d;
        p.blk_info = c.blk_info;
        p.q = c.q;
        p.ldq = c.ldq;
        p.qscale = c.qscale;
        p.heads = c.d / c.hd;
        p.part = c.part;
    }
    p.group_m = c.group_m > 0 ? c.group_m : (c.K <= 4096 ? 32 : 16);
    if (const char* g = std::getenv("HC_GEMM_GROUP_M")) p.group_m = std::max(1, std::atoi(g));  // tuning knob
    static const int group_n_env = [] {
        const char* g = std::getenv("HC_GEMM_GROUP_N");  // tuning knob: weight-stationary raster
        return g ? std::atoi(g) : 0;
    }();
    p.group_n = group_n_env;
    static const int l2_env = [] {
        const char* e = std::getenv("HC_GEMM_L2HINT");  // tuning knob: gemm::kL2* bits
        return e ? std::atoi(e) : -1;
    }();
    // by shape: the recompute GEMM keeps its A group in L2 and streams its K|V
    // out (scripts/gemm_sustained.py: +8 % sustained for the pair kernel)
    p.l2_hint = c.l2_hint >= 0 ? c.l2_hint
                : c.epi == gemm::kKvPaged ? (gemm::kL2KeepA | gemm::kL2StreamC)
                : c.epi == gemm::kAttnPart ? gemm::kL2KeepA : 0;
    if (l2_env >= 0) p.l2_hint = l2_env;
    p.splits = 1;
    p.kb_per_split = (c.K + gemm::BK - 1) / gemm::BK;
    GemmCall cc = c;
    if (cc.a_rows <= 0) cc.a_rows = c.M;
    int bn = c.bn ? c.bn : pick_bn(p.num_m_tiles, c.N);
    const bool can_split = c.ws && c.ws_floats && !c.m_tile_rows && p.num_m_tiles <= 2 &&
                           (c.epi == gemm::kStore || c.epi == gemm::kRelu || c.epi == gemm::kF32) && c.ldc == c.N &&
                           (!c.bn || c.splits);
    if (can_split) {
        int s = 1;
        if (c.splits)
            s = c.splits;
        else
            pick_split(p.num_m_tiles, c.M, c.N, c.K, c.ws_floats, bn, s);
        if (static_cast<size_t>(s) * c.M * c.N > c.ws_floats) s = 1;
        if (const char* e = std::getenv("HC_GEMM_SPLITS")) s = std::max(1, std::atoi(e));  // tuning knob
        if (s > 1) {
            const int num_kb = (c.K + gemm::BK - 1) / gemm::BK;
            p.kb_per_split = (num_kb + s - 1) / s;
            p.splits = (num_kb + p.kb_per_split - 1) / p.kb_per_split;
            p.out = c.ws;
            p.ldc = c.N;
            p.bias = nullptr;  // applied once, by the reduce
            p.res = nullptr;
            cc.epi = gemm::kSplitF32;
        }
    }
    // large M: CTA-pair (cta_group::2) 256x256 tiles
    static const bool pair_ok = [] {
        const char* e = std::getenv("HC_GEMM_PAIR");
        return !(e && e[0] == '0');
    }();
    // Sustained under the 1 kW cap (scripts/gemm_sustained.py, 3 s back to back,
    // profiles/r02_gemm_sustained.txt): at K = 4096 the pair kernel runs 1.75
    // PFLOP/s against the 1-SM kernel's 1.61 (the 256 x 256 tile halves the
    // smem / L2 feed per MAC); at K = 7168 [Wk|Wv] (205 MB) outgrows L2, the
    // pair kernel's rasters re-read it to 26-40 GB of DRAM per 122880-row launch
    // (1-SM: 14 GB, profiles/r02_recompute_dram_sweep.txt), and the extra HBM
    // power costs it the clock: 1.58 vs 1.62 PFLOP/s (1432 vs 1560 MHz)
    static const int pair_max_k = [] {
        const char* e = std::getenv("HC_GEMM_PAIR_MAX_K");  // tuning knob
        return e ? std::atoi(e) : 4096;
    }();
    if (pair_ok && p.splits == 1 && !c.bn && p.num_m_tiles >= 8 && c.K <= pair_max_k && cc.epi != gemm::kSplitF32) {
        p.num_n_tiles = (c.N + gemm::Cfg2::BN - 1) / gemm::Cfg2::BN;
        p.group_m = c.group_m > 0 ? std::max(1, c.group_m / 2) : 16;
        // weight-stationary by default: 16 N tiles (16 x 256 rows of B, 33.5 MB at
        // K = 4096) stay in L2 while M is swept — 0.70 GB of DRAM per 33792-row
        // recompute vs 1.06 GB for the M-grouped raster (r02_recompute_dram_sweep.txt)
        if (!group_n_env && c.group_m <= 0) p.group_n = 16;
        if (const char* g = std::getenv("HC_GEMM_GROUP_M")) p.group_m = std::max(1, std::atoi(g) / 2);
        switch (cc.epi) {
            case gemm::kAttnPart: dispatch_attn<true>(cc, p, st); return;
            case gemm::kStore: launch_pair<gemm::kStore>(cc, p, st); return;
            case gemm::kRelu: launch_pair<gemm::kRelu>(cc, p, st); return;
            case gemm::kKvPaged: launch_pair<gemm::kKvPaged>(cc, p, st); return;
            case gemm::kF32: launch_pair<gemm::kF32>(cc, p, st); return;
        }
    }
    if (cc.epi == gemm::kAttnPart) {
        p.num_n_tiles = c.N / 256;
        dispatch_attn<false>(cc, p, st);
        return;
    }
    p.num_n_tiles = (c.N + bn - 1) / bn;
    switch (bn) {
        case 32: dispatch_epi<32>(cc, p, st); break;
        case 64: dispatch_epi<64>(cc, p, st); break;
        case 128: dispatch_epi<128>(cc, p, st); break;
        case 256: dispatch_epi<256>(cc, p, st); break;
        default: throw std::invalid_argument("gemm: bn must be 32/64/128/256");
    }
    if (p.splits > 1 && c.epi == gemm::kF32)
        splitk_reduce_f32(c.ws, p.splits, c.M, c.N, static_cast<float*>(c.out), st);
    else if (p.splits > 1)
        splitk_reduce(c.ws, p.splits, c.M, c.N, static_cast<f16*>(c.out), c.epi == gemm::kRelu, st, c.bias, c.res,
                      c.ldr);
}

}  // namespace hc
