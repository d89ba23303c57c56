// Host launcher for the weight-streaming decode GEMM (wstream.cuh).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"
#include "launch.hpp"
#include "tma.hpp"
#include "wstream.cuh"

namespace hc {

namespace {

int batch_cols(int M) {
    for (int mp : {16, 32, 64, 128, 256})
        if (M <= mp) return mp;
    return 0;
}

template <int MP, int EPI>
void launch_ws(const GemmCall& c, wstream::Params p, cudaStream_t st) {
    using Cf = wstream::Cfg<MP>;
    auto kern = wstream::wstream_kernel<MP, EPI>;
    static std::atomic<uint64_t> attr_set{0};
    max_dynamic_smem_once(kern, Cf::kSmemBytes, attr_set);
    const CUtensorMap tw = make_map(c.B, c.N, c.K, c.ldb, 128);
    const CUtensorMap tx = make_map(c.A, c.a_rows, c.K, c.lda, MP);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    {
        // c.pdl: the previous operation on `st` is a kernel, so this launch may
        // overlap its tail (the weight prefetch runs before griddepcontrol.wait)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.G);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = Cf::kSmemBytes;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = c.pdl ? 1 : 0;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tw, tx, p);
        if (e != cudaSuccess) throw std::runtime_error(std::string("wstream launch: ") + cudaGetErrorString(e));
    }
    // any CTA boundary inside a unit leaves partials to reduce
    bool cut = false;
    for (int c = 1; c < p.G && !cut; ++c) cut = (static_cast<long long>(c) * p.T / p.G) % p.NK != 0;
    if (!cut) return;
    cudaLaunchConfig_t cfg = {};
    const long long items = static_cast<long long>(p.units) * ((p.M + 1024 / Cf::WT - 1) / (1024 / Cf::WT));
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<long long>(items, 4LL * num_sms())));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, wstream::wstream_reduce_kernel<MP, EPI>, p);
    if (e != cudaSuccess) throw std::runtime_error(std::string("wstream reduce launch: ") + cudaGetErrorString(e));
}

template <int MP>
bool dispatch_ws(const GemmCall& c, cudaStream_t st) {
    using Cf = wstream::Cfg<MP>;
    wstream::Params p{};
    p.M = c.M;
    p.N = c.N;
    p.K = c.K;
    p.NK = (c.K + gemm::BK - 1) / gemm::BK;
    p.units = (c.N + Cf::WT - 1) / Cf::WT;
    p.T = static_cast<long long>(p.units) * p.NK;
    // every SM streams an equal share of W; at least 4 k-blocks per CTA so a
    // tiny GEMM is not cut into slivers. When the units alone nearly fill the
    // SMs (>= 3/4), one whole unit per CTA beats cutting: no partials, no reduce
    long long g = std::min<long long>(num_sms(), std::max<long long>(1, p.T / 4));
    if (p.units <= num_sms() && 4 * p.units >= 3 * num_sms()) g = p.units;
    const long long slot_floats = static_cast<long long>(MP) * Cf::WT;
    g = std::min<long long>(g, static_cast<long long>(c.ws_floats / (2 * slot_floats)));
    if (c.max_ctas > 0) g = std::min<long long>(g, c.max_ctas);
    // the reduce kernel resolves at most kMaxCut segments per unit
    while (g > 1 && (p.NK + p.T / g - 1) / (p.T / g) + 1 > wstream::kMaxCut) --g;
    if (g < 1) return false;
    p.G = static_cast<int>(g);
    p.out = c.out;
    p.ldc = c.ldc;
    p.bias = c.bias;
    p.res = c.res;
    p.ldr = c.ldr;
    p.part = c.ws;
    switch (c.epi) {
        case gemm::kStore: launch_ws<MP, gemm::kStore>(c, p, st); return true;
        case gemm::kRelu: launch_ws<MP, gemm::kRelu>(c, p, st); return true;
        case gemm::kF32: launch_ws<MP, gemm::kF32>(c, p, st); return true;
    }
    return false;
}

}  // namespace

size_t wstream_ws_floats(int M) {
    const int mp = batch_cols(M);
    if (!mp) return 0;
    const int wt = mp == 256 ? 128 : 256;
    return static_cast<size_t>(2) * num_sms() * mp * wt;
}

bool run_wstream(const GemmCall& c, cudaStream_t st) {
    static const bool enabled = [] {
        const char* e = std::getenv("HC_WSTREAM");  // 0: the tile kernel + split-K for decode GEMMs (A/B knob)
        return !(e && e[0] == '0');
    }();
    if (!enabled || !c.ws || c.m_tile_rows || c.splits || c.bn) return false;
    if (c.epi != gemm::kStore && c.epi != gemm::kRelu && c.epi != gemm::kF32) return false;
    if (c.M < 1 || c.a_rows < c.M || c.N % 16 || c.ldc % 4 || (c.res && c.ldr % 4) || (c.epi == gemm::kF32 && (c.bias || c.res))) return false;
    if (reinterpret_cast<uintptr_t>(c.out) % 16) return false;
    switch (batch_cols(c.M)) {
        case 16: return dispatch_ws<16>(c, st);
        case 32: return dispatch_ws<32>(c, st);
        case 64: return dispatch_ws<64>(c, st);
        case 128: return dispatch_ws<128>(c, st);
        case 256: return dispatch_ws<256>(c, st);
    }
    return false;
}

}  // namespace hc
