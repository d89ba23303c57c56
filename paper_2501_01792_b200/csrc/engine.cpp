#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_set>

#include "capi_util.hpp"
#include "kernels/gemm_types.hpp"

namespace hc {

namespace {

// region ids of packed block refs (kernels.hpp: ref = region << 28 | index)
enum Region : int {
    R_KV_STAGE = 0,   // streamed KV/host blocks of the current layer (slot l%2)
    R_KV_GPU = 1,     // resident KV/gpu pool, layer l
    R_KVR = 2,        // K|V recomputed from ACT blocks this layer
    R_ACT_STAGE = 3,  // streamed ACT/host blocks (slot l%2)
    R_ACT_GPU = 4,    // resident ACT/gpu pool, layer l
    R_KV_HOST = 5,    // pinned KV/host pool, physical layer l%Lp (mapped)
    R_ACT_HOST = 6,   // pinned ACT/host pool (mapped)
    R_TOKREC = 7,     // K|V of token-recompute prefixes, rebuilt every layer of every step
};

struct Run {
    int start, count;
    int dst = 0;  // staging position of `start` (decode steps)
};

std::vector<Run> runs_of(std::vector<int> pbns) {
    std::sort(pbns.begin(), pbns.end());
    pbns.erase(std::unique(pbns.begin(), pbns.end()), pbns.end());
    std::vector<Run> r;
    for (int p : pbns) {
        if (!r.empty() && r.back().start + r.back().count == p)
            ++r.back().count;
        else
            r.push_back({p, 1, 0});
    }
    return r;
}

// first pool rows of the 128-row GEMM tiles touching the listed blocks
std::vector<int> tiles_of(const std::vector<int>& pbns, int tpb) {
    std::vector<int> t;
    for (int p : pbns) {
        const long r0 = static_cast<long>(p) * tpb, r1 = r0 + tpb - 1;
        for (long r = r0 / gemm::BM; r <= r1 / gemm::BM; ++r) t.push_back(static_cast<int>(r * gemm::BM));
    }
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    return t;
}

template <class T>
T* dalloc(size_t n) {
    if (!n) return nullptr;
    void* p = nullptr;
    HC_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

template <class T>
T* halloc(size_t n, bool mapped) {
    if (!n) return nullptr;
    void* p = nullptr;
    HC_CUDA(cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable | (mapped ? cudaHostAllocMapped : 0)));
    return static_cast<T*>(p);
}

}  // namespace

void gemm_rows(int epi, const f16* A, int M, int K, const f16* W, int N, void* out, long long ldc, cudaStream_t st,
               long long lda = 0, const GemmScratch& sc = GemmScratch{}, const f16* bias = nullptr,
               const f16* res = nullptr, long long ldr = 0);

struct Engine::Impl {
    int L = 0, d = 0, H = 0, hd = 0, f = 0, V = 0, tpb = 0, B = 0, max_seq = 0, max_blocks = 0, Lp = 0, Lw = 0;
    int arch = kArchReference;
    // head-sharded tensor parallelism (tp.hpp): this rank's heads / hidden
    // columns / FFN slice; ACT/host blocks are owned round-robin by pbn and
    // staged at act_pos(pbn) so one all-gather of the per-rank chunks fills
    // every rank's staging
    TpGroup* tp = nullptr;
    int tpr = 0, tpn = 1, Hg = 0, dg = 0, fg = 0;
    long act_cap_n = 0;  // ACT/host blocks per rank = ceil(act_host_cap / tpn)
    f16* wfull = nullptr;  // init only: one unsharded layer when tpn > 1
    bool owns(int pbn) const { return pbn % tpn == tpr; }
    int act_pos(int pbn) const { return static_cast<int>((pbn % tpn) * act_cap_n + pbn / tpn); }
    f16* lnf = nullptr;  // kArchOpt final LayerNorm gamma | beta [2d]
    f16* xn = nullptr;   // kArchOpt decode LN output [B x d]
    f16* pxn = nullptr;  // kArchOpt prefill LN1 output [prefill_rows x d]
    size_t LE = 0, kvb = 0, actb = 0;
    LayerOffsets off{};        // this rank's packed layer (== offF when tpn == 1)
    LayerOffsets offF{};       // the unsharded packed layer
    size_t LEF = 0;
    f16 *emb = nullptr, *pos = nullptr;
    f16* w_all = nullptr;
    f16* wbuf[2] = {nullptr, nullptr};
    uint16_t* h_w = nullptr;
    f16 *kv_gpu = nullptr, *act_gpu = nullptr, *kvr = nullptr;
    // fused recompute + attention (Engine::set_fused_recompute): partial
    // records [(act_gpu_cap + stage_act_cap) blocks][nseg][Hg][hd + 4] fp32
    // take the place of kvr
    float* part = nullptr;
    bool fused = false;
    int nseg = 1;  // records per block: tpb / min(tpb, 32)
    bool fused_supported() const { return dg % 128 == 0 && (hd == 64 || hd == 128) && tpb >= 4 && tpb <= 64; }
    f16 *kv_stage[2] = {nullptr, nullptr}, *act_stage[2] = {nullptr, nullptr};
    f16 *kv_host = nullptr, *act_host = nullptr;  // pinned, mapped (views into h_arena)
    f16* h_arena = nullptr;
    size_t h_arena_elems = 0;
    long kv_host_cap = 0, kv_gpu_cap = 0, act_host_cap = 0, act_gpu_cap = 0;
    f16 *x[2] = {nullptr, nullptr}, *qkvb = nullptr, *att = nullptr, *proj = nullptr, *hbuf = nullptr;
    float* logits = nullptr;
    int* amax = nullptr;
    float* attn_work = nullptr;
    float* splitk_ws = nullptr;  // split-K / stream-K partials of the weight-streaming decode GEMMs
    size_t splitk_floats = 0;
    // pdl: the tail GEMMs (proj / FFN1 / FFN2) always follow a kernel of this
    // stream, so they may launch programmatically (weight prefetch under the
    // predecessor's tail); off while profiling (span events sit between them)
    GemmScratch scratch(bool pdl = false) const { return GemmScratch{splitk_ws, splitk_floats, pdl ? 1 : 0}; }
    size_t attn_work_elems = 0;
    int* d_meta = nullptr;
    int* h_meta = nullptr;
    size_t meta_cap = 0;
    // prefill scratch
    f16 *px[2] = {nullptr, nullptr}, *pqkv = nullptr, *patt = nullptr, *pproj = nullptr, *ph = nullptr;
    size_t prefill_rows = 0, prefill_chunk_rows = 0;
    cudaEvent_t loaded[2]{}, consumed[2]{}, stored[2]{}, h2d_act[2]{}, gathered[2]{}, ev0{}, ev1{}, tg0{}, tg1{},
        wpre{};
    bool w_prefetched = false;  // wbuf[0/1] hold layers 0/1 for the next decode step
    // shared weight stream (EngineOptions::weight_share): this rank's slice of
    // wsS elements at wsr * wsS; wbuf slots hold wsn * wsS >= LE elements
    TpGroup* ws = nullptr;
    int wsn = 1, wsr = 0;
    size_t wsS = 0;
    cudaEvent_t w_h2d[2]{}, w_gath[2]{};
    cudaEvent_t w_consumed[2]{};  // wbuf[slot] released: the last unit of the layer that used it ended
    // mini-batched decode (set_minibatching): staging slots sized by the
    // packer's capacities instead of the whole host pools
    bool mb_on = false;
    PackerConfig packer{};
    TimingBundle packer_bundle{};
    long stage_kv_cap = 0, stage_act_cap = 0;  // blocks one staging slot holds
    float* agree_buf = nullptr;                // shared-weight-stream error agreement (1 float)
    // ranks sharing a weight stream agree on a step's validation outcome
    // before its first collective (an all-reduce of a failure flag)
    void agree_or_throw(const std::string& local_error, cudaStream_t st) {
        if (!agree_buf) agree_buf = dalloc<float>(1);
        const float flag = local_error.empty() ? 0.f : 1.f;
        HC_CUDA(cudaMemcpyAsync(agree_buf, &flag, 4, cudaMemcpyHostToDevice, st));
        ws->all_reduce_sum(agree_buf, 1, st);
        float sum = 0.f;
        HC_CUDA(cudaMemcpyAsync(&sum, agree_buf, 4, cudaMemcpyDeviceToHost, st));
        HC_CUDA(cudaStreamSynchronize(st));
        if (!local_error.empty()) throw InputError(local_error);
        if (sum > 0.f) throw InputError("decode_step: a rank sharing the weight stream rejected the step");
    }
    bool pools_filled = false;
    bool configured = false;  // false while (or after a failed) configure_cache: pools may be missing
    void require_configured() const {
        if (!configured) throw ConfigError("Engine: cache pools are not configured (configure_cache failed)");
    }
    f16* tr_kv = nullptr;  // [max_batch * max_blocks] KV blocks for token-recompute prefixes
    void ensure_tr() {
        if (!tr_kv) {
            clear_graphs();
            tr_kv = dalloc<f16>(static_cast<size_t>(B) * max_blocks * kvb);
        }
    }
    // CUDA graphs of the decode step, keyed by the step's launch structure
    // (the per-step data travels in the pinned metadata block the graph's
    // first node uploads, so a graph replays until blocks are appended)
    struct StepGraph {
        cudaGraphExec_t exec = nullptr;
        StepStats stats{};
        long last_use = 0;
    };
    std::unordered_map<std::string, StepGraph> graphs;
    long graph_gen = 0;  // bumped when any buffer a graph references is reallocated
    long graph_clock = 0;
    uint16_t* h_x = nullptr;   // pinned outputs of graph-mode steps
    float* h_logits = nullptr;
    int* h_amax = nullptr;
    void clear_graphs() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
        graphs.clear();
        ++graph_gen;
    }
    // profiling: timing events handed out per step
    std::vector<cudaEvent_t> pev;
    size_t pev_used = 0;
    cudaEvent_t take_event() {
        if (pev_used == pev.size()) {
            cudaEvent_t e;
            HC_CUDA(cudaEventCreate(&e));
            pev.push_back(e);
        }
        return pev[pev_used++];
    }
    struct Span {
        int kind;  // 0 recompute, 1 attention, 2 other gemm, 3 copy
        cudaEvent_t a, b;
        int layer;
        int minibatch;
    };
    std::vector<Span> spans;
    int cur_layer = -1, cur_mb = 0;
    void span_begin(bool on, cudaStream_t s, int kind) {
        if (!on) return;
        spans.push_back({kind, take_event(), nullptr, cur_layer, cur_mb});
        HC_CUDA(cudaEventRecord(spans.back().a, s));
    }
    void span_end(bool on, cudaStream_t s) {
        if (!on) return;
        spans.back().b = take_event();
        HC_CUDA(cudaEventRecord(spans.back().b, s));
    }

    void regions(int l, int slot, f16* r[16]) const {
        for (int i = 0; i < 16; ++i) r[i] = nullptr;
        r[R_KV_STAGE] = kv_stage[slot];
        r[R_KV_GPU] = kv_gpu ? kv_gpu + static_cast<size_t>(l) * kv_gpu_cap * kvb : nullptr;
        r[R_KVR] = kvr;
        r[R_ACT_STAGE] = act_stage[slot];
        r[R_ACT_GPU] = act_gpu ? act_gpu + static_cast<size_t>(l) * act_gpu_cap * actb : nullptr;
        r[R_KV_HOST] = kv_host ? kv_host + static_cast<size_t>(l % Lp) * kv_host_cap * kvb : nullptr;
        r[R_ACT_HOST] = act_host ? act_host + static_cast<size_t>(l % Lp) * act_cap_n * actb : nullptr;
        r[R_TOKREC] = tr_kv;
    }
    const f16* layer_w(int l, int slot) const { return w_all ? w_all + static_cast<size_t>(l) * LE : wbuf[slot]; }

    // unsharded packed layer `full` (device) -> this rank's shard at dst
    // (device or pinned host; kind says which)
    void extract_shard(const f16* full, void* dstv, cudaMemcpyKind kind, cudaStream_t st) const {
        uint16_t* dst = static_cast<uint16_t*>(dstv);
        const uint16_t* F = reinterpret_cast<const uint16_t*>(full);
        const size_t D = d, Fd = f, g = tpr, DG = dg, FG = fg;
        auto cp = [&](size_t o, size_t so, size_t n) {
            HC_CUDA(cudaMemcpyAsync(dst + o, F + so, n * 2, kind, st));
        };
        auto cp2 = [&](size_t o, size_t dpitch, size_t so, size_t spitch, size_t width, size_t rows) {
            HC_CUDA(cudaMemcpy2DAsync(dst + o, dpitch * 2, F + so, spitch * 2, width * 2, rows, kind, st));
        };
        for (size_t k = 0; k < 3; ++k) cp(off.wqkv + k * DG * D, offF.wqkv + (k * D + g * DG) * D, DG * D);  // head rows
        cp2(off.wproj, DG, offF.wproj + g * DG, D, DG, D);  // Wproj^T columns = the heads' input rows of W_o
        cp(off.w1, offF.w1 + g * FG * D, FG * D);
        cp2(off.w2, FG, offF.w2 + g * FG, Fd, FG, D);
        if (opt()) {
            for (size_t k = 0; k < 3; ++k) cp(off.bqkv + k * DG, offF.bqkv + k * D + g * DG, DG);
            cp(off.bproj, offF.bproj, D);
            cp(off.b1, offF.b1 + g * FG, FG);
            cp(off.b2, offF.b2, D);
            cp(off.ln1g, offF.ln1g, 4 * D);
        }
    }

    // ---- decoder-layer arithmetic shared by decode, prefill and traces ----
    bool opt() const { return arch == kArchOpt; }
    const f16* bias(const f16* W, size_t o) const { return opt() ? W + o : nullptr; }
    // LN1 (which = 1) / LN2 (2) of T rows of x into out for kArchOpt; the
    // reference arch has no LayerNorm and returns x itself
    const f16* ln(const f16* W, int which, const f16* x, int T, f16* out, cudaStream_t st) const {
        if (!opt()) return x;
        layernorm_rows(x, d, W + (which == 1 ? off.ln1g : off.ln2g), W + (which == 1 ? off.ln1b : off.ln2b), out, d,
                       T, d, static_cast<float>(kLnEps), st);
        return out;
    }
    // qkv [T x 3dg] = LN1(x) . Wqkv (+ b_qkv) for this rank's heads
    // (qkv_generate, decoder.cpp:97-103)
    // q_only: the Q columns alone (rows 0..dg of Wqkv^T) into the same [T x 3dg]
    // layout — a fused decode step whose new tokens all land in ACT blocks gets
    // their K|V from the recompute, so the K|V thirds of the weights need not stream
    void qkv(const f16* W, const f16* xa, int T, f16* out, cudaStream_t st,
             const GemmScratch& sc = GemmScratch{}, bool q_only = false) const {
        // no programmatic launch: QKV may follow a cross-stream event wait
        const GemmScratch s{sc.ws, sc.floats, 0};
        gemm_rows(gemm::kStore, xa, T, d, W + off.wqkv, (q_only ? 1 : 3) * dg, out, 3 * dg, st, 0, s,
                  bias(W, off.bqkv));
    }
    // project_ffn (decoder.cpp:113-121) of T attention rows [T x dg]; kArchOpt
    // adds the biases, the two residuals (x, then x') and LN2. Head-sharded:
    // W_proj / W2 are row slices, so their outputs are partial sums that one
    // all-reduce each completes (bias and residual enter once, on rank 0).
    // lnbuf may alias att.
    void tail(const f16* W, const f16* att, const f16* x, int T, f16* proj, f16* lnbuf, f16* h, f16* out,
              cudaStream_t st, const GemmScratch& sc = GemmScratch{}) {
        if (tpn == 1) {  // bias + residual fused into the GEMM epilogues
            gemm_rows(gemm::kStore, att, T, d, W + off.wproj, d, proj, d, st, 0, sc, bias(W, off.bproj),
                      opt() ? x : nullptr, d);
            const f16* p2 = ln(W, 2, proj, T, lnbuf, st);
            gemm_rows(gemm::kRelu, p2, T, d, W + off.w1, f, h, f, st, 0, sc, bias(W, off.b1));
            gemm_rows(gemm::kStore, h, T, f, W + off.w2, d, out, d, st, 0, sc, bias(W, off.b2),
                      opt() ? proj : nullptr, d);
            return;
        }
        // head-sharded: fp32 partial sums -> all-reduce -> + bias + residual
        float* r = ensure_red(static_cast<size_t>(T) * d);
        gemm_rows(gemm::kF32, att, T, dg, W + off.wproj, d, r, d, st, 0, sc);
        tp->all_reduce_sum(r, static_cast<size_t>(T) * d, st);
        add_bias_residual(r, bias(W, off.bproj), opt() ? x : nullptr, d, T, d, proj, st);
        const f16* p2 = ln(W, 2, proj, T, lnbuf, st);
        gemm_rows(gemm::kRelu, p2, T, d, W + off.w1, fg, h, fg, st, 0, sc, bias(W, off.b1));
        gemm_rows(gemm::kF32, h, T, fg, W + off.w2, d, r, d, st, 0, sc);
        tp->all_reduce_sum(r, static_cast<size_t>(T) * d, st);
        add_bias_residual(r, bias(W, off.b2), opt() ? proj : nullptr, d, T, d, out, st);
    }
    int tail_launches() const { return (opt() ? 4 : 3) + (tpn > 1 ? 2 : 0); }
    float* red = nullptr;  // tensor-parallel partial sums [rows x d] fp32
    size_t red_elems = 0;
    float* ensure_red(size_t elems) {
        if (elems > red_elems) {
            if (red) HC_CUDA(cudaFree(red));
            red = nullptr;  // stays null if the new allocation fails
            red_elems = 0;
            red = dalloc<float>(elems);
            red_elems = elems;
        }
        return red;
    }
    // model output: LN_f(x) for kArchOpt (into out), x itself otherwise
    const f16* final_norm(const f16* x, int T, f16* out, cudaStream_t st) const {
        if (!opt()) return x;
        layernorm_rows(x, d, lnf, lnf + d, out, d, T, d, static_cast<float>(kLnEps), st);
        return out;
    }

    void ensure_meta(size_t ints) {
        if (ints <= meta_cap) return;
        clear_graphs();
        if (d_meta) cudaFree(d_meta);
        if (h_meta) cudaFreeHost(h_meta);
        meta_cap = ints + ints / 2 + 1024;
        d_meta = dalloc<int>(meta_cap);
        h_meta = halloc<int>(meta_cap, false);
    }
    void ensure_attn_work(size_t elems) {
        if (elems <= attn_work_elems) return;
        clear_graphs();
        if (attn_work) cudaFree(attn_work);
        attn_work_elems = elems;
        attn_work = dalloc<float>(elems);
    }
    // px: layer input/output rows of the whole prefill (all requests);
    // pqkv/patt/pproj/ph: per-chunk scratch (chunk_rows <= rows)
    void ensure_prefill(size_t rows, size_t chunk_rows = 0) {
        if (!chunk_rows) chunk_rows = rows;
        if (rows > prefill_rows || chunk_rows > prefill_chunk_rows) clear_graphs();
        if (rows > prefill_rows) {
            for (f16* p : {px[0], px[1], pxn})
                if (p) cudaFree(p);
            prefill_rows = rows;
            px[0] = dalloc<f16>(rows * d);
            px[1] = dalloc<f16>(rows * d);
            pxn = opt() ? dalloc<f16>(rows * d) : nullptr;
        }
        if (chunk_rows > prefill_chunk_rows) {
            for (f16* p : {pqkv, patt, pproj, ph})
                if (p) cudaFree(p);
            prefill_chunk_rows = chunk_rows;
            pqkv = dalloc<f16>(chunk_rows * 3 * d);
            patt = dalloc<f16>(chunk_rows * d);
            pproj = dalloc<f16>(chunk_rows * d);
            ph = dalloc<f16>(chunk_rows * f);
        }
    }
};

namespace {
struct HostWeightsCtx {
    const HostWeights* w;
};
void fill_from_hostweights(const void* ctx, int l, uint16_t* dst) {
    const HostWeights* w = static_cast<const HostWeightsCtx*>(ctx)->w;
    std::memcpy(dst, w->layer(l), w->layer_elems() * 2);
}
}  // namespace

Engine::Engine(const HostWeights& w, const EngineOptions& o) : opt_(o) {
    HostWeightsCtx ctx{&w};
    opt_.arch = w.arch;
    if (w.arch == kArchOpt && w.final_ln.size() != 2 * static_cast<size_t>(w.config.hidden_dim))
        throw InputError("opt arch weights need the final LayerNorm (2 x hidden_dim)");
    init(w.config, w.max_seq, w.embedding.data(), w.positional.data(), w.arch == kArchOpt ? w.final_ln.data() : nullptr,
         fill_from_hostweights, &ctx);
}

Engine::Engine(const ModelConfig& c, uint64_t seed, int max_seq, bool rescale, const EngineOptions& o) : opt_(o) {
    ModelConfig cc = c;
    cc.validate();
    if (max_seq < 1) throw InputError("DecoderWeights: max_seq must be >= 1");
    // draw on the GPU (bit-exact with the host generator, weights_gen.cu);
    // the kArchOpt vectors (a few d-sized draws per layer) on the host
    std::vector<uint16_t> lnf;
    if (opt_.arch == kArchOpt) {
        lnf.resize(2 * static_cast<size_t>(cc.hidden_dim));
        generate_final_ln(cc, seed, lnf.data());
    }
    init(cc, max_seq, nullptr, nullptr, lnf.empty() ? nullptr : lnf.data(), nullptr, nullptr);
    Impl& m = *impl_;
    gen_weights_plain(reinterpret_cast<uint16_t*>(m.emb), static_cast<size_t>(m.V) * m.d, mix_seed(seed, 0),
                      s_compute_);
    gen_weights_plain(reinterpret_cast<uint16_t*>(m.pos), static_cast<size_t>(max_seq) * m.d, mix_seed(seed, 1),
                      s_compute_);
    double fac[6];
    rescale_factors(cfg_, fac);
    const int d = m.d, f = m.f;
    // the unsharded layer (reference tags and layout), drawn in place or into
    // wfull and then cut to this rank's shard
    auto draw_layer = [&](int l, f16* dst) {
        uint16_t* L = reinterpret_cast<uint16_t*>(dst);
        const LayerOffsets& o = m.offF;
        const uint64_t base = 100 + static_cast<uint64_t>(l) * 8;  // model.cpp:90, 106-113
        for (int k = 0; k < 3; ++k)
            gen_weights_transposed(L + o.wqkv + static_cast<size_t>(k) * d * d, d, d, mix_seed(seed, base + k),
                                   fac[k], rescale, s_compute_);
        gen_weights_transposed(L + o.wproj, d, d, mix_seed(seed, base + 3), fac[3], rescale, s_compute_);
        gen_weights_transposed(L + o.w1, d, f, mix_seed(seed, base + 4), fac[4], rescale, s_compute_);
        gen_weights_transposed(L + o.w2, f, d, mix_seed(seed, base + 5), fac[5], rescale, s_compute_);
        if (m.opt()) {
            const size_t n = m.LEF - o.bqkv;
            std::vector<uint16_t> ex(m.LEF);
            generate_layer_extras(cfg_, seed, l, ex.data());
            HC_CUDA(cudaMemcpyAsync(L + o.bqkv, ex.data() + o.bqkv, n * 2, cudaMemcpyHostToDevice, s_compute_));
            HC_CUDA(cudaStreamSynchronize(s_compute_));  // ex is pageable and goes out of scope
        }
    };
    for (int l = 0; l < (m.w_all ? m.L : m.Lw); ++l) {
        f16* shard = m.w_all ? m.w_all + static_cast<size_t>(l) * m.LE : m.wbuf[l & 1];
        if (m.tpn == 1) {
            draw_layer(l, shard);
        } else {
            draw_layer(l, m.wfull);
            m.extract_shard(m.wfull, shard, cudaMemcpyDeviceToDevice, s_compute_);
        }
        if (!m.w_all)
            HC_CUDA(cudaMemcpyAsync(m.h_w + static_cast<size_t>(l) * m.LE, shard, m.LE * 2, cudaMemcpyDeviceToHost,
                                    s_compute_));
    }
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    if (m.wfull) {
        HC_CUDA(cudaFree(m.wfull));
        m.wfull = nullptr;
    }
}

void Engine::init(const ModelConfig& c, int w_max_seq, const uint16_t* emb, const uint16_t* pos, const uint16_t* lnf,
                  void (*fill_layer)(const void*, int, uint16_t*), const void* ctx) {
    cfg_ = c;
    cfg_.validate();
    impl_ = std::make_unique<Impl>();
    Impl& m = *impl_;
    if (opt_.arch != kArchReference && opt_.arch != kArchOpt) throw InputError("Engine: unknown arch");
    if (const char* e = std::getenv("HC_DECODE_GRAPHS")) graphs_ = e[0] != '0';
    m.arch = opt_.arch;
    if (cfg_.hidden_dim % 64) throw InputError("Engine: hidden_dim must be a multiple of 64");
    if (cfg_.head_dim() != 64 && cfg_.head_dim() != 128) throw InputError("Engine: head_dim must be 64 or 128");
    if (!decode_attention_supported(cfg_.head_dim(), cfg_.tokens_per_block))
        throw InputError("Engine: tokens_per_block must be 4, 8, 16, 32 or 64");
    if (cfg_.ffn_dim % 64) throw InputError("Engine: ffn_dim must be a multiple of 64");
    if (cfg_.vocab_size % 16) throw InputError("Engine: vocab_size must be a multiple of 16");
    if (opt_.max_batch < 1) throw InputError("Engine: max_batch must be >= 1");
    HC_CUDA(cudaSetDevice(opt_.device));
    m.L = cfg_.num_layers;
    m.d = cfg_.hidden_dim;
    m.H = cfg_.num_heads;
    m.hd = cfg_.head_dim();
    m.f = cfg_.ffn_dim;
    m.V = cfg_.vocab_size;
    m.tpb = cfg_.tokens_per_block;
    m.B = opt_.max_batch;
    m.max_seq = opt_.max_seq > 0 ? std::min(opt_.max_seq, w_max_seq) : w_max_seq;
    m.max_blocks = (m.max_seq + m.tpb - 1) / m.tpb;
    m.Lp = opt_.host_layers > 0 ? std::min(opt_.host_layers, m.L) : m.L;
    m.Lw = opt_.weight_layers > 0 ? std::min(opt_.weight_layers, m.L) : m.L;
    m.tp = opt_.tp;
    m.tpn = m.tp ? m.tp->size() : 1;
    m.tpr = m.tp ? m.tp->rank() : 0;
    if (opt_.weight_share && opt_.weight_share->size() > 1) {
        if (opt_.weights_on_device) throw ConfigError("weight_share: needs streamed weights (weights_on_device = 0)");
        if (m.tp) throw ConfigError("weight_share: not combined with tensor parallelism (heads already shard weights)");
        m.ws = opt_.weight_share;
        m.wsn = m.ws->size();
        m.wsr = m.ws->rank();
    }
    if (m.H % m.tpn || m.f % m.tpn) throw InputError("tensor parallel size must divide num_heads and ffn_dim");
    m.Hg = m.H / m.tpn;
    m.dg = m.d / m.tpn;
    m.fg = m.f / m.tpn;
    if (m.dg % 64 || m.fg % 64) throw InputError("tensor parallel: per-rank hidden / ffn slices must be multiples of 64");
    {
        const char* e = std::getenv("HC_FUSED_RECOMPUTE");  // 0: recompute writes K|V (kKvPaged) by default
        m.fused = m.fused_supported() && !(e && e[0] == '0');
    }
    m.off = LayerOffsets::of(cfg_, m.arch, m.tpn);
    m.offF = LayerOffsets::of(cfg_, m.arch, 1);
    m.LE = m.off.total;
    m.LEF = m.offF.total;
    m.wsS = (m.LE + m.wsn - 1) / m.wsn;
    m.wsS = (m.wsS + 63) / 64 * 64;  // 128-byte aligned slices
    m.kvb = static_cast<size_t>(2) * m.dg * m.tpb;  // this rank's heads of a KV block
    m.actb = static_cast<size_t>(m.d) * m.tpb;

    HC_CUDA(cudaStreamCreateWithFlags(&s_compute_, cudaStreamNonBlocking));
    HC_CUDA(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking));
    HC_CUDA(cudaStreamCreateWithFlags(&s_store_, cudaStreamNonBlocking));
    HC_CUDA(cudaStreamCreateWithFlags(&s_gather_, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        HC_CUDA(cudaEventCreateWithFlags(&m.loaded[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.consumed[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.stored[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.h2d_act[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.gathered[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.w_h2d[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.w_gath[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&m.w_consumed[i], cudaEventDisableTiming));
    }
    HC_CUDA(cudaEventCreate(&m.ev0));
    HC_CUDA(cudaEventCreate(&m.ev1));
    HC_CUDA(cudaEventCreate(&m.tg0));
    HC_CUDA(cudaEventCreate(&m.tg1));
    HC_CUDA(cudaEventCreateWithFlags(&m.wpre, cudaEventDisableTiming));

    // tables
    m.emb = dalloc<f16>(static_cast<size_t>(m.V) * m.d);
    m.pos = dalloc<f16>(static_cast<size_t>(w_max_seq) * m.d);
    if (emb) HC_CUDA(cudaMemcpy(m.emb, emb, static_cast<size_t>(m.V) * m.d * 2, cudaMemcpyHostToDevice));
    if (pos) HC_CUDA(cudaMemcpy(m.pos, pos, static_cast<size_t>(w_max_seq) * m.d * 2, cudaMemcpyHostToDevice));
    if (m.opt()) {
        if (!lnf) throw InputError("Engine: opt arch needs the final LayerNorm");
        m.lnf = dalloc<f16>(2 * static_cast<size_t>(m.d));
        HC_CUDA(cudaMemcpy(m.lnf, lnf, 2 * static_cast<size_t>(m.d) * 2, cudaMemcpyHostToDevice));
        m.xn = dalloc<f16>(static_cast<size_t>(m.B) * m.d);
    }

    // weights (fill_layer == nullptr: the caller draws them on the device);
    // fill_layer delivers the unsharded layer, cut to the rank's shard here
    if (m.tpn > 1) m.wfull = dalloc<f16>(m.LEF);
    std::vector<uint16_t> tmp(fill_layer && m.tpn > 1 ? m.LEF : 0);
    auto place = [&](int l, void* dst, cudaMemcpyKind kind) {
        fill_layer(ctx, l, tmp.data());
        HC_CUDA(cudaMemcpy(m.wfull, tmp.data(), m.LEF * 2, cudaMemcpyHostToDevice));
        m.extract_shard(m.wfull, dst, kind, s_compute_);
        HC_CUDA(cudaStreamSynchronize(s_compute_));
    };
    if (opt_.weights_on_device) {
        m.w_all = dalloc<f16>(m.LE * m.L);
        std::vector<uint16_t> t1(fill_layer && m.tpn == 1 ? m.LE : 0);
        for (int l = 0; fill_layer && l < m.L; ++l) {
            f16* dst = m.w_all + static_cast<size_t>(l) * m.LE;
            if (m.tpn > 1) {
                place(l, dst, cudaMemcpyDeviceToDevice);
            } else {
                fill_layer(ctx, l, t1.data());
                HC_CUDA(cudaMemcpy(dst, t1.data(), m.LE * 2, cudaMemcpyHostToDevice));
            }
        }
    } else {
        m.h_w = halloc<uint16_t>(m.LE * m.Lw, false);
        for (int l = 0; fill_layer && l < m.Lw; ++l) {
            if (m.tpn > 1)
                place(l, m.h_w + static_cast<size_t>(l) * m.LE, cudaMemcpyDeviceToHost);
            else
                fill_layer(ctx, l, m.h_w + static_cast<size_t>(l) * m.LE);
        }
        m.wbuf[0] = dalloc<f16>(m.wsn * m.wsS);  // >= LE (padded slices when the stream is shared)
        m.wbuf[1] = dalloc<f16>(m.wsn * m.wsS);
    }
    if (fill_layer && m.wfull) {
        HC_CUDA(cudaFree(m.wfull));
        m.wfull = nullptr;
    }

    // decode scratch
    m.x[0] = dalloc<f16>(static_cast<size_t>(m.B) * m.d);
    m.x[1] = dalloc<f16>(static_cast<size_t>(m.B) * m.d);
    m.qkvb = dalloc<f16>(static_cast<size_t>(m.B) * 3 * m.d);
    m.att = dalloc<f16>(static_cast<size_t>(m.B) * m.d);
    m.proj = dalloc<f16>(static_cast<size_t>(m.B) * m.d);
    m.hbuf = dalloc<f16>(static_cast<size_t>(m.B) * m.f);
    m.logits = dalloc<float>(static_cast<size_t>(m.B) * m.V);
    m.amax = dalloc<int>(m.B);
    m.splitk_floats = std::max(static_cast<size_t>(16) * m.B * std::max(3 * m.d, m.f), wstream_ws_floats(m.B));
    m.splitk_ws = dalloc<float>(m.splitk_floats);
    configure_cache(PoolCaps{opt_.kv_host_cap, opt_.kv_gpu_cap, opt_.act_host_cap, opt_.act_gpu_cap}, opt_.kv_on_gpu != 0,
                    opt_.mode, opt_.alloc, opt_.host_layers, opt_.recompute_ratio);
}

void Engine::configure_cache(const PoolCaps& caps, bool kv_on_gpu, CacheMode mode, const HostAllocation& alloc,
                             int host_layers, double recompute_ratio) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    opt_.recompute_ratio = recompute_ratio;
    if (mode == CacheMode::TokenRecompute && (opt_.recompute_ratio < 0.0 || opt_.recompute_ratio > 1.0))
        throw ConfigError("Engine: recompute_ratio must lie in [0, 1]");
    if (mode == CacheMode::Hybrid && alloc.act_host + alloc.kv_host <= 0)
        throw ConfigError("Engine: hybrid mode needs a nonempty host allocation (ratio target)");
    if (mode == CacheMode::TokenRecompute && m.tpn > 1)
        throw ConfigError("Engine: the token-recompute baseline runs without tensor parallelism");
    HC_CUDA(cudaDeviceSynchronize());
    m.configured = false;
    m.clear_graphs();
    for (f16** p : {&m.kv_gpu, &m.act_gpu, &m.kvr, &m.kv_stage[0], &m.kv_stage[1], &m.act_stage[0], &m.act_stage[1]}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    m.kv_host = m.act_host = nullptr;  // views into the pinned arena (re-carved below)
    assigner_.reset();
    opt_.kv_host_cap = caps.kv_host;
    opt_.kv_gpu_cap = caps.kv_gpu;
    opt_.act_host_cap = caps.act_host;
    opt_.act_gpu_cap = caps.act_gpu;
    opt_.kv_on_gpu = kv_on_gpu;
    opt_.mode = mode;
    opt_.alloc = alloc;
    opt_.host_layers = host_layers;
    m.kv_host_cap = caps.kv_host;
    m.kv_gpu_cap = caps.kv_gpu;
    m.act_host_cap = caps.act_host;
    m.act_gpu_cap = caps.act_gpu;
    m.Lp = host_layers > 0 ? std::min(host_layers, m.L) : m.L;
    // rebuilt IN PLACE: borrowed handles (hc_engine_cache) stay valid
    if (cache_)
        *cache_ = HybridCache(m.tpb, caps, kv_on_gpu);
    else
        cache_ = std::make_unique<HybridCache>(m.tpb, caps, kv_on_gpu);
    // token recompute keeps a block-aligned PREFIX of every prompt as ids only
    // (exact recompute needs a prefix) and caches the rest as KV
    token_mode_ = mode == CacheMode::TokenRecompute;
    rc_ids_.clear();
    assigner_ = std::make_unique<BlockAssigner>(*cache_, token_mode_ ? CacheMode::KvOnly : mode, alloc, 0.0);
    m.kv_gpu = dalloc<f16>(static_cast<size_t>(m.L) * m.kv_gpu_cap * m.kvb);
    m.act_gpu = dalloc<f16>(static_cast<size_t>(m.L) * m.act_gpu_cap * m.actb);
    if (std::getenv("HC_POISON")) {  // debug: NaN in every slot no writer has filled yet
        if (m.kv_gpu) HC_CUDA(cudaMemset(m.kv_gpu, 0xFF, static_cast<size_t>(m.L) * m.kv_gpu_cap * m.kvb * 2));
        if (m.act_gpu) HC_CUDA(cudaMemset(m.act_gpu, 0xFF, static_cast<size_t>(m.L) * m.act_gpu_cap * m.actb * 2));
    }
    m.act_cap_n = (m.act_host_cap + m.tpn - 1) / m.tpn;
    // pinned, mapped host pools: one arena, kept across configure_cache calls
    // while it is large enough (pinning tens of GB takes seconds per call)
    {
        const size_t kv_e = static_cast<size_t>(m.Lp) * m.kv_host_cap * m.kvb;
        const size_t kv_e_al = (kv_e + 127) / 128 * 128;  // 256-byte aligned ACT pool
        const size_t act_e = static_cast<size_t>(m.Lp) * m.act_cap_n * m.actb;
        const size_t need = kv_e_al + act_e;
        if (need > m.h_arena_elems) {
            if (m.h_arena) HC_CUDA(cudaFreeHost(m.h_arena));
            m.h_arena = nullptr;  // stays null if the new allocation fails
            m.h_arena_elems = 0;
            m.h_arena = halloc<f16>(need, true);
            m.h_arena_elems = need;
        }
        m.kv_host = kv_e ? m.h_arena : nullptr;
        m.act_host = act_e ? m.h_arena + kv_e_al : nullptr;
    }
    alloc_staging();
    m.pools_filled = false;
    HC_CUDA(cudaDeviceSynchronize());
    m.configured = true;
}

// Staging slots (two, double-buffered) for the host blocks of one decode unit
// and the recompute output: the whole host pools for whole-batch steps (the
// slot mirrors the pool's pbn layout), the packer's capacities plus one
// growth block per request for mini-batched steps.
void Engine::alloc_staging() {
    Impl& m = *impl_;
    for (f16** p : {&m.kvr, &m.kv_stage[0], &m.kv_stage[1], &m.act_stage[0], &m.act_stage[1]}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    if (m.part) cudaFree(m.part);
    m.part = nullptr;
    m.stage_kv_cap = m.kv_host_cap;
    m.stage_act_cap = static_cast<long>(m.tpn) * m.act_cap_n;
    if (m.mb_on) {
        m.stage_kv_cap = std::min(m.stage_kv_cap, m.packer.kv_max + m.B);
        m.stage_act_cap = std::min(m.stage_act_cap, m.packer.act_max + m.B);
    }
    for (int s = 0; s < 2; ++s) {
        m.kv_stage[s] = dalloc<f16>(static_cast<size_t>(m.stage_kv_cap) * m.kvb);
        m.act_stage[s] = dalloc<f16>(static_cast<size_t>(m.stage_act_cap) * m.actb);
    }
    m.nseg = m.tpb / std::min(m.tpb, 32);
    if (m.fused) {  // partial records instead of recomputed K|V blocks
        const size_t n = static_cast<size_t>(m.act_gpu_cap + m.stage_act_cap) * m.nseg * m.Hg * (m.hd + 4);
        m.part = dalloc<float>(n);
        if (std::getenv("HC_POISON"))  // debug: NaN records expose any record read before it is written
            HC_CUDA(cudaMemset(m.part, 0xFF, n * sizeof(float)));
    }
    else
        m.kvr = dalloc<f16>(static_cast<size_t>(m.act_gpu_cap + m.stage_act_cap) * m.kvb);
    // staging slots start zeroed: whole-chunk copies (D2H runs, TP all-gathers)
    // never move uninitialised bytes, even for slots no block occupies yet
    for (int s = 0; s < 2; ++s) {
        const int fill = std::getenv("HC_POISON") ? 0xFF : 0;  // debug: NaN staging
        if (m.kv_stage[s]) HC_CUDA(cudaMemset(m.kv_stage[s], fill, static_cast<size_t>(m.stage_kv_cap) * m.kvb * 2));
        if (m.act_stage[s]) HC_CUDA(cudaMemset(m.act_stage[s], fill, static_cast<size_t>(m.stage_act_cap) * m.actb * 2));
    }
}

bool Engine::set_fused_recompute(bool on) {
    HC_CUDA(cudaSetDevice(opt_.device));
    Impl& m = *impl_;
    on = on && m.fused_supported();
    if (on == m.fused) return on;
    HC_CUDA(cudaDeviceSynchronize());
    m.clear_graphs();
    m.fused = on;
    if (m.configured) {
        m.configured = false;
        alloc_staging();
        HC_CUDA(cudaDeviceSynchronize());
        m.configured = true;
    }
    return on;
}

bool Engine::fused_recompute() const { return impl_->fused; }

void Engine::set_minibatching(long act_max, long kv_max, const TimingBundle& bundle) {
    HC_CUDA(cudaSetDevice(opt_.device));
    Impl& m = *impl_;
    m.require_configured();
    const bool on = act_max > 0 || kv_max > 0;
    if (on && (act_max < 1 || kv_max < 1)) throw InputError("form_minibatches: capacities must be >= 1");
    if (on && (m.tpn > 1 || m.wsn > 1))
        throw ConfigError("Engine: mini-batched decode runs without tensor parallelism or a shared weight stream");
    HC_CUDA(cudaDeviceSynchronize());
    m.clear_graphs();
    m.mb_on = on;
    m.packer = PackerConfig{act_max, kv_max};
    m.packer_bundle = bundle;
    m.configured = false;
    alloc_staging();
    HC_CUDA(cudaDeviceSynchronize());
    m.configured = true;
}

void Engine::forward_trace(const std::vector<int>& ids, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                           uint16_t* out) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    const int T = static_cast<int>(ids.size());
    if (T == 0) return;
    if (T > m.max_seq) throw InputError("embed: sequence longer than max_seq");
    for (int t : ids)
        if (t < 0 || t >= m.V) throw InputError("embed: token id out of range: " + std::to_string(t));
    m.ensure_prefill(T);
    std::vector<int> meta(ids);
    for (int t = 0; t < T; ++t) meta.push_back(t);
    meta.push_back(0);
    meta.push_back(T);
    m.ensure_meta(meta.size());
    std::memcpy(m.h_meta, meta.data(), meta.size() * 4);
    HC_CUDA(cudaMemcpyAsync(m.d_meta, m.h_meta, meta.size() * 4, cudaMemcpyHostToDevice, s_compute_));
    embed(m.emb, m.pos, m.d_meta, m.d_meta + T, T, m.d, m.px[0], m.d, s_compute_);
    run_layers(T, 0, m.L, m.d_meta + 2 * T, layer_inputs, k, v, out, true);
}

void Engine::layer_forward(int layer, const uint16_t* x, int T, uint16_t* k, uint16_t* v, uint16_t* out) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    if (layer < 0 || layer >= m.L) throw InputError("layer index out of range: " + std::to_string(layer));
    if (T <= 0) return;
    if (T > m.max_seq) throw InputError("layer_forward: more rows than max_seq");
    m.ensure_prefill(T);
    const int cu[2] = {0, T};
    m.ensure_meta(2);
    std::memcpy(m.h_meta, cu, sizeof cu);
    HC_CUDA(cudaMemcpyAsync(m.d_meta, m.h_meta, sizeof cu, cudaMemcpyHostToDevice, s_compute_));
    HC_CUDA(cudaMemcpyAsync(m.px[layer & 1], x, static_cast<size_t>(T) * m.d * 2, cudaMemcpyHostToDevice, s_compute_));
    run_layers(T, layer, layer + 1, m.d_meta, nullptr, k, v, out, false);
}

Engine::~Engine() {
    if (!impl_) return;
    Impl& m = *impl_;
    cudaSetDevice(opt_.device);
    cudaDeviceSynchronize();
    for (void* p : {(void*)m.emb, (void*)m.pos, (void*)m.w_all, (void*)m.wbuf[0], (void*)m.wbuf[1], (void*)m.kv_gpu,
                    (void*)m.act_gpu, (void*)m.kvr, (void*)m.kv_stage[0], (void*)m.kv_stage[1], (void*)m.act_stage[0],
                    (void*)m.act_stage[1], (void*)m.x[0], (void*)m.x[1], (void*)m.qkvb, (void*)m.att, (void*)m.proj,
                    (void*)m.hbuf, (void*)m.logits, (void*)m.amax, (void*)m.attn_work, (void*)m.d_meta,
                    (void*)m.px[0], (void*)m.px[1], (void*)m.pqkv, (void*)m.patt, (void*)m.pproj, (void*)m.ph,
                    (void*)m.tr_kv, (void*)m.splitk_ws, (void*)m.lnf, (void*)m.xn, (void*)m.pxn, (void*)m.red,
                    (void*)m.agree_buf, (void*)m.part})
        if (p) cudaFree(p);
    for (auto& g : m.graphs) cudaGraphExecDestroy(g.second.exec);
    for (void* p : {(void*)m.h_w, (void*)m.h_arena, (void*)m.h_meta, (void*)m.h_x,
                    (void*)m.h_logits, (void*)m.h_amax})
        if (p) cudaFreeHost(p);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(m.loaded[i]);
        cudaEventDestroy(m.consumed[i]);
        cudaEventDestroy(m.w_consumed[i]);
        cudaEventDestroy(m.stored[i]);
        cudaEventDestroy(m.h2d_act[i]);
        cudaEventDestroy(m.gathered[i]);
        cudaEventDestroy(m.w_h2d[i]);
        cudaEventDestroy(m.w_gath[i]);
    }
    cudaEventDestroy(m.ev0);
    cudaEventDestroy(m.ev1);
    cudaEventDestroy(m.tg0);
    cudaEventDestroy(m.tg1);
    cudaEventDestroy(m.wpre);
    for (cudaEvent_t e : m.pev) cudaEventDestroy(e);
    cudaStreamDestroy(s_compute_);
    cudaStreamDestroy(s_copy_);
    cudaStreamDestroy(s_store_);
    cudaStreamDestroy(s_gather_);
}

// Causal forward of T rows (one sequence) through layers [l0, l1); the input
// is in px[l0 & 1]; captures are [l1-l0][T][d] host arrays (optional).
void Engine::run_layers(int T, int l0, int l1, const int* d_cu, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                        uint16_t* out, bool final_ln) {
    Impl& m = *impl_;
    if (m.tpn > 1) throw ConfigError("forward_trace / layer_forward run on an engine without tensor parallelism");
    m.w_prefetched = false;
    const size_t per = static_cast<size_t>(T) * m.d;
    std::vector<uint16_t> qkv_h((k || v) ? static_cast<size_t>(T) * 3 * m.d : 0);
    for (int l = l0; l < l1; ++l) {
        const int slot = l & 1;
        const size_t li = static_cast<size_t>(l - l0);
        if (!m.w_all) {
            HC_CUDA(cudaStreamSynchronize(s_compute_));
            HC_CUDA(cudaMemcpy(m.wbuf[slot], m.h_w + static_cast<size_t>(l % m.Lw) * m.LE, m.LE * 2,
                               cudaMemcpyHostToDevice));
        }
        const f16* W = m.layer_w(l, slot);
        f16* xin = m.px[l & 1];
        f16* xout = m.px[(l + 1) & 1];
        if (layer_inputs)
            HC_CUDA(cudaMemcpyAsync(layer_inputs + per * li, xin, per * 2, cudaMemcpyDeviceToHost, s_compute_));
        m.qkv(W, m.ln(W, 1, xin, T, m.pxn, s_compute_), T, m.pqkv, s_compute_);
        if (k || v) {
            HC_CUDA(cudaMemcpyAsync(qkv_h.data(), m.pqkv, qkv_h.size() * 2, cudaMemcpyDeviceToHost, s_compute_));
            HC_CUDA(cudaStreamSynchronize(s_compute_));
            for (int t = 0; t < T; ++t) {
                const uint16_t* row = qkv_h.data() + static_cast<size_t>(t) * 3 * m.d;
                if (k) std::memcpy(k + per * li + static_cast<size_t>(t) * m.d, row + m.d, m.d * 2);
                if (v) std::memcpy(v + per * li + static_cast<size_t>(t) * m.d, row + 2 * m.d, m.d * 2);
            }
        }
        prefill_attention(m.pqkv, m.patt, d_cu, 1, T, m.H, m.hd,
                          opt_.scaled ? 1.0f / std::sqrt(static_cast<float>(m.hd)) : 1.0f, s_compute_, T);
        m.tail(W, m.patt, xin, T, m.pproj, m.patt, m.ph, xout, s_compute_);
    }
    const f16* y = final_ln ? m.final_norm(m.px[l1 & 1], T, m.pxn, s_compute_) : m.px[l1 & 1];
    if (out) HC_CUDA(cudaMemcpyAsync(out, y, per * 2, cudaMemcpyDeviceToHost, s_compute_));
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaStreamSynchronize(s_compute_));
}

// ---------------------------------------------------------------------------
// GEMM helpers (weights transposed [out][in]; see model.hpp)
void gemm_rows(int epi, const f16* A, int M, int K, const f16* W, int N, void* out, long long ldc, cudaStream_t st,
               long long lda, const GemmScratch& sc, const f16* bias, const f16* res, long long ldr) {
    GemmCall c;
    c.epi = epi;
    c.A = A;
    c.lda = lda ? lda : K;
    c.a_rows = M;
    c.B = W;
    c.ldb = K;
    c.M = M;
    c.N = N;
    c.K = K;
    c.out = out;
    c.ldc = ldc;
    c.ws = sc.ws;
    c.ws_floats = sc.floats;
    c.pdl = sc.pdl;
    c.bias = bias;
    c.res = res;
    c.ldr = ldr;
    run_gemm(c, st);
}

// ---------------------------------------------------------------------------
void Engine::prefill(const std::vector<std::string>& ids, const std::vector<std::vector<int>>& prompts) {
    Impl& m = *impl_;
    HC_CUDA(cudaSetDevice(opt_.device));
    m.require_configured();
    m.w_prefetched = false;  // the prefill streams weights through the same slots
    if (ids.size() != prompts.size()) throw InputError("prefill: ids and prompts differ in length");
    {
        std::unordered_set<std::string> seen;
        for (size_t r = 0; r < ids.size(); ++r) {
            if (cache_->has_request(ids[r]) || !seen.insert(ids[r]).second)
                throw InputError("duplicate request id: " + ids[r]);
            if (static_cast<int>(prompts[r].size()) > m.max_seq) throw InputError("embed: sequence longer than max_seq");
            for (int t : prompts[r])
                if (t < 0 || t >= m.V) throw InputError("embed: token id out of range: " + std::to_string(t));
        }
    }
    // Offloaded prefill pipeline (forward_prompt semantics per request,
    // decoder.cpp:144-157; one compute stage, sim.cpp:237-253):
    //   layer-outer / request-chunk-inner, so each layer's weights cross the
    //   host link once for the whole prefill (copy stream, double-buffered);
    //   host-located blocks are scattered into the device staging slot of
    //   the layer (indexed by pbn, the host pool's own layout) and leave on a
    //   store stream as pbn-contiguous D2H runs that overlap the next layer's
    //   compute (full duplex with the weight stream).
    // 1. bookkeeping, prompt tokens request by request (sim.cpp:222-223);
    //    all requests' rows laid end to end.
    struct Chunk {
        int row0 = 0, rows = 0, n = 0, max_len = 0;
        std::vector<int> cu, k_src, k_n, k_ref;
        size_t o_cu = 0, o_ks = 0, o_kn = 0, o_kr = 0;
    };
    std::vector<Chunk> chunks;
    std::vector<int> tokens, positions, a_src, a_n, a_ref, acth, kvh;
    long direct_act = 0, direct_kv = 0;  // host blocks written through mapped stores (mini-batched staging)
    try {  // none of ids existed before this call (checked above): on failure all are released again
    for (size_t r = 0; r < ids.size(); ++r) {
        const int P = static_cast<int>(prompts[r].size());
        if (chunks.empty() || (chunks.back().rows > 0 && chunks.back().rows + P > opt_.max_prefill_tokens)) {
            chunks.emplace_back();
            chunks.back().row0 = static_cast<int>(tokens.size());
            chunks.back().cu.push_back(0);
        }
        Chunk& c = chunks.back();
        assigner_->add_request(ids[r], P);
        const int base = static_cast<int>(tokens.size());
        const int rc = rc_prefix(P);
        if (token_mode_) rc_ids_[ids[r]].assign(prompts[r].begin(), prompts[r].begin() + rc);
        for (int t = 0; t < P; ++t) {
            tokens.push_back(prompts[r][t]);
            positions.push_back(t);
            if (t >= rc) assigner_->add_token(ids[r]);
        }
        int row = base + rc;
        for (const auto& e : cache_->table(ids[r]).entries) {
            const bool gpu = e.location == Location::GpuMem;
            if (e.kind == BlockKind::ACT) {
                if (gpu || m.owns(e.pbn)) {  // a host ACT block is written by its owning rank only
                    a_src.push_back(row);
                    a_n.push_back(e.filled_tokens);
                    if (gpu)
                        a_ref.push_back(pack_ref(R_ACT_GPU, e.pbn));
                    else if (m.mb_on) {  // staging smaller than the pool: straight into the mapped pool
                        a_ref.push_back(pack_ref(R_ACT_HOST, e.pbn / m.tpn));
                        direct_act += 1;
                    }
                    else
                        a_ref.push_back(pack_ref(R_ACT_STAGE, m.act_pos(e.pbn)));
                    if (!gpu && !m.mb_on) acth.push_back(e.pbn / m.tpn);
                }
            } else {
                c.k_src.push_back(row - c.row0);
                c.k_n.push_back(e.filled_tokens);
                c.k_ref.push_back(pack_ref(gpu ? R_KV_GPU : (m.mb_on ? R_KV_HOST : R_KV_STAGE), e.pbn));
                if (!gpu && m.mb_on) direct_kv += 1;
                if (!gpu && !m.mb_on) kvh.push_back(e.pbn);
            }
            row += e.filled_tokens;
        }
        c.rows += P;
        c.n += 1;
        c.cu.push_back(c.rows);
        c.max_len = std::max(c.max_len, P);
    }
    } catch (...) {  // pools exhausted part-way: the prefill admits every request or none
        for (const std::string& id : ids)
            if (cache_->has_request(id)) free_request(id);
        throw;
    }
    const int T = static_cast<int>(tokens.size());
    if (T == 0) return;
    int max_chunk = 0;
    for (const Chunk& c : chunks) max_chunk = std::max(max_chunk, c.rows);
    m.ensure_prefill(T, max_chunk);
    const std::vector<Run> act_runs = runs_of(acth), kv_runs = runs_of(kvh);
    const bool stores = !act_runs.empty() || !kv_runs.empty();

    std::vector<int> meta;
    auto put = [&](const std::vector<int>& v) {
        const size_t o = meta.size();
        meta.insert(meta.end(), v.begin(), v.end());
        return o;
    };
    const size_t o_tok = put(tokens), o_pos = put(positions), o_as = put(a_src), o_an = put(a_n), o_ar = put(a_ref);
    for (Chunk& c : chunks) {
        c.o_cu = put(c.cu);
        c.o_ks = put(c.k_src);
        c.o_kn = put(c.k_n);
        c.o_kr = put(c.k_ref);
    }
    m.ensure_meta(meta.size());
    std::memcpy(m.h_meta, meta.data(), meta.size() * 4);
    const int* dm = m.d_meta;

    StepStats st{};
    m.pev_used = 0;
    m.spans.clear();
    const float scale = opt_.scaled ? 1.0f / std::sqrt(static_cast<float>(m.hd)) : 1.0f;
    HC_CUDA(cudaEventRecord(m.ev0, s_compute_));
    HC_CUDA(cudaMemcpyAsync(m.d_meta, m.h_meta, meta.size() * 4, cudaMemcpyHostToDevice, s_compute_));
    embed(m.emb, m.pos, dm + o_tok, dm + o_pos, T, m.d, m.px[0], m.d, s_compute_);
    st.launches += 1;
    for (int l = 0; l < m.L; ++l) {
        const int slot = l & 1;
        m.cur_layer = l;
        if (!m.w_all) {
            HC_CUDA(cudaStreamWaitEvent(s_copy_, m.consumed[slot]));
            m.span_begin(profile_, s_copy_, 3);
            HC_CUDA(cudaMemcpyAsync(m.wbuf[slot], m.h_w + static_cast<size_t>(l % m.Lw) * m.LE, m.LE * 2,
                                    cudaMemcpyHostToDevice, s_copy_));
            m.span_end(profile_, s_copy_);
            st.h2d_bytes += m.LE * 2.0;
            st.h2d_weights += m.LE * 2.0;
            HC_CUDA(cudaEventRecord(m.loaded[slot], s_copy_));
            HC_CUDA(cudaStreamWaitEvent(s_compute_, m.loaded[slot]));
        }
        // the staging slot is free once layer l-2's stores have left
        if (stores && l >= 2) HC_CUDA(cudaStreamWaitEvent(s_compute_, m.stored[slot]));
        const f16* W = m.layer_w(l, slot);
        f16* R[16];
        m.regions(l, slot, R);
        f16* xin = m.px[l & 1];
        f16* xout = m.px[(l + 1) & 1];
        // the layer's GEMM input: x (reference arch) or LN1(x) (kArchOpt)
        const f16* xa = m.ln(W, 1, xin, T, m.pxn, s_compute_);
        st.launches += m.opt();
        // activation-cache writer: this layer's input rows of every ACT block
        BlockScatter sa;
        sa.src = xa;
        sa.ld = m.d;
        sa.src_row = dm + o_as;
        sa.n_tok = dm + o_an;
        sa.dst_ref = dm + o_ar;
        std::copy(R, R + 16, sa.region);
        sa.n_blocks = static_cast<int>(a_src.size());
        sa.d = m.d;
        sa.H = m.H;
        sa.hd = m.hd;
        sa.tpb = m.tpb;
        scatter_act_blocks(sa, s_compute_);
        st.launches += sa.n_blocks > 0;
        for (const Chunk& c : chunks) {
            const f16* cin = xin + static_cast<size_t>(c.row0) * m.d;
            f16* cout = xout + static_cast<size_t>(c.row0) * m.d;
            m.span_begin(profile_, s_compute_, 2);
            m.qkv(W, xa + static_cast<size_t>(c.row0) * m.d, c.rows, m.pqkv, s_compute_);
            m.span_end(profile_, s_compute_);
            BlockScatter sk = sa;
            sk.src = m.pqkv;
            sk.ld = 3 * m.dg;
            sk.d = m.dg;
            sk.H = m.Hg;
            sk.src_row = dm + c.o_ks;
            sk.n_tok = dm + c.o_kn;
            sk.dst_ref = dm + c.o_kr;
            sk.n_blocks = static_cast<int>(c.k_src.size());
            scatter_kv_blocks(sk, s_compute_);
            m.span_begin(profile_, s_compute_, 1);
            prefill_attention(m.pqkv, m.patt, dm + c.o_cu, c.n, c.max_len, m.Hg, m.hd, scale, s_compute_, c.rows);
            m.span_end(profile_, s_compute_);
            m.span_begin(profile_, s_compute_, 2);
            m.tail(W, m.patt, cin, c.rows, m.pproj, m.patt, m.ph, cout, s_compute_);
            m.span_end(profile_, s_compute_);
            st.launches += 2 + m.tail_launches() + (sk.n_blocks > 0);
        }
        HC_CUDA(cudaEventRecord(m.consumed[slot], s_compute_));
        if (stores) {  // this layer's host blocks: staging slot -> pinned pool (copy engine, D2H)
            HC_CUDA(cudaStreamWaitEvent(s_store_, m.consumed[slot]));
            m.span_begin(profile_, s_store_, 4);
            const size_t lp = static_cast<size_t>(l % m.Lp);
            const f16* own = m.act_stage[slot] + static_cast<size_t>(m.tpr) * m.act_cap_n * m.actb;
            for (const Run& r : act_runs) {
                const size_t bytes = static_cast<size_t>(r.count) * m.actb * 2;
                HC_CUDA(cudaMemcpyAsync(m.act_host + (lp * m.act_cap_n + r.start) * m.actb,
                                        own + static_cast<size_t>(r.start) * m.actb, bytes, cudaMemcpyDeviceToHost,
                                        s_store_));
                st.d2h_bytes += bytes;
                st.d2h_act += bytes;
            }
            for (const Run& r : kv_runs) {
                const size_t bytes = static_cast<size_t>(r.count) * m.kvb * 2;
                HC_CUDA(cudaMemcpyAsync(m.kv_host + (lp * m.kv_host_cap + r.start) * m.kvb,
                                        m.kv_stage[slot] + static_cast<size_t>(r.start) * m.kvb, bytes,
                                        cudaMemcpyDeviceToHost, s_store_));
                st.d2h_bytes += bytes;
                st.d2h_kv += bytes;
            }
            m.span_end(profile_, s_store_);
            HC_CUDA(cudaEventRecord(m.stored[slot], s_store_));
        }
    }
    if (stores) {
        HC_CUDA(cudaStreamWaitEvent(s_compute_, m.stored[0]));
        HC_CUDA(cudaStreamWaitEvent(s_compute_, m.stored[1]));
    }
    HC_CUDA(cudaEventRecord(m.ev1, s_compute_));
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    float ms = 0;
    HC_CUDA(cudaEventElapsedTime(&ms, m.ev0, m.ev1));
    st.step_ms = ms;
    st.d2h_act += static_cast<double>(direct_act) * m.actb * 2 * m.L;
    st.d2h_kv += static_cast<double>(direct_kv) * m.kvb * 2 * m.L;
    st.d2h_bytes += static_cast<double>(direct_act) * m.actb * 2 * m.L + static_cast<double>(direct_kv) * m.kvb * 2 * m.L;
    for (const auto& sp : m.spans) {
        float t = 0;
        HC_CUDA(cudaEventElapsedTime(&t, sp.a, sp.b));
        if (sp.kind == 1)
            st.attn_ms += t;
        else if (sp.kind == 2)
            st.gemm_ms += t;
        else if (sp.kind == 3)
            st.copy_ms += t;
        else if (sp.kind == 4)
            st.store_ms += t;
    }
    stats_ = st;
}

void Engine::admit_synthetic(const std::vector<std::string>& ids, const std::vector<int>& prompt_lens, uint64_t seed) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    m.require_configured();
    if (ids.size() != prompt_lens.size()) throw InputError("admit_synthetic: ids and lengths differ");
    for (size_t r = 0; r < ids.size(); ++r) {
        if (prompt_lens[r] > m.max_seq) throw InputError("embed: sequence longer than max_seq");
        assigner_->add_request(ids[r], prompt_lens[r]);
        const int rc = rc_prefix(prompt_lens[r]);
        if (token_mode_) {
            std::vector<int>& v = rc_ids_[ids[r]];
            v.resize(rc);
            for (int t = 0; t < rc; ++t) v[t] = static_cast<int>((seed + 7919u * (t + 1) + 31u * r) % m.V);
        }
        for (int t = rc; t < prompt_lens[r]; ++t) assigner_->add_token(ids[r]);
    }
    if (!m.pools_filled) fill_pools(seed);
}

void Engine::fill_pools(uint64_t seed) {
    HC_CUDA(cudaSetDevice(opt_.device));
    Impl& m = *impl_;
    m.require_configured();
    // activations ~U(-0.1,0.1) like the embeddings; K,V of matching scale
    auto fill = [&](f16* p, size_t n, uint64_t s) {
        if (p && n) fill_pattern(p, n, s, 0.1f, s_compute_);
    };
    fill(m.kv_gpu, static_cast<size_t>(m.L) * m.kv_gpu_cap * m.kvb, seed + 1);
    fill(m.act_gpu, static_cast<size_t>(m.L) * m.act_gpu_cap * m.actb, seed + 2);
    fill(m.kv_host, static_cast<size_t>(m.Lp) * m.kv_host_cap * m.kvb, seed + 3);
    fill(m.act_host, static_cast<size_t>(m.Lp) * m.act_cap_n * m.actb, seed + 4);
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    m.pools_filled = true;
}

void Engine::advance_synthetic(const std::vector<std::string>& ids, int n_tokens) {
    Impl& m = *impl_;
    m.require_configured();
    if (n_tokens < 0) throw InputError("advance_synthetic: negative token count");
    for (const std::string& id : ids)
        if (cache_->table(id).context_len() + recompute_prefix_len(id) + n_tokens > m.max_seq)
            throw InputError("embed: sequence longer than max_seq");
    // decode order: one token per request per iteration (sim.cpp:308-310), so
    // the block tables are the ones n_tokens real decode steps would leave
    for (int t = 0; t < n_tokens; ++t)
        for (const std::string& id : ids) assigner_->add_token(id);
}

void Engine::free_request(const std::string& id) {
    cache_->free_request(id);
    rc_ids_.erase(id);
}

int Engine::rc_prefix(int prompt_len) const {
    if (!token_mode_) return 0;
    const int tpb = cfg_.tokens_per_block;
    return static_cast<int>(std::floor(opt_.recompute_ratio * prompt_len / tpb)) * tpb;
}

long Engine::recompute_prefix_len(const std::string& id) const {
    auto it = rc_ids_.find(id);
    return it == rc_ids_.end() ? 0 : static_cast<long>(it->second.size());
}

// ---------------------------------------------------------------------------
void Engine::decode_step(const std::vector<std::string>& ids_in, const int* tokens_in, uint16_t* x_out,
                         float* logits_out, int* argmax_out) {
    Impl& m = *impl_;
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may differ from the constructing one
    m.require_configured();
    const int n = static_cast<int>(ids_in.size());
    // ranks sharing one weight stream run the same collective sequence every
    // step, so validation failures are agreed on before the first all-gather
    // and an empty batch still streams (and gathers) every layer
    std::string local_error;
    std::vector<int> pos_in(n);
    try {
        if (n > m.B) throw InputError("decode_step: batch larger than max_batch");
        std::unordered_set<std::string> seen;
        for (int b = 0; b < n; ++b) {
            if (!seen.insert(ids_in[b]).second) throw InputError("decode_step: duplicate request id " + ids_in[b]);
            if (tokens_in[b] < 0 || tokens_in[b] >= m.V)
                throw InputError("embed: token id out of range: " + std::to_string(tokens_in[b]));
            pos_in[b] = cache_->table(ids_in[b]).context_len() + static_cast<int>(recompute_prefix_len(ids_in[b]));
            if (pos_in[b] >= m.max_seq)
                throw InputError("embed: position exceeds max_seq: " + std::to_string(pos_in[b]));
        }
        if (n) assigner_->check_batch_capacity(ids_in);  // all contexts grow, or none (no half-applied step)
    } catch (const std::exception& e) {
        if (m.wsn == 1) throw;
        local_error = e.what();
    }
    if (m.wsn > 1) {
        m.agree_or_throw(local_error, s_compute_);
    } else if (n == 0) {
        return;
    }

    // ---- mini-batches (paper §4.3.3; sim.cpp:258-275): requests packed by
    // form_minibatches (minibatch.cpp:36-83) on their PRE-growth block counts
    // into units whose blocks fit one staging slot; a step is then the
    // (layer, mini-batch) units of sim.cpp:324-358, double-buffered
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<int> mb_row{0};
    if (m.mb_on && n > 0) {
        std::vector<RequestBlocks> reqs;
        std::unordered_map<std::string, int> idx;
        for (int b = 0; b < n; ++b) {
            const auto ak = cache_->table(ids_in[b]).blocks_by_kind();
            reqs.push_back(RequestBlocks{ids_in[b], ak.first, ak.second});
            idx[ids_in[b]] = b;
        }
        std::vector<MiniBatch> mbs;
        try {
            mbs = form_minibatches(reqs, m.packer, m.packer_bundle, m.tpb);
        } catch (const InputError& e) {
            throw CapacityError(std::string("decode_step: request too large for the staging buffers: ") + e.what());
        }
        order.clear();
        for (const MiniBatch& mb : mbs) {
            for (const std::string& id : mb.ids) order.push_back(idx.at(id));
            mb_row.push_back(static_cast<int>(order.size()));
        }
    } else {
        mb_row.push_back(n);
    }
    const int M = static_cast<int>(mb_row.size()) - 1;
    const bool permuted = M > 1;
    // rows of the step in mini-batch order
    std::vector<std::string> ids(n);
    std::vector<int> tokv(n), pos(n);
    for (int i = 0; i < n; ++i) {
        ids[i] = ids_in[order[i]];
        tokv[i] = tokens_in[order[i]];
        pos[i] = pos_in[order[i]];
    }

    // token-recompute prefixes: rows of a batched causal forward rebuilt
    // through every layer each step (the FlexGen-style baseline, sim.cpp:196-206)
    std::vector<int> rc_tok, rc_pos, rc_cu(1, 0), tr_src, tr_n, tr_ref;
    int rc_max = 0;
    if (token_mode_) m.ensure_tr();
    for (int b = 0; b < n; ++b) {
        const std::vector<int>* pre = nullptr;
        if (token_mode_) {
            auto it = rc_ids_.find(ids[b]);
            if (it != rc_ids_.end()) pre = &it->second;
        }
        const int rc = pre ? static_cast<int>(pre->size()) : 0;
        for (int t = 0; t < rc; ++t) {
            rc_tok.push_back((*pre)[t]);
            rc_pos.push_back(t);
        }
        for (int i = 0; i < rc / m.tpb; ++i) {
            tr_src.push_back(rc_cu.back() + i * m.tpb);
            tr_n.push_back(m.tpb);
            tr_ref.push_back(pack_ref(R_TOKREC, b * m.max_blocks + i));
        }
        rc_cu.push_back(rc_cu.back() + rc);
        rc_max = std::max(rc_max, rc);
    }
    const int n_rc = rc_cu.back();
    if (n_rc) m.ensure_prefill(n_rc);

    // grow every context by this step's token, in mini-batch order (the
    // reference's add_token order, sim.cpp:294-310)
    std::vector<TokenSlot> grown;
    grown.reserve(n);
    for (int b = 0; b < n; ++b) grown.push_back(assigner_->add_token(ids[b]));

    // per mini-batch: the host blocks it stages (staging position = the host
    // pool's own pbn layout for a whole-batch step; packed in pbn order for a
    // mini-batch, so pbn runs stay contiguous DMA runs), recompute tiles and
    // copy runs
    struct Unit {
        std::vector<Run> kv_runs, act_runs;  // start = host index, dst = staging position
        std::vector<int> tiles_h, tiles_g;
        // fused recompute: per (tile, block slot) request << 8 | valid tokens, -1 = not in the unit
        std::vector<int> info_h, info_g;
        int splits = 1;
        bool any_act = false, any_kv = false;
        bool records_only = false;  // fused and every context block recomputed: the records-only attention
        size_t o_th = 0, o_tg = 0, o_ih = 0, o_ig = 0;
    };
    std::vector<Unit> units(M);
    std::vector<int> act_dev(n, -1), act_host(n, -1), kv_dev(n, -1), kv_host(n, -1), tok(n, 0), nblk(n), ctx(n);
    std::vector<int> refs(static_cast<size_t>(n) * m.max_blocks, 0);
    bool gather_act = false;
    long stage_kv_need = 0, stage_act_need = 0;
    for (int u = 0; u < M; ++u) {
        Unit& U = units[u];
        std::vector<int> kvh, acth, actg;
        for (int b = mb_row[u]; b < mb_row[u + 1]; ++b)
            for (const auto& en : cache_->table(ids[b]).entries) {
                if (en.location == Location::GpuMem) {
                    if (en.kind == BlockKind::ACT) actg.push_back(en.pbn);
                } else {
                    (en.kind == BlockKind::KV ? kvh : acth).push_back(en.pbn);
                }
            }
        for (auto* v : {&kvh, &acth}) {
            std::sort(v->begin(), v->end());
            v->erase(std::unique(v->begin(), v->end()), v->end());
        }
        std::unordered_map<int, int> kvp, actp;  // pbn -> staging position
        for (size_t i = 0; i < kvh.size(); ++i) kvp[kvh[i]] = permuted ? static_cast<int>(i) : kvh[i];
        std::vector<int> apos;
        for (size_t i = 0; i < acth.size(); ++i) {
            const int p = permuted ? static_cast<int>(i) : m.act_pos(acth[i]);
            actp[acth[i]] = p;
            apos.push_back(p);
        }
        stage_kv_need = std::max(stage_kv_need, kvh.empty() ? 0L : static_cast<long>(kvp[kvh.back()]) + 1);
        stage_act_need = std::max(stage_act_need, static_cast<long>(acth.size()));
        for (const Run& r : runs_of(kvh)) U.kv_runs.push_back({r.start, r.count, kvp[r.start]});
        std::vector<int> own;  // host indices of the ACT blocks this rank streams
        for (int p : acth)
            if (m.owns(p)) own.push_back(p);
        for (const Run& r : runs_of(own))  // (tpn > 1: own pbns are g, g+N, ...; host index pbn / N)
            U.act_runs.push_back({r.start / m.tpn, r.count, actp[r.start]});
        if (m.tpn > 1) {
            U.act_runs.clear();
            std::vector<int> hidx;
            for (int p : own) hidx.push_back(p / m.tpn);
            for (const Run& r : runs_of(hidx))
                U.act_runs.push_back({r.start, r.count, static_cast<int>(m.tpr * m.act_cap_n) + r.start});
            gather_act = !acth.empty();
        }
        U.tiles_h = tiles_of(apos, m.tpb);
        U.tiles_g = tiles_of(actg, m.tpb);
        int max_ctx = 0;
        std::unordered_map<int, int> binfo_h, binfo_g;  // fused: block position -> request << 8 | valid
        U.records_only = m.fused;
        for (int b = mb_row[u]; b < mb_row[u + 1]; ++b) {
            const int rcb = (rc_cu[b + 1] - rc_cu[b]) / m.tpb;
            const BlockTableEntry& e = grown[b].entry;
            const bool gpu = e.location == Location::GpuMem;
            tok[b] = grown[b].token_index;
            if (e.kind == BlockKind::ACT) {
                U.any_act = true;
                act_dev[b] = pack_ref(gpu ? R_ACT_GPU : R_ACT_STAGE, gpu ? e.pbn : actp.at(e.pbn));
                if (!gpu && m.owns(e.pbn)) act_host[b] = pack_ref(R_ACT_HOST, e.pbn / m.tpn);
            } else {
                U.any_kv = true;
                kv_dev[b] = pack_ref(gpu ? R_KV_GPU : R_KV_STAGE, gpu ? e.pbn : kvp.at(e.pbn));
                if (!gpu) kv_host[b] = pack_ref(R_KV_HOST, e.pbn);
            }
            const BlockTable& t = cache_->table(ids[b]);
            nblk[b] = rcb + static_cast<int>(t.entries.size());
            ctx[b] = rcb * m.tpb + t.context_len();
            max_ctx = std::max(max_ctx, ctx[b]);
            int* rb = refs.data() + static_cast<size_t>(b) * m.max_blocks;
            if (rcb > 0) U.records_only = false;
            for (int i = 0; i < rcb; ++i) *rb++ = pack_ref(R_TOKREC, b * m.max_blocks + i);
            for (size_t i = 0; i < t.entries.size(); ++i) {
                const auto& en = t.entries[i];
                const bool g = en.location == Location::GpuMem;
                if (en.kind == BlockKind::KV) {
                    U.records_only = false;
                    rb[i] = g ? pack_ref(R_KV_GPU, en.pbn) : pack_ref(R_KV_STAGE, kvp.at(en.pbn));
                } else {
                    const int pos = g ? en.pbn : actp.at(en.pbn);
                    rb[i] = pack_ref(R_KVR, g ? pos : static_cast<int>(m.act_gpu_cap) + pos);
                    if (m.fused) {
                        const int valid = std::min(m.tpb, static_cast<int>(t.context_len() - static_cast<long>(i) * m.tpb));
                        if (!(g ? binfo_g : binfo_h).emplace(pos, b << 8 | valid).second)
                            throw std::logic_error("decode_step: an ACT block is listed by two requests");
                    }
                }
            }
        }
        if (m.fused) {  // per (tile, block slot) of the recompute tiles
            const int bpt = gemm::BM / m.tpb;
            for (int which = 0; which < 2; ++which) {
                const std::vector<int>& tl = which == 0 ? U.tiles_h : U.tiles_g;
                const auto& mp = which == 0 ? binfo_h : binfo_g;
                std::vector<int>& info = which == 0 ? U.info_h : U.info_g;
                info.assign(tl.size() * bpt, -1);
                for (size_t ti = 0; ti < tl.size(); ++ti)
                    for (int k = 0; k < bpt; ++k) {
                        const auto it = mp.find(tl[ti] / m.tpb + k);
                        if (it != mp.end()) info[ti * bpt + k] = it->second;
                    }
            }
        }
        U.splits = attention_splits(mb_row[u + 1] - mb_row[u], m.Hg, max_ctx, m.tpb);
        if (U.splits > 1)
            m.ensure_attn_work(static_cast<size_t>(mb_row[u + 1] - mb_row[u]) * m.Hg * U.splits * (m.hd + 2));
    }
    if (stage_kv_need > m.stage_kv_cap || stage_act_need > m.stage_act_cap)
        throw CapacityError("decode_step: a mini-batch's blocks exceed the staging buffers");

    // one upload of all step metadata
    std::vector<int> meta;
    auto put = [&](const std::vector<int>& v) {
        const size_t o = meta.size();
        meta.insert(meta.end(), v.begin(), v.end());
        return o;
    };
    const size_t o_tok = put(tokv), o_pos = put(pos), o_ad = put(act_dev), o_ah = put(act_host), o_kd = put(kv_dev),
                 o_kh = put(kv_host), o_t = put(tok), o_nb = put(nblk), o_ctx = put(ctx), o_ref = put(refs),
                 o_rtok = put(rc_tok), o_rpos = put(rc_pos), o_rcu = put(rc_cu), o_trs = put(tr_src),
                 o_trn = put(tr_n), o_trr = put(tr_ref);
    for (Unit& U : units) {
        U.o_th = put(U.tiles_h);
        U.o_tg = put(U.tiles_g);
        U.o_ih = put(U.info_h);
        U.o_ig = put(U.info_g);
    }
    m.ensure_meta(meta.size() + 1);
    if (!meta.empty()) std::memcpy(m.h_meta, meta.data(), meta.size() * 4);
    const int* dm = m.d_meta;

    StepStats st{};
    m.pev_used = 0;
    m.spans.clear();
    bool stream_any = !m.w_all;
    for (const Unit& U : units) stream_any = stream_any || !U.kv_runs.empty() || !U.act_runs.empty();
    stream_any = stream_any || gather_act;
    // layers 0/1 weights already in their slots (prefetched at the end of the
    // previous step; never with a shared weight stream, whose ranks must issue
    // the same gathers every step)
    const bool prefetched = m.w_prefetched && !m.w_all && m.wsn == 1;
    m.w_prefetched = false;
    bool capturing = false;  // enqueue() runs under stream capture (graph mode)
    // one layer's weights into wbuf[slot] on the copy stream; with a shared
    // weight stream only this rank's slice crosses its host link and an
    // in-place all-gather on the gather stream (NVLink) completes the layer
    // while the copy stream moves on to the layer's KV / ACT blocks
    auto stream_weights = [&](int l, int slot, StepStats& st) {
        const uint16_t* src = m.h_w + static_cast<size_t>(l % m.Lw) * m.LE;
        if (m.wsn == 1) {
            HC_CUDA(cudaMemcpyAsync(m.wbuf[slot], src, m.LE * 2, cudaMemcpyHostToDevice, s_copy_));
            st.h2d_bytes += m.LE * 2.0;
            st.h2d_weights += m.LE * 2.0;
            return;
        }
        const size_t s0 = static_cast<size_t>(m.wsr) * m.wsS;
        const size_t cnt = s0 < m.LE ? std::min(m.wsS, m.LE - s0) : 0;
        if (cnt)
            HC_CUDA(cudaMemcpyAsync(m.wbuf[slot] + s0, src + s0, cnt * 2, cudaMemcpyHostToDevice, s_copy_));
        st.h2d_bytes += cnt * 2.0;
        st.h2d_weights += cnt * 2.0;
        HC_CUDA(cudaEventRecord(m.w_h2d[slot], s_copy_));
        HC_CUDA(cudaStreamWaitEvent(s_gather_, m.w_h2d[slot]));
        m.ws->copy_channel()->all_gather(m.wbuf[slot] + s0, m.wbuf[slot], m.wsS, s_gather_);
        HC_CUDA(cudaEventRecord(m.w_gath[slot], s_gather_));
        HC_CUDA(cudaStreamWaitEvent(s_compute_, m.w_gath[slot]));
    };
    // everything the step puts on the streams; outputs land in xo / lo / ao
    auto enqueue = [&](StepStats& st, uint16_t* xo, float* lo, int* ao) {
        HC_CUDA(cudaEventRecord(m.ev0, s_compute_));
        if (!meta.empty())
            HC_CUDA(cudaMemcpyAsync(m.d_meta, m.h_meta, meta.size() * 4, cudaMemcpyHostToDevice, s_compute_));
        if (n) {
            embed(m.emb, m.pos, dm + o_tok, dm + o_pos, n, m.d, m.x[0], m.d, s_compute_);
            st.launches += 1;
        }
        if (n_rc) {
            embed(m.emb, m.pos, dm + o_rtok, dm + o_rpos, n_rc, m.d, m.px[0], m.d, s_compute_);
            st.launches += 1;
        }
        if (capture_inputs_) captured_.assign(static_cast<size_t>(m.L) * n * m.d, 0);
        const float scale = opt_.scaled ? 1.0f / std::sqrt(static_cast<float>(m.hd)) : 1.0f;

        for (int l = 0; l < m.L; ++l) {
            const int wslot = l & 1;
            m.cur_layer = l;
            const f16* W = m.layer_w(l, wslot);
            for (int u = 0; u < M; ++u) {
                const Unit& U = units[u];
                const int j = l * M + u;  // unit index: staging slot j % 2 (sim.cpp:372-377)
                m.cur_mb = u;
                const int slot = j & 1;
                const int r0 = mb_row[u], nb = mb_row[u + 1] - r0;
                if (stream_any) {
                    // copy stream: weights (first unit of the layer, once the layer
                    // two back released wbuf[l%2]) then this unit's host blocks
                    // into staging slot j%2 once unit j-2 released it; the first
                    // two of the step wait for the step start only, so a captured
                    // graph waits on events it records itself
                    m.span_begin(profile_, s_copy_, 3);
                    if (u == 0 && !m.w_all && !(prefetched && l < 2)) {  // layers 0/1 may have come with the previous step
                        HC_CUDA(cudaStreamWaitEvent(s_copy_, l >= 2 ? m.w_consumed[wslot] : m.ev0));
                        stream_weights(l, wslot, st);
                    }
                    HC_CUDA(cudaStreamWaitEvent(s_copy_, j >= 2 ? m.consumed[slot] : m.ev0));
                    const size_t lp = static_cast<size_t>(l % m.Lp);
                    for (const Run& r : U.act_runs) {
                        const size_t bytes = static_cast<size_t>(r.count) * m.actb * 2;
                        HC_CUDA(cudaMemcpyAsync(m.act_stage[slot] + static_cast<size_t>(r.dst) * m.actb,
                                                m.act_host + (lp * m.act_cap_n + r.start) * m.actb, bytes,
                                                cudaMemcpyHostToDevice, s_copy_));
                        st.h2d_bytes += bytes;
                        st.h2d_act += bytes;
                    }
                    // every rank streamed its 1/tpn of the ACT blocks; an NVLink all-gather
                    // on the gather stream completes the staging (the recompute needs all
                    // of X for its heads) while the copy stream moves on to the KV blocks
                    // and the next layer
                    if (gather_act) {
                        f16* own = m.act_stage[slot] + static_cast<size_t>(m.tpr) * m.act_cap_n * m.actb;
                        HC_CUDA(cudaEventRecord(m.h2d_act[slot], s_copy_));
                        HC_CUDA(cudaStreamWaitEvent(s_gather_, m.h2d_act[slot]));
                        m.tp->copy_channel()->all_gather(own, m.act_stage[slot], m.act_cap_n * m.actb, s_gather_);
                        HC_CUDA(cudaEventRecord(m.gathered[slot], s_gather_));
                        HC_CUDA(cudaStreamWaitEvent(s_compute_, m.gathered[slot]));
                    }
                    for (const Run& r : U.kv_runs) {
                        const size_t bytes = static_cast<size_t>(r.count) * m.kvb * 2;
                        HC_CUDA(cudaMemcpyAsync(m.kv_stage[slot] + static_cast<size_t>(r.dst) * m.kvb,
                                                m.kv_host + (lp * m.kv_host_cap + r.start) * m.kvb, bytes,
                                                cudaMemcpyHostToDevice, s_copy_));
                        st.h2d_bytes += bytes;
                        st.h2d_kv += bytes;
                    }
                    m.span_end(profile_, s_copy_);
                    HC_CUDA(cudaEventRecord(m.loaded[slot], s_copy_));
                    HC_CUDA(cudaStreamWaitEvent(s_compute_, m.loaded[slot]));
                }
                f16* R[16];
                m.regions(l, slot, R);
                f16* xin = m.x[l & 1];
                f16* xout = m.x[(l + 1) & 1];
                if (n_rc && u == 0) {
                    // token recompute: full layer l over every prefix (FullLayer(rc) FLOPs,
                    // flops.cpp:20-22), its K|V written into the prefix blocks
                    m.span_begin(profile_, s_compute_, 0);
                    f16* pin = m.px[l & 1];
                    f16* pout = m.px[(l + 1) & 1];
                    m.qkv(W, m.ln(W, 1, pin, n_rc, m.pxn, s_compute_), n_rc, m.pqkv, s_compute_);
                    st.launches += m.opt();
                    BlockScatter sk;
                    sk.src = m.pqkv;
                    sk.ld = 3 * m.d;
                    sk.src_row = dm + o_trs;
                    sk.n_tok = dm + o_trn;
                    sk.dst_ref = dm + o_trr;
                    std::copy(R, R + 16, sk.region);
                    sk.n_blocks = static_cast<int>(tr_src.size());
                    sk.d = m.d;
                    sk.H = m.H;
                    sk.hd = m.hd;
                    sk.tpb = m.tpb;
                    scatter_kv_blocks(sk, s_compute_);
                    if (l + 1 < m.L) {  // the last layer's prefix output is never needed
                        prefill_attention(m.pqkv, m.patt, dm + o_rcu, n, rc_max, m.H, m.hd, scale, s_compute_, n_rc);
                        m.tail(W, m.patt, pin, n_rc, m.pproj, m.patt, m.ph, pout, s_compute_);
                        st.launches += 1 + m.tail_launches();
                    }
                    st.launches += 2;
                    st.recompute_tokens += n_rc;
                    m.span_end(profile_, s_compute_);
                }
                if (capture_inputs_ && u == 0)
                    HC_CUDA(cudaMemcpyAsync(captured_.data() + static_cast<size_t>(l) * n * m.d, xin,
                                            static_cast<size_t>(n) * m.d * 2, cudaMemcpyDeviceToHost, s_compute_));
                if (nb > 0) {
                    const size_t rd = static_cast<size_t>(r0) * m.d;
                    // the layer's GEMM input (and ACT payload): x, or LN1(x) for kArchOpt
                    const f16* xa = m.ln(W, 1, xin + rd, nb, m.xn + (m.xn ? rd : 0), s_compute_);
                    st.launches += m.opt();
                    AppendCall ap;
                    std::copy(R, R + 16, ap.region);
                    ap.B = nb;
                    ap.d = m.d;  // ACT rows are full width; K|V slots below are this rank's heads
                    ap.H = m.H;
                    ap.hd = m.hd;
                    ap.tpb = m.tpb;
                    ap.tok = dm + o_t + r0;
                    if (U.any_act) {  // ACT writer: X of the new token -> its ACT slot (device + host)
                        ap.src = xa;
                        ap.ld = m.d;
                        ap.dev_ref = dm + o_ad + r0;
                        ap.host_ref = dm + o_ah + r0;
                        act_append(ap, s_compute_);
                        st.launches += 1;
                    }
                    // recompute K|V of the unit's ACT blocks (streamed and resident): into
                    // R_KVR (kKvPaged), or fused with the attention (kAttnPart: partial
                    // records against the unit's queries, so the QKV GEMM runs first)
                    f16* qkvb = m.qkvb + static_cast<size_t>(r0) * 3 * m.dg;
                    f16* att = m.att + static_cast<size_t>(r0) * m.dg;
                    auto recompute = [&] {
                        for (int which = 0; which < 2; ++which) {
                            const std::vector<int>& tl = which == 0 ? U.tiles_h : U.tiles_g;
                            if (tl.empty()) continue;
                            GemmCall c;
                            c.epi = m.fused ? gemm::kAttnPart : gemm::kKvPaged;
                            c.A = which == 0 ? m.act_stage[slot] : R[R_ACT_GPU];
                            c.lda = m.d;
                            c.a_rows = static_cast<int>((which == 0 ? m.stage_act_cap : m.act_gpu_cap) * m.tpb);
                            c.B = W + m.off.wqkv + static_cast<size_t>(m.dg) * m.d;  // rows dg..3dg of Wqkv^T = [Wk|Wv]^T (own heads)
                            c.ldb = m.d;
                            c.M = c.a_rows;
                            c.N = 2 * m.dg;
                            c.K = m.d;
                            c.m_tile_rows = dm + (which == 0 ? U.o_th : U.o_tg);
                            c.num_m_tiles = static_cast<int>(tl.size());
                            c.out = m.kvr;
                            c.tpb = m.tpb;
                            c.d = m.dg;
                            c.hd = m.hd;
                            c.blk_off = which == 0 ? static_cast<int>(m.act_gpu_cap) : 0;
                            c.bias = m.bias(W, m.off.bqkv + m.dg);  // [b_k | b_v] of the own heads
                            if (m.fused) {
                                c.blk_info = dm + (which == 0 ? U.o_ih : U.o_ig);
                                c.q = m.qkvb;  // request rows of the step (own heads' Q at column 0)
                                c.ldq = 3 * m.dg;
                                c.qscale = scale * 1.4426950408889634f;
                                c.part = m.part;
                            }
                            m.span_begin(profile_, s_compute_, 0);
                            run_gemm(c, s_compute_);
                            m.span_end(profile_, s_compute_);
                            st.launches += 1;
                            st.recompute_tokens += static_cast<double>(tl.size()) * gemm::BM;
                        }
                    };
                    if (!m.fused) recompute();
                    m.span_begin(profile_, s_compute_, 2);
                    // every new token of the unit goes to an ACT block: the fused recompute
                    // produces its K|V from the appended X row, QKV needs only Q
                    m.qkv(W, xa, nb, qkvb, s_compute_, m.scratch(), m.fused && !U.any_kv && U.any_act);
                    m.span_end(profile_, s_compute_);
                    if (m.fused) recompute();
                    if (U.any_kv) {  // new token's K|V -> its KV slot (device + host)
                        ap.src = qkvb;
                        ap.ld = 3 * m.dg;
                        ap.d = m.dg;
                        ap.H = m.Hg;
                        ap.dev_ref = dm + o_kd + r0;
                        ap.host_ref = dm + o_kh + r0;
                        kv_append(ap, s_compute_);
                        st.launches += 1;
                    }
                    AttnCall a;
                    a.q = qkvb;
                    a.ldq = 3 * m.dg;
                    a.out = att;
                    a.blk_ref = dm + o_ref + static_cast<size_t>(r0) * m.max_blocks;
                    a.n_blocks = dm + o_nb + r0;
                    a.ctx_len = dm + o_ctx + r0;
                    a.max_blocks = m.max_blocks;
                    for (int i = 0; i < 16; ++i) a.region[i] = R[i];
                    a.B = nb;
                    a.H = m.Hg;
                    a.hd = m.hd;
                    a.tpb = m.tpb;
                    a.scale = scale;
                    a.work = m.attn_work;
                    a.splits = U.splits;
                    if (m.fused) {
                        a.part = m.part;
                        a.part_region = R_KVR;
                        a.records_only = U.records_only ? 1 : 0;
                    }
                    m.span_begin(profile_, s_compute_, 1);
                    decode_attention(a, s_compute_);
                    m.span_end(profile_, s_compute_);
                    m.span_begin(profile_, s_compute_, 2);
                    m.tail(W, att, xin + rd, nb, m.proj + rd, att, m.hbuf + static_cast<size_t>(r0) * m.fg,
                           xout + rd, s_compute_, m.scratch(!profile_));
                    m.span_end(profile_, s_compute_);
                    st.launches += 1 + m.tail_launches() + (U.splits > 1 ? 2 : 1);
                }
                // events the next step / prefill waits on from outside the graph: the
                // last two units' staging slots and the last two layers' weight slots
                const bool external = capturing && l >= m.L - 2;
                if (capturing && j >= m.L * M - 2)
                    HC_CUDA(cudaEventRecordWithFlags(m.consumed[slot], s_compute_, cudaEventRecordExternal));
                else
                    HC_CUDA(cudaEventRecord(m.consumed[slot], s_compute_));
                if (u == M - 1) {
                    if (external)
                        HC_CUDA(cudaEventRecordWithFlags(m.w_consumed[wslot], s_compute_, cudaEventRecordExternal));
                    else
                        HC_CUDA(cudaEventRecord(m.w_consumed[wslot], s_compute_));
                }
            }
        }
        const f16* xf = n ? m.final_norm(m.x[m.L & 1], n, m.xn, s_compute_) : m.x[m.L & 1];
        st.launches += n ? m.opt() : 0;
        if ((lo || ao) && n) {
            gemm_rows(gemm::kF32, xf, n, m.d, m.emb, m.V, m.logits, m.V, s_compute_, 0, m.scratch());
            st.launches += 1;
            if (ao) {
                argmax_rows(m.logits, n, m.V, m.amax, s_compute_);
                st.launches += 1;
            }
        }
        HC_CUDA(cudaEventRecord(m.ev1, s_compute_));
        HC_CUDA(cudaGetLastError());
        if (xo && n)
            HC_CUDA(cudaMemcpyAsync(xo, xf, static_cast<size_t>(n) * m.d * 2, cudaMemcpyDeviceToHost, s_compute_));
        if (lo && n)
            HC_CUDA(cudaMemcpyAsync(lo, m.logits, static_cast<size_t>(n) * m.V * 4, cudaMemcpyDeviceToHost, s_compute_));
        if (ao && n) HC_CUDA(cudaMemcpyAsync(ao, m.amax, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, s_compute_));
    };

    // outputs of a permuted (mini-batched) step land in the pinned staging
    // buffers and are put back in the caller's order on the host
    auto ensure_host_out = [&] {
        if (!m.h_x) {
            m.h_x = halloc<uint16_t>(static_cast<size_t>(m.B) * m.d, false);
            m.h_logits = halloc<float>(static_cast<size_t>(m.B) * m.V, false);
            m.h_amax = halloc<int>(m.B, false);
        }
    };
    // CUDA graph of the step: its launch structure (sizes, copy runs, splits,
    // outputs) is the key; the data rides in the metadata block
    const bool use_graph = graphs_ && !profile_ && !capture_inputs_ && m.tpn == 1 && m.wsn == 1 && n > 0;
    const bool via_host = use_graph || permuted;
    if (via_host) ensure_host_out();
    uint16_t* xo = x_out ? (via_host ? m.h_x : x_out) : nullptr;
    float* lo = logits_out ? (via_host ? m.h_logits : logits_out) : nullptr;
    int* ao = argmax_out ? (via_host ? m.h_amax : argmax_out) : nullptr;
    if (!use_graph) {
        enqueue(st, xo, lo, ao);
    } else {
        std::string key;
        auto add = [&](long v) { key.append(reinterpret_cast<const char*>(&v), sizeof v); };
        for (long v : {static_cast<long>(n), static_cast<long>(n_rc), static_cast<long>(rc_max),
                       static_cast<long>(meta.size()), static_cast<long>(tr_src.size()), static_cast<long>(M),
                       static_cast<long>(stream_any), static_cast<long>(x_out != nullptr),
                       static_cast<long>(logits_out != nullptr), static_cast<long>(argmax_out != nullptr),
                       static_cast<long>(prefetched), m.graph_gen})
            add(v);
        for (int u = 0; u < M; ++u) {
            const Unit& U = units[u];
            for (long v : {static_cast<long>(mb_row[u + 1]), static_cast<long>(U.tiles_h.size()),
                           static_cast<long>(U.tiles_g.size()), static_cast<long>(U.splits),
                           static_cast<long>(U.any_act), static_cast<long>(U.any_kv), static_cast<long>(U.o_th),
                           static_cast<long>(U.o_tg)})
                add(v);
            for (const auto* runs : {&U.kv_runs, &U.act_runs}) {
                add(static_cast<long>(runs->size()));
                for (const Run& r : *runs) {
                    add((static_cast<long>(r.start) << 32) | r.count);
                    add(r.dst);
                }
            }
        }
        auto it = m.graphs.find(key);
        if (it == m.graphs.end()) {
            if (m.graphs.size() >= 8) {  // evict the least recently used
                auto lru = m.graphs.begin();
                for (auto g = m.graphs.begin(); g != m.graphs.end(); ++g)
                    if (g->second.last_use < lru->second.last_use) lru = g;
                cudaGraphExecDestroy(lru->second.exec);
                m.graphs.erase(lru);
            }
            Impl::StepGraph sg;
            cudaGraph_t g = nullptr;
            HC_CUDA(cudaStreamBeginCapture(s_compute_, cudaStreamCaptureModeThreadLocal));
            capturing = true;
            try {
                enqueue(sg.stats, xo, lo, ao);
            } catch (...) {
                capturing = false;
                cudaStreamEndCapture(s_compute_, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            capturing = false;
            HC_CUDA(cudaStreamEndCapture(s_compute_, &g));
            const cudaError_t e = cudaGraphInstantiate(&sg.exec, g, 0);
            cudaGraphDestroy(g);
            HC_CUDA(e);
            it = m.graphs.emplace(key, sg).first;
        }
        it->second.last_use = ++m.graph_clock;
        st = it->second.stats;
        // timing events around the launch (events recorded inside a graph
        // cannot be timed)
        HC_CUDA(cudaEventRecord(m.tg0, s_compute_));
        HC_CUDA(cudaGraphLaunch(it->second.exec, s_compute_));
    }
    // next step's layer 0/1 weights (step-independent) over the link while the
    // last two layers compute — the reference arms weight(step+1) before the
    // step's tail too (sim.cpp:534-537); the step ends when they have landed
    if (!m.w_all && stream_any && m.wsn == 1) {
        for (int l = 0; l < std::min(2, m.L); ++l) {
            HC_CUDA(cudaStreamWaitEvent(s_copy_, m.w_consumed[l & 1]));
            stream_weights(l, l & 1, st);
        }
        HC_CUDA(cudaEventRecord(m.wpre, s_copy_));
        HC_CUDA(cudaStreamWaitEvent(s_compute_, m.wpre));
        m.w_prefetched = true;
    }
    HC_CUDA(cudaEventRecord(use_graph ? m.tg1 : m.ev1, s_compute_));
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    if (via_host) {  // back to the caller's request order
        for (int i = 0; i < n; ++i) {
            const int b = order[i];
            if (x_out) std::memcpy(x_out + static_cast<size_t>(b) * m.d, m.h_x + static_cast<size_t>(i) * m.d, m.d * 2);
            if (logits_out)
                std::memcpy(logits_out + static_cast<size_t>(b) * m.V, m.h_logits + static_cast<size_t>(i) * m.V,
                            static_cast<size_t>(m.V) * 4);
            if (argmax_out) argmax_out[b] = m.h_amax[i];
        }
    }
    if (capture_inputs_ && permuted) {  // captured rows back to the caller's order too
        std::vector<uint16_t> c(captured_);
        for (int l = 0; l < m.L; ++l)
            for (int i = 0; i < n; ++i)
                std::memcpy(captured_.data() + (static_cast<size_t>(l) * n + order[i]) * m.d,
                            c.data() + (static_cast<size_t>(l) * n + i) * m.d, static_cast<size_t>(m.d) * 2);
    }
    float ms = 0;
    HC_CUDA(cudaEventElapsedTime(&ms, use_graph ? m.tg0 : m.ev0, use_graph ? m.tg1 : m.ev1));
    st.step_ms = ms;
    st.minibatches = M;
    // trace of the profiled step: the reference's SimEvent schema
    // (sim.hpp:50-58; trace.json main.cpp:263-275) from CUDA events
    std::string trace;
    if (profile_) {
        trace = "{\"events\":[";
        bool first = true;
        for (const auto& sp : m.spans) {
            float t0 = 0, t1 = 0;
            HC_CUDA(cudaEventElapsedTime(&t0, m.ev0, sp.a));
            HC_CUDA(cudaEventElapsedTime(&t1, m.ev0, sp.b));
            static const char* names[4] = {"kv_gen", "attention", "qkv_and_forward", "host_load"};
            char buf[256];
            std::snprintf(buf, sizeof buf,
                          "%s{\"name\":\"%s\",\"track\":\"%s\",\"start_us\":%.3f,\"end_us\":%.3f,\"iteration\":%ld,"
                          "\"layer\":%d,\"minibatch\":%d}",
                          first ? "" : ",", (sp.kind == 0 && token_mode_) ? "token_recompute" : names[sp.kind],
                          sp.kind == 3 ? "PCIe" : "GPU", t0 * 1e3, t1 * 1e3, static_cast<long>(step_counter_),
                          sp.layer, sp.minibatch);
            trace += buf;
            first = false;
        }
        trace += "]}";
        last_trace_ = trace;
    }
    ++step_counter_;
    for (const auto& sp : m.spans) {
        float t = 0;
        HC_CUDA(cudaEventElapsedTime(&t, sp.a, sp.b));
        if (sp.kind == 0) {
            st.recompute_ms += t;
            st.recompute_launches += 1;
        } else if (sp.kind == 1) {
            st.attn_ms += t;
        } else if (sp.kind == 2) {
            st.gemm_ms += t;
        } else {
            st.copy_ms += t;
        }
    }
    for (int b = 0; b < n; ++b) {
        if (act_host[b] >= 0) {
            st.d2h_bytes += static_cast<double>(m.d) * 2 * m.L;
            st.d2h_act += static_cast<double>(m.d) * 2 * m.L;
        }
        if (kv_host[b] >= 0) {
            st.d2h_bytes += static_cast<double>(m.dg) * 4 * m.L;
            st.d2h_kv += static_cast<double>(m.dg) * 4 * m.L;
        }
    }
    stats_ = st;
}

// ---------------------------------------------------------------------------
void Engine::read_weights(int layer, uint16_t* out) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    if (layer == -1) {
        HC_CUDA(cudaMemcpy(out, m.emb, static_cast<size_t>(m.V) * m.d * 2, cudaMemcpyDeviceToHost));
    } else if (layer == -2) {
        HC_CUDA(cudaMemcpy(out, m.pos, static_cast<size_t>(m.max_seq) * m.d * 2, cudaMemcpyDeviceToHost));
    } else if (layer == -3) {
        if (!m.opt()) throw InputError("read_weights: the reference arch has no final LayerNorm");
        HC_CUDA(cudaMemcpy(out, m.lnf, 2 * static_cast<size_t>(m.d) * 2, cudaMemcpyDeviceToHost));
    } else if (layer >= 0 && layer < m.L) {
        if (m.w_all)
            HC_CUDA(cudaMemcpy(out, m.w_all + static_cast<size_t>(layer) * m.LE, m.LE * 2, cudaMemcpyDeviceToHost));
        else
            std::memcpy(out, m.h_w + static_cast<size_t>(layer % m.Lw) * m.LE, m.LE * 2);
    } else {
        throw InputError("read_weights: layer out of range");
    }
}

void Engine::read_block(BlockKind kind, Location loc, int pbn, int layer, uint16_t* out) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    m.require_configured();
    if (layer < 0 || layer >= m.L) throw InputError("read_block: layer out of range");
    const bool kv = kind == BlockKind::KV;
    const long cap = kv ? (loc == Location::GpuMem ? m.kv_gpu_cap : m.kv_host_cap)
                        : (loc == Location::GpuMem ? m.act_gpu_cap : m.act_host_cap);
    if (pbn < 0 || pbn >= cap) throw InputError("read_block: pbn out of range");
    const bool act_host = !kv && loc == Location::HostMem;
    if (act_host && !m.owns(pbn)) throw InputError("read_block: ACT block owned by another tensor-parallel rank");
    const size_t be = kv ? m.kvb : m.actb;
    HC_CUDA(cudaStreamSynchronize(s_compute_));
    if (loc == Location::GpuMem) {
        const f16* base = kv ? m.kv_gpu : m.act_gpu;
        HC_CUDA(cudaMemcpy(out, base + (static_cast<size_t>(layer) * cap + pbn) * be, be * 2, cudaMemcpyDeviceToHost));
    } else {
        const f16* base = kv ? m.kv_host : m.act_host;
        const long hcap = kv ? cap : m.act_cap_n;
        const int idx = kv ? pbn : pbn / m.tpn;
        std::memcpy(out, base + (static_cast<size_t>(layer % m.Lp) * hcap + idx) * be, be * 2);
    }
}

// ---------------------------------------------------------------------------
double Engine::time_kv_gen(int n_tokens, int reps) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    if (n_tokens <= 0) throw InputError("time_kv_gen: n_tokens must be positive");
    if (reps <= 0) throw InputError("time_kv_gen: reps must be positive");
    // recompute GEMM over n tokens of the ACT staging (or GPU) pool, layer 0
    const long stage_rows = m.stage_act_cap * m.tpb;
    const long cap_rows = std::max(stage_rows, m.act_gpu_cap * m.tpb);
    if (n_tokens > cap_rows) throw InputError("time_kv_gen: more tokens than the ACT pools hold");
    const bool from_stage = stage_rows >= n_tokens;
    const f16* A = from_stage ? m.act_stage[0] : m.act_gpu;
    m.w_prefetched = false;  // wbuf[0] is reloaded with layer 0 below
    if (!m.w_all)
        HC_CUDA(cudaMemcpy(m.wbuf[0], m.h_w, m.LE * 2, cudaMemcpyHostToDevice));
    const f16* W = m.layer_w(0, 0);
    std::vector<int> tiles;
    for (int r = 0; r < n_tokens; r += gemm::BM) tiles.push_back(r);
    const size_t n_tiles = tiles.size();
    if (m.fused)  // every block full, all rows one request (query row 0)
        tiles.resize(n_tiles + n_tiles * (gemm::BM / m.tpb), m.tpb);
    m.ensure_meta(tiles.size());
    std::memcpy(m.h_meta, tiles.data(), tiles.size() * 4);
    HC_CUDA(cudaMemcpy(m.d_meta, m.h_meta, tiles.size() * 4, cudaMemcpyHostToDevice));
    if (m.fused) HC_CUDA(cudaMemset(m.qkvb, 0, static_cast<size_t>(3) * m.dg * 2));
    GemmCall c;
    c.epi = gemm::kKvPaged;
    c.A = A;
    c.lda = m.d;
    // the TMA map may not reach past the pool A points into (the last tile
    // of a non-multiple-of-128 n reads up to 127 rows further)
    c.a_rows = static_cast<int>(from_stage ? stage_rows : m.act_gpu_cap * m.tpb);
    c.B = W + m.off.wqkv + static_cast<size_t>(m.dg) * m.d;
    c.ldb = m.d;
    c.M = n_tokens;
    c.N = 2 * m.dg;
    c.K = m.d;
    c.m_tile_rows = m.d_meta;
    c.num_m_tiles = static_cast<int>(n_tiles);
    c.out = m.kvr;
    c.tpb = m.tpb;
    c.d = m.dg;
    c.hd = m.hd;
    c.bias = m.bias(W, m.off.bqkv + m.dg);
    if (m.fused) {  // the kernel the decode step runs: recompute fused with attention
        c.epi = gemm::kAttnPart;
        c.blk_info = m.d_meta + n_tiles;
        c.q = m.qkvb;
        c.ldq = 3 * m.dg;
        c.qscale = 1.f;
        c.part = m.part;
    }
    run_gemm(c, s_compute_);  // warm-up
    HC_CUDA(cudaEventRecord(m.ev0, s_compute_));
    for (int i = 0; i < reps; ++i) run_gemm(c, s_compute_);
    HC_CUDA(cudaEventRecord(m.ev1, s_compute_));
    HC_CUDA(cudaEventSynchronize(m.ev1));
    float ms = 0;
    HC_CUDA(cudaEventElapsedTime(&ms, m.ev0, m.ev1));
    return ms / 1e3 / reps;
}

double Engine::time_load_bytes(size_t bytes, int reps) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    Impl& m = *impl_;
    // pinned arena (KV then ACT host pools) -> the larger staging slot pair
    const bool kv_dst = m.stage_kv_cap * m.kvb >= m.stage_act_cap * m.actb;
    f16* dst[2] = {kv_dst ? m.kv_stage[0] : m.act_stage[0], kv_dst ? m.kv_stage[1] : m.act_stage[1]};
    const size_t cap = std::min(m.h_arena_elems, kv_dst ? m.stage_kv_cap * m.kvb : m.stage_act_cap * m.actb) * 2;
    if (bytes == 0 || bytes > cap) throw InputError("time_load: byte count exceeds the host pools / staging");
    if (reps <= 0) throw InputError("time_load: reps must be positive");
    HC_CUDA(cudaMemcpyAsync(dst[0], m.h_arena, bytes, cudaMemcpyHostToDevice, s_copy_));
    HC_CUDA(cudaEventRecord(m.ev0, s_copy_));
    for (int i = 0; i < reps; ++i)
        HC_CUDA(cudaMemcpyAsync(dst[i & 1], m.h_arena, bytes, cudaMemcpyHostToDevice, s_copy_));
    HC_CUDA(cudaEventRecord(m.ev1, s_copy_));
    HC_CUDA(cudaEventSynchronize(m.ev1));
    float ms = 0;
    HC_CUDA(cudaEventElapsedTime(&ms, m.ev0, m.ev1));
    return ms / 1e3 / reps;
}

double Engine::time_load_kv(int n_tokens, int reps) {
    HC_CUDA(cudaSetDevice(opt_.device));  // the calling thread may be on another device
    // this rank's bytes of n KV tokens (all heads, or its 1/tpn under tensor parallelism)
    return time_load_bytes(static_cast<size_t>(n_tokens) * 2 * impl_->dg * 2, reps);
}

}  // namespace hc
