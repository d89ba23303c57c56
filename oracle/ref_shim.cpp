// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" adapter over the UNMODIFIED reference library (hybridsim,
// /root/reference/proj/src/*.cpp compiled in place by oracle/Makefile) so the
// Python test-suite and bench.py's cpu_baseline leg can drive the reference
// itself through ctypes. Every entry point forwards to one reference API:
//
//   ref_weights_*          -> DecoderWeights::generate      model.cpp:94-117
//   ref_forward_prompt     -> forward_prompt                decoder.cpp:144-157
//   ref_generation_step    -> generation_step               decoder.cpp:159-174
//   ref_recompute_kv       -> recompute_kv_from_activation  decoder.cpp:123-129
//   ref_token_recompute_kv -> token_recompute_kv            decoder.cpp:131-142
//   ref_attention_step     -> attention_step                decoder.cpp:105-111
//   ref_project_ffn        -> project_ffn                   decoder.cpp:113-121
//   ref_cache_*            -> HybridCache                   cache.cpp:35-166
//   ref_next_block_kind    -> next_block_kind               plan.cpp:154-164
//   ref_plan_*             -> initial/alloc_remaining/plan  plan.cpp:53-152
//   ref_fit_linear         -> fit_linear                    timing.cpp:38-73
//   ref_flop_count         -> flop_count                    flops.cpp:7-33
//   ref_equivalence        -> run_equivalence_case          verify.cpp:26-95
//   ref_simulate           -> simulate                      sim.cpp:134-633
//
// Status codes: 0 ok, 1 InputError, 2 CapacityError, 3 ConfigError, 4 other.
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hybridsim/cache.hpp"
#include "hybridsim/decoder.hpp"
#include "hybridsim/errors.hpp"
#include "hybridsim/flops.hpp"
#include "hybridsim/minibatch.hpp"
#include "hybridsim/plan.hpp"
#include "hybridsim/sim.hpp"
#include "hybridsim/timing.hpp"
#include "hybridsim/verify.hpp"

using namespace hybridsim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const InputError& e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Matrix* weight_slot(DecoderWeights& w, int which, int layer) {
    if (which == 0) return &w.embedding;
    if (which == 1) return &w.positional;
    if (layer < 0 || layer >= static_cast<int>(w.layers.size())) return nullptr;
    LayerWeights& lw = w.layers[static_cast<std::size_t>(layer)];
    switch (which) {
        case 2: return &lw.w_q;
        case 3: return &lw.w_k;
        case 4: return &lw.w_v;
        case 5: return &lw.w_proj;
        case 6: return &lw.w_ffn1;
        case 7: return &lw.w_ffn2;
        default: return nullptr;
    }
}

Matrix from_raw(const double* p, int rows, int cols) {
    Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data.data(), p, sizeof(double) * m.data.size());
    return m;
}

void to_raw(const Matrix& m, double* p) {
    if (!m.data.empty()) std::memcpy(p, m.data.data(), sizeof(double) * m.data.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- model + weights ------------------------------------------------------
// ModelConfig::preset (model.cpp:37-43): out6 = {layers, d, heads, ffn, vocab, tpb}
int ref_model_preset(const char* name, int* out6) {
    return guarded([&] {
        const ModelConfig c = ModelConfig::preset(name);
        out6[0] = c.num_layers;
        out6[1] = c.hidden_dim;
        out6[2] = c.num_heads;
        out6[3] = c.ffn_dim;
        out6[4] = c.vocab_size;
        out6[5] = c.tokens_per_block;
    });
}

int ref_weights_new(int layers, int d, int heads, int ffn, int vocab, int tpb, uint64_t seed,
                    int max_seq, void** out) {
    return guarded([&] {
        ModelConfig c;
        c.num_layers = layers;
        c.hidden_dim = d;
        c.num_heads = heads;
        c.ffn_dim = ffn;
        c.vocab_size = vocab;
        c.tokens_per_block = tpb;
        *out = new DecoderWeights(DecoderWeights::generate(c, seed, max_seq));
    });
}

void ref_weights_free(void* h) { delete static_cast<DecoderWeights*>(h); }

int ref_weights_shape(void* h, int which, int layer, int* rows, int* cols) {
    return guarded([&] {
        Matrix* m = weight_slot(*static_cast<DecoderWeights*>(h), which, layer);
        if (!m) throw InputError("bad weight slot");
        *rows = m->rows;
        *cols = m->cols;
    });
}

int ref_weights_get(void* h, int which, int layer, double* out) {
    return guarded([&] {
        Matrix* m = weight_slot(*static_cast<DecoderWeights*>(h), which, layer);
        if (!m) throw InputError("bad weight slot");
        to_raw(*m, out);
    });
}

int ref_weights_set(void* h, int which, int layer, const double* in) {
    return guarded([&] {
        Matrix* m = weight_slot(*static_cast<DecoderWeights*>(h), which, layer);
        if (!m) throw InputError("bad weight slot");
        std::memcpy(m->data.data(), in, sizeof(double) * m->data.size());
    });
}

// ---- decoder numerics -----------------------------------------------------
int ref_forward_prompt(void* h, const int* ids, int n, int scaled, double* layer_inputs,
                       double* k, double* v, double* out) {
    return guarded([&] {
        const auto& w = *static_cast<DecoderWeights*>(h);
        const ForwardTrace t = forward_prompt(std::span<const int>(ids, n), w, scaled != 0);
        const std::size_t per = static_cast<std::size_t>(n) * w.config.hidden_dim;
        for (int l = 0; l < w.config.num_layers; ++l) {
            if (layer_inputs) to_raw(t.layer_inputs[l], layer_inputs + per * l);
            if (k) to_raw(t.kv[l].k, k + per * l);
            if (v) to_raw(t.kv[l].v, v + per * l);
        }
        if (out) to_raw(t.output, out);
    });
}

// ctx_k/ctx_v: [L][ctx][d]
int ref_generation_step(void* h, int token, int pos, const double* ctx_k, const double* ctx_v,
                        int ctx, int scaled, double* out, double* new_k, double* new_v) {
    return guarded([&] {
        const auto& w = *static_cast<DecoderWeights*>(h);
        const int d = w.config.hidden_dim;
        const std::size_t per = static_cast<std::size_t>(ctx) * d;
        std::vector<KvPair> context;
        for (int l = 0; l < w.config.num_layers; ++l)
            context.push_back(KvPair{from_raw(ctx_k + per * l, ctx, d),
                                     from_raw(ctx_v + per * l, ctx, d)});
        const StepResult r = generation_step(token, pos, context, w, scaled != 0);
        to_raw(r.output, out);
        for (int l = 0; l < w.config.num_layers; ++l) {
            if (new_k) to_raw(r.new_kv[l].k, new_k + static_cast<std::size_t>(d) * l);
            if (new_v) to_raw(r.new_kv[l].v, new_v + static_cast<std::size_t>(d) * l);
        }
    });
}

int ref_recompute_kv(void* h, int layer, const double* a, int n, double* k, double* v) {
    return guarded([&] {
        const auto& w = *static_cast<DecoderWeights*>(h);
        const KvPair kv = recompute_kv_from_activation(from_raw(a, n, w.config.hidden_dim), layer, w);
        to_raw(kv.k, k);
        to_raw(kv.v, v);
    });
}

int ref_token_recompute_kv(void* h, const int* ids, int n, int layer, int scaled, double* k,
                           double* v) {
    return guarded([&] {
        const auto& w = *static_cast<DecoderWeights*>(h);
        const KvPair kv = token_recompute_kv(std::span<const int>(ids, n), w, layer, scaled != 0);
        to_raw(kv.k, k);
        to_raw(kv.v, v);
    });
}

int ref_attention_step(const double* q, const double* k, const double* v, int ctx, int d,
                       int heads, int scaled, double* out) {
    return guarded([&] {
        const Matrix o = attention_step(from_raw(q, 1, d), KvPair{from_raw(k, ctx, d), from_raw(v, ctx, d)},
                                        heads, scaled != 0);
        to_raw(o, out);
    });
}

int ref_project_ffn(void* h, int layer, const double* att, int n, double* out) {
    return guarded([&] {
        const auto& w = *static_cast<DecoderWeights*>(h);
        to_raw(project_ffn(from_raw(att, n, w.config.hidden_dim), layer, w), out);
    });
}

int ref_equivalence(uint64_t seed, int fault, int scaled, double* max_rel_dev, int* exact) {
    return guarded([&] {
        const EquivalenceResult r = run_equivalence_case(seed, fault != 0, scaled != 0);
        *max_rel_dev = r.max_rel_dev;
        *exact = r.exact ? 1 : 0;
    });
}

double ref_flop_count(int kind, int d, int ffn, long n, int k, int layers) {
    ModelConfig c;
    c.num_layers = layers;
    c.hidden_dim = d;
    c.num_heads = 1;
    c.ffn_dim = ffn;
    c.validate();
    return flop_count(static_cast<FlopKind>(kind), c, n, k);
}

// ---- cache bookkeeping ----------------------------------------------------
void* ref_cache_new(int tpb, long kv_host, long kv_gpu, long act_host, long act_gpu, int kv_on_gpu) {
    try {
        return new HybridCache(tpb, PoolCaps{kv_host, kv_gpu, act_host, act_gpu}, kv_on_gpu != 0);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_cache_free(void* c) { delete static_cast<HybridCache*>(c); }

int ref_cache_create_request(void* c, const char* id, int prompt_len) {
    return guarded([&] { static_cast<HybridCache*>(c)->create_request(id, prompt_len); });
}

// kind: 0 KV, 1 ACT. loc out: 0 host, 1 gpu.
int ref_cache_append_block(void* c, const char* id, int kind, int* loc, int* pbn) {
    return guarded([&] {
        const BlockTableEntry& e = static_cast<HybridCache*>(c)->append_block(
            id, kind == 1 ? BlockKind::ACT : BlockKind::KV);
        *loc = e.location == Location::GpuMem ? 1 : 0;
        *pbn = e.pbn;
    });
}

int ref_cache_fill_token(void* c, const char* id) {
    return guarded([&] { static_cast<HybridCache*>(c)->fill_token(id); });
}

int ref_cache_free_request(void* c, const char* id) {
    return guarded([&] { static_cast<HybridCache*>(c)->free_request(id); });
}

int ref_cache_context_len(void* c, const char* id, int* out) {
    return guarded([&] { *out = static_cast<HybridCache*>(c)->table(id).context_len(); });
}

int ref_cache_blocks_by_kind(void* c, const char* id, long* act, long* kv) {
    return guarded([&] {
        auto [a, k] = static_cast<HybridCache*>(c)->blocks_by_kind(id);
        *act = a;
        *kv = k;
    });
}

long ref_cache_free_blocks(void* c, int kind, int loc) {
    return static_cast<HybridCache*>(c)->free_blocks(kind == 1 ? BlockKind::ACT : BlockKind::KV,
                                                     loc == 1 ? Location::GpuMem : Location::HostMem);
}

// Writes dump_json().dump() into buf; returns required length (incl. NUL).
long ref_cache_dump_json(void* c, char* buf, long len) {
    const std::string s = static_cast<HybridCache*>(c)->dump_json().dump();
    if (buf && len > 0) {
        const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(len - 1));
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return static_cast<long>(s.size() + 1);
}

unsigned long ref_bytes_of(int kind, int d, int tpb, int bps) {
    ModelConfig c;
    c.hidden_dim = d;
    c.tokens_per_block = tpb;
    c.bytes_per_scalar = bps;
    return HybridCache::bytes_of(kind == 1 ? BlockKind::ACT : BlockKind::KV, c);
}

// ---- planner --------------------------------------------------------------
static TimingBundle bundle_of(const double* b) {
    // b = {kvgen_slope, kvgen_icept, load_slope, load_icept, t_load_w}
    TimingBundle t;
    t.t_kv_gen = LinearTimeModel{b[0], b[1], 1.0, false};
    t.t_load_kv = LinearTimeModel{b[2], b[3], 1.0, false};
    t.t_load_w = b[4];
    return t;
}

int ref_next_block_kind(long act_req, long kv_req, long act_host, long kv_host, int* kind) {
    return guarded([&] {
        HostAllocation a;
        a.act_host = act_host;
        a.kv_host = kv_host;
        *kind = next_block_kind(act_req, kv_req, a) == BlockKind::ACT ? 1 : 0;
    });
}

int ref_initial_cache_allocation(const double* bundle, int tpb, long act_gpu, long* out2) {
    return guarded([&] {
        auto [a, k] = initial_cache_allocation(bundle_of(bundle), tpb, GpuResidency{act_gpu});
        out2[0] = a;
        out2[1] = k;
    });
}

// mem = {m_host, s_weight, s_kv_block, s_act_block}
int ref_alloc_remaining(const double* bundle, const double* mem, int tpb, long act_init,
                        long kv_init, long* out2) {
    return guarded([&] {
        MemoryBudget m{mem[0], mem[1], mem[2], mem[3]};
        auto [x, y] = alloc_remaining(bundle_of(bundle), m, tpb, act_init, kv_init);
        out2[0] = x;
        out2[1] = y;
    });
}

// out6 = {act_host, kv_host, act_init, kv_init, act_remain, kv_remain}
int ref_plan_host_allocation(const double* bundle, const double* mem, int tpb, long act_gpu,
                             long* out6) {
    return guarded([&] {
        MemoryBudget m{mem[0], mem[1], mem[2], mem[3]};
        const HostAllocation a = plan_host_allocation(bundle_of(bundle), m, tpb, GpuResidency{act_gpu});
        out6[0] = a.act_host;
        out6[1] = a.kv_host;
        out6[2] = a.act_init;
        out6[3] = a.kv_init;
        out6[4] = a.act_remain;
        out6[5] = a.kv_remain;
    });
}

// Parse a bundle.json / plan.json with the reference's own loaders
// (TimingBundle::from_json timing.cpp:155-163, HostAllocation::from_json
// plan.cpp:30-39): out7 = {kv slope, kv icept, load slope, load icept,
// t_load_w, s_weight_layer, s_weight_total}; alloc6 as ref_plan_host_allocation.
int ref_parse_artifacts(const char* bundle_json, const char* plan_json, double* out7, long* alloc6) {
    return guarded([&] {
        if (bundle_json) {
            const TimingBundle b = TimingBundle::from_json(nlohmann::json::parse(bundle_json));
            out7[0] = b.t_kv_gen.slope;
            out7[1] = b.t_kv_gen.intercept;
            out7[2] = b.t_load_kv.slope;
            out7[3] = b.t_load_kv.intercept;
            out7[4] = b.t_load_w;
            out7[5] = static_cast<double>(b.s_weight_layer);
            out7[6] = static_cast<double>(b.s_weight_total);
        }
        if (plan_json) {
            const HostAllocation a = HostAllocation::from_json(nlohmann::json::parse(plan_json));
            alloc6[0] = a.act_host;
            alloc6[1] = a.kv_host;
            alloc6[2] = a.act_init;
            alloc6[3] = a.kv_init;
            alloc6[4] = a.act_remain;
            alloc6[5] = a.kv_remain;
        }
    });
}

// form_minibatches (minibatch.cpp:36-83): order / batch_of as hc_form_minibatches
int ref_form_minibatches(int n, const char* const* ids, const long* act, const long* kv, long act_max, long kv_max,
                         const double* b5, int tpb, int* order, int* batch_of, int* n_batches) {
    return guarded([&] {
        std::vector<RequestBlocks> reqs;
        for (int i = 0; i < n; ++i) reqs.push_back(RequestBlocks{ids[i], act[i], kv[i]});
        const auto mbs = form_minibatches(reqs, PackerConfig{act_max, kv_max}, bundle_of(b5), tpb);
        int k = 0;
        for (size_t m = 0; m < mbs.size(); ++m)
            for (const std::string& id : mbs[m].ids) {
                int i = 0;
                while (reqs[i].id != id) ++i;
                order[k++] = i;
                batch_of[i] = static_cast<int>(m);
            }
        *n_batches = static_cast<int>(mbs.size());
    });
}

// out4 = {slope, intercept, r2, clamped}
int ref_fit_linear(const double* n_tokens, const double* seconds, int count, double* out4) {
    return guarded([&] {
        std::vector<Sample> s;
        for (int i = 0; i < count; ++i) s.push_back(Sample{n_tokens[i], seconds[i]});
        const LinearTimeModel m = fit_linear(s);
        out4[0] = m.slope;
        out4[1] = m.intercept;
        out4[2] = m.r_squared;
        out4[3] = m.intercept_clamped ? 1.0 : 0.0;
    });
}


// The reference's discrete-event simulator (sim.cpp:134-633) as the PREDICTOR
// for a measured B200 bundle: uniform batch of `batch` requests (prompt, gen),
// allocation counts double as pool capacities (sim.cpp:181), one mini-batch.
// bundle5 = {kv slope, kv icept, load slope, load icept, t_load_w}; mode 0 hybrid,
// 1 kv_only, 2 act_only, 3 token_recompute.
// out6 = {throughput tok/s, makespan s, prefill s, gen s, pcie_busy, gpu_busy}
int ref_simulate(int layers, int d, int heads, int ffn, int vocab, int tpb, const double* bundle5, long act_host,
                 long kv_host, long act_gpu, int mode, double recompute_ratio, int batch, int prompt, int gen,
                 int full_duplex, double* out6) {
    return guarded([&] {
        SimConfig cfg;
        cfg.model.num_layers = layers;
        cfg.model.hidden_dim = d;
        cfg.model.num_heads = heads;
        cfg.model.ffn_dim = ffn;
        cfg.model.vocab_size = vocab;
        cfg.model.tokens_per_block = tpb;
        cfg.bundle = bundle_of(bundle5);
        const WeightBytes wb = weight_bytes(cfg.model);
        cfg.bundle.s_weight_layer = wb.per_layer;
        cfg.bundle.s_weight_total = wb.total;
        cfg.allocation.act_host = act_host;
        cfg.allocation.kv_host = kv_host;
        cfg.act_gpu = GpuResidency{act_gpu};
        cfg.packer = PackerConfig{1L << 40, 1L << 40};
        cfg.batch.assign(static_cast<std::size_t>(batch), RequestSpec{prompt, gen});
        cfg.mode = static_cast<SimMode>(mode);
        cfg.recompute_ratio = recompute_ratio;
        cfg.full_duplex_pcie = full_duplex != 0;
        const SimMetrics m = simulate(cfg).metrics;
        const double v[6] = {m.throughput, m.makespan, m.prefill_seconds, m.gen_seconds, m.pcie_busy, m.gpu_busy};
        std::memcpy(out6, v, sizeof v);
    });
}
// OpenMP threads of the reference's parallel loops (matrix.cpp:28,
// decoder.cpp:58); returns the count now in effect. Overrides an
// OMP_NUM_THREADS read at load time (torchrun sets it to 1).
int ref_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}

}  // extern "C"
