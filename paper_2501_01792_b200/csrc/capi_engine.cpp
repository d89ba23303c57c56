// C-ABI: model, cache bookkeeping, planner and engine entry points
// (include/hybridcache.h). Pure forwarding onto the C++ host API.
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "capi_util.hpp"
#include "engine.hpp"
#include "host/cache.hpp"
#include "host/minibatch.hpp"
#include "host/model.hpp"
#include "host/plan.hpp"
#include "hybridcache.h"

using namespace hc;

namespace {

ModelConfig to_cfg(const hc_model_config* c) {
    if (!c) throw InputError("null model config");
    ModelConfig m;
    m.num_layers = c->num_layers;
    m.hidden_dim = c->hidden_dim;
    m.num_heads = c->num_heads;
    m.ffn_dim = c->ffn_dim;
    m.vocab_size = c->vocab_size;
    m.tokens_per_block = c->tokens_per_block;
    m.bytes_per_scalar = c->bytes_per_scalar;
    return m;
}

void from_cfg(const ModelConfig& m, hc_model_config* c) {
    c->num_layers = m.num_layers;
    c->hidden_dim = m.hidden_dim;
    c->num_heads = m.num_heads;
    c->ffn_dim = m.ffn_dim;
    c->vocab_size = m.vocab_size;
    c->tokens_per_block = m.tokens_per_block;
    c->bytes_per_scalar = m.bytes_per_scalar;
}

BlockKind kind_of(int k) {
    if (k != 0 && k != 1) throw InputError("block kind must be 0 (KV) or 1 (ACT)");
    return k ? BlockKind::ACT : BlockKind::KV;
}
Location loc_of(int l) {
    if (l != 0 && l != 1) throw InputError("location must be 0 (host) or 1 (gpu)");
    return l ? Location::GpuMem : Location::HostMem;
}

TimingBundle bundle_of(const double* b) {
    TimingBundle t;
    t.t_kv_gen = LinearTimeModel{b[0], b[1], 1.0, false};
    t.t_load_kv = LinearTimeModel{b[2], b[3], 1.0, false};
    t.t_load_w = b[4];
    return t;
}

MemoryBudget mem_of(const double* m) { return MemoryBudget{m[0], m[1], m[2], m[3]}; }

EngineOptions opts_of(const hc_engine_options* o) {
    if (!o) throw InputError("null engine options");
    EngineOptions e;
    e.max_batch = o->max_batch;
    e.max_seq = o->max_seq;
    e.weights_on_device = o->weights_on_device;
    e.kv_host_cap = o->kv_host_cap;
    e.kv_gpu_cap = o->kv_gpu_cap;
    e.act_host_cap = o->act_host_cap;
    e.act_gpu_cap = o->act_gpu_cap;
    e.kv_on_gpu = o->kv_on_gpu;
    e.host_layers = o->host_layers;
    if (o->mode < 0 || o->mode > 3)
        throw InputError("engine mode must be 0 hybrid, 1 kv_only, 2 act_only, 3 token_recompute");
    e.mode = static_cast<CacheMode>(o->mode);
    e.alloc.act_host = o->alloc_act_host;
    e.alloc.kv_host = o->alloc_kv_host;
    e.scaled = o->scaled;
    e.max_prefill_tokens = o->max_prefill_tokens > 0 ? o->max_prefill_tokens : 65536;
    e.device = o->device;
    e.weight_layers = o->weight_layers;
    e.recompute_ratio = o->recompute_ratio;
    e.arch = o->arch;
    e.tp = static_cast<TpGroup*>(o->tp);
    e.weight_share = static_cast<TpGroup*>(o->weight_share);
    return e;
}

Engine* eng(void* e) {
    if (!e) throw InputError("null engine handle");
    return static_cast<Engine*>(e);
}
HybridCache* cch(void* c) {
    if (!c) throw InputError("null cache handle");
    return static_cast<HybridCache*>(c);
}
std::string sid(const char* s) {
    if (!s) throw InputError("null request id");
    return s;
}
std::vector<std::string> ids_of(int n, const char* const* ids) {
    std::vector<std::string> v;
    for (int i = 0; i < n; ++i) v.push_back(sid(ids[i]));
    return v;
}

}  // namespace

extern "C" {

int hc_model_validate(hc_model_config* cfg) {
    return hc_guard([&] {
        ModelConfig m = to_cfg(cfg);
        m.validate();
        from_cfg(m, cfg);
    });
}

int hc_model_preset(const char* name, hc_model_config* out) {
    return hc_guard([&] { from_cfg(ModelConfig::preset(sid(name)), out); });
}

int hc_generate_weights(const hc_model_config* cfg, uint64_t seed, int max_seq, int rescale, uint16_t* emb,
                        uint16_t* pos, uint16_t* layers) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        if (max_seq < 1) throw InputError("DecoderWeights: max_seq must be >= 1");
        std::vector<uint16_t> e(emb ? 0 : static_cast<size_t>(c.vocab_size) * c.hidden_dim);
        std::vector<uint16_t> p(pos ? 0 : static_cast<size_t>(max_seq) * c.hidden_dim);
        generate_tables(c, seed, max_seq, emb ? emb : e.data(), pos ? pos : p.data());
        if (layers) {
            const size_t le = LayerOffsets::of(c).total;
            for (int l = 0; l < c.num_layers; ++l) generate_layer(c, seed, l, rescale != 0, layers + le * l);
        }
    });
}

// ---- cache --------------------------------------------------------------
int hc_cache_create(int tpb, long kv_host, long kv_gpu, long act_host, long act_gpu, int kv_on_gpu, void** out) {
    return hc_guard([&] { *out = new HybridCache(tpb, PoolCaps{kv_host, kv_gpu, act_host, act_gpu}, kv_on_gpu != 0); });
}
int hc_cache_destroy(void* c) {
    return hc_guard([&] { delete cch(c); });
}
int hc_cache_create_request(void* c, const char* id, int prompt_len) {
    return hc_guard([&] { cch(c)->create_request(sid(id), prompt_len); });
}
int hc_cache_append_block(void* c, const char* id, int kind, int* loc, int* pbn) {
    return hc_guard([&] {
        const BlockTableEntry& e = cch(c)->append_block(sid(id), kind_of(kind));
        if (loc) *loc = static_cast<int>(e.location);
        if (pbn) *pbn = e.pbn;
    });
}
int hc_cache_fill_token(void* c, const char* id) {
    return hc_guard([&] { cch(c)->fill_token(sid(id)); });
}
int hc_cache_free_request(void* c, const char* id) {
    return hc_guard([&] { cch(c)->free_request(sid(id)); });
}
int hc_cache_context_len(void* c, const char* id, int* out) {
    return hc_guard([&] { *out = cch(c)->table(sid(id)).context_len(); });
}
int hc_cache_blocks_by_kind(void* c, const char* id, long* act, long* kv) {
    return hc_guard([&] {
        const auto [a, k] = cch(c)->blocks_by_kind(sid(id));
        *act = a;
        *kv = k;
    });
}
int hc_cache_free_blocks(void* c, int kind, int loc, long* out) {
    return hc_guard([&] { *out = cch(c)->free_blocks(kind_of(kind), loc_of(loc)); });
}
int hc_cache_capacity(void* c, int kind, int loc, long* out) {
    return hc_guard([&] { *out = cch(c)->capacity(kind_of(kind), loc_of(loc)); });
}
int hc_cache_table(void* c, const char* id, int* kinds, int* locs, int* pbns, int* filled, int cap, int* n) {
    return hc_guard([&] {
        const BlockTable& t = cch(c)->table(sid(id));
        *n = static_cast<int>(t.entries.size());
        for (int i = 0; i < *n && i < cap; ++i) {
            const auto& e = t.entries[i];
            if (kinds) kinds[i] = static_cast<int>(e.kind);
            if (locs) locs[i] = static_cast<int>(e.location);
            if (pbns) pbns[i] = e.pbn;
            if (filled) filled[i] = e.filled_tokens;
        }
    });
}
int hc_cache_dump_json(void* c, char* buf, long len, long* needed) {
    return hc_guard([&] {
        const std::string s = cch(c)->dump_json();
        if (needed) *needed = static_cast<long>(s.size() + 1);
        if (buf && len > 0) {
            const size_t k = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
            std::memcpy(buf, s.data(), k);
            buf[k] = '\0';
        }
    });
}
int hc_bytes_of(int kind, int hidden_dim, int tpb, int bps, uint64_t* out) {
    return hc_guard([&] {
        ModelConfig m;
        m.hidden_dim = hidden_dim;
        m.tokens_per_block = tpb;
        m.bytes_per_scalar = bps;
        *out = HybridCache::bytes_of(kind_of(kind), m);
    });
}

// ---- planner ------------------------------------------------------------
int hc_next_block_kind(long act_req, long kv_req, long act_host, long kv_host, int* kind) {
    return hc_guard([&] {
        HostAllocation a;
        a.act_host = act_host;
        a.kv_host = kv_host;
        *kind = static_cast<int>(next_block_kind(act_req, kv_req, a));
    });
}
int hc_fit_linear(const double* n, const double* s, int count, double* out4) {
    return hc_guard([&] {
        std::vector<Sample> v;
        for (int i = 0; i < count; ++i) v.push_back(Sample{n[i], s[i]});
        const LinearTimeModel m = fit_linear(v);
        out4[0] = m.slope;
        out4[1] = m.intercept;
        out4[2] = m.r_squared;
        out4[3] = m.intercept_clamped ? 1.0 : 0.0;
    });
}
int hc_initial_cache_allocation(const double* b, int tpb, long act_gpu, long* out2) {
    return hc_guard([&] {
        const auto [a, k] = initial_cache_allocation(bundle_of(b), tpb, act_gpu);
        out2[0] = a;
        out2[1] = k;
    });
}
int hc_alloc_remaining(const double* b, const double* m, int tpb, long act_init, long kv_init, long* out2) {
    return hc_guard([&] {
        const auto [x, y] = alloc_remaining(bundle_of(b), mem_of(m), tpb, act_init, kv_init);
        out2[0] = x;
        out2[1] = y;
    });
}
int hc_plan_host_allocation(const double* b, const double* m, int tpb, long act_gpu, long* a6) {
    return hc_guard([&] {
        const HostAllocation a = plan_host_allocation(bundle_of(b), mem_of(m), tpb, act_gpu);
        const long v[6] = {a.act_host, a.kv_host, a.act_init, a.kv_init, a.act_remain, a.kv_remain};
        std::memcpy(a6, v, sizeof v);
    });
}
int hc_plan_hbm_residency(const hc_model_config* cfg, long requests, long bpr, double hbm_bytes, double* share,
                          long* out4) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        const HbmPlan p = plan_hbm_residency(c, requests, bpr, hbm_bytes);
        *share = p.act_share;
        const long v[4] = {p.act_gpu, p.kv_gpu, p.act_host, p.kv_host};
        std::memcpy(out4, v, sizeof v);
    });
}
int hc_plan_hbm_tiers(const hc_model_config* cfg, long requests, long bpr, double hbm_bytes, double host_bytes,
                      const double* b, int weights_streamed, double* share, long* out4, double* times2) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        const HbmTierPlan p = plan_hbm_tiers(c, requests, bpr, hbm_bytes, bundle_of(b), host_bytes, weights_streamed != 0);
        *share = p.act_share;
        const long v[4] = {p.act_gpu, p.kv_gpu, p.act_host, p.kv_host};
        std::memcpy(out4, v, sizeof v);
        times2[0] = p.t_comp;
        times2[1] = p.t_link;
    });
}
int hc_plan_host_min_step(const hc_model_config* cfg, long requests, long bpr, double host_bytes, const double* b,
                          double* share, long* out2, double* times2) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        const HostStepPlan p = plan_host_min_step(c, requests, bpr, bundle_of(b), host_bytes);
        *share = p.act_share;
        out2[0] = p.act_host;
        out2[1] = p.kv_host;
        times2[0] = p.t_comp;
        times2[1] = p.t_link;
    });
}
int hc_planned_times(const double* b, int tpb, long act_host, long kv_host, long act_gpu, double* out2) {
    return hc_guard([&] {
        HostAllocation a;
        a.act_host = act_host;
        a.kv_host = kv_host;
        const TimingBundle t = bundle_of(b);
        out2[0] = planned_t_pcie(t, tpb, a);
        out2[1] = planned_t_computation(t, tpb, a, act_gpu);
    });
}
int hc_bundle_from_samples(const double* kv_n, const double* kv_s, int kv_count, const double* ld_n,
                           const double* ld_s, int ld_count, double bw, const hc_model_config* cfg, double* o) {
    return hc_guard([&] {
        std::vector<Sample> a, b;
        for (int i = 0; i < kv_count; ++i) a.push_back(Sample{kv_n[i], kv_s[i]});
        for (int i = 0; i < ld_count; ++i) b.push_back(Sample{ld_n[i], ld_s[i]});
        ModelConfig c = to_cfg(cfg);
        c.validate();
        const TimingBundle t = bundle_from_samples(a, b, bw, c);
        const double v[11] = {t.t_kv_gen.slope,  t.t_kv_gen.intercept,  t.t_kv_gen.r_squared,
                              t.t_kv_gen.intercept_clamped ? 1.0 : 0.0, t.t_load_kv.slope,
                              t.t_load_kv.intercept, t.t_load_kv.r_squared,
                              t.t_load_kv.intercept_clamped ? 1.0 : 0.0, t.t_load_w,
                              static_cast<double>(t.s_weight_layer), static_cast<double>(t.s_weight_total)};
        std::memcpy(o, v, sizeof v);
    });
}
int hc_budget_for(double host_mem, const hc_model_config* cfg, double s_weight_total, double* mem4) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        TimingBundle t;
        t.s_weight_total = static_cast<uint64_t>(s_weight_total);
        const MemoryBudget m = budget_for(host_mem, c, t);
        mem4[0] = m.m_host;
        mem4[1] = m.s_weight;
        mem4[2] = m.s_kv_block;
        mem4[3] = m.s_act_block;
    });
}
int hc_flop_count(int kind, const hc_model_config* cfg, long n, int k, double* out) {
    return hc_guard([&] {
        const ModelConfig c = to_cfg(cfg);  // pure arithmetic: no validation (flops.cpp:7-33)
        *out = flop_count(kind, c, n, k);
    });
}
int hc_weight_bytes(const hc_model_config* cfg, uint64_t* out2) {
    return hc_guard([&] {
        const ModelConfig c = to_cfg(cfg);  // pure arithmetic: no validation (timing.cpp:118-127)
        const WeightBytes w = weight_bytes(c);
        out2[0] = w.per_layer;
        out2[1] = w.total;
    });
}

// ---- mini-batch packer ----------------------------------------------------
namespace {
int pack_into(decltype(&form_minibatches) fn, int n, const char* const* ids, const long* act_blocks,
              const long* kv_blocks, long act_max, long kv_max, const double* b5, int tpb, int* order, int* batch_of,
              int* n_batches) {
    return hc_guard([&] {
        std::vector<RequestBlocks> reqs;
        for (int i = 0; i < n; ++i) reqs.push_back(RequestBlocks{sid(ids[i]), act_blocks[i], kv_blocks[i]});
        const auto mbs = fn(reqs, PackerConfig{act_max, kv_max}, bundle_of(b5), tpb);
        std::unordered_map<std::string, int> pos;
        for (int i = 0; i < n; ++i) pos[reqs[i].id] = i;
        int k = 0;
        for (size_t m = 0; m < mbs.size(); ++m)
            for (const std::string& id : mbs[m].ids) {
                order[k++] = pos.at(id);
                batch_of[pos.at(id)] = static_cast<int>(m);
            }
        *n_batches = static_cast<int>(mbs.size());
    });
}
}  // namespace

int hc_form_minibatches(int n, const char* const* ids, const long* act_blocks, const long* kv_blocks, long act_max,
                        long kv_max, const double* b5, int tpb, int* order, int* batch_of, int* n_batches) {
    return pack_into(&form_minibatches, n, ids, act_blocks, kv_blocks, act_max, kv_max, b5, tpb, order, batch_of,
                     n_batches);
}
int hc_brute_force_pack(int n, const char* const* ids, const long* act_blocks, const long* kv_blocks, long act_max,
                        long kv_max, const double* b5, int tpb, int* order, int* batch_of, int* n_batches) {
    return pack_into(&brute_force_pack, n, ids, act_blocks, kv_blocks, act_max, kv_max, b5, tpb, order, batch_of,
                     n_batches);
}
int hc_cost_fb(long act_mb, long kv_mb, const double* b5, int tpb, double* out2) {
    return hc_guard([&] {
        out2[0] = balance(act_mb, kv_mb, bundle_of(b5), tpb);
        out2[1] = cost_fb(act_mb, kv_mb, bundle_of(b5), tpb);
    });
}
int hc_default_packer(double gpu_mem_bytes, const hc_model_config* cfg, long* out2) {
    return hc_guard([&] {
        ModelConfig c = to_cfg(cfg);
        c.validate();
        const PackerConfig p = default_packer(gpu_mem_bytes, c);
        out2[0] = p.act_max;
        out2[1] = p.kv_max;
    });
}

// ---- engine -------------------------------------------------------------
int hc_engine_create(const hc_model_config* cfg, uint64_t seed, int max_seq, int rescale, const hc_engine_options* opt,
                     void** out) {
    return hc_guard([&] { *out = new Engine(to_cfg(cfg), seed, max_seq, rescale != 0, opts_of(opt)); });
}
int hc_engine_create_from_f64(const hc_model_config* cfg, int max_seq, const double* emb, const double* pos,
                              const double* const* layer_tensors, const hc_engine_options* opt, void** out) {
    return hc_guard([&] {
        const HostWeights w = weights_from_f64(to_cfg(cfg), max_seq, emb, pos, layer_tensors);
        *out = new Engine(w, opts_of(opt));
    });
}
int hc_engine_create_from_f64_opt(const hc_model_config* cfg, int max_seq, const double* emb, const double* pos,
                                  const double* const* layer_tensors, const double* const* layer_extras,
                                  const double* final_ln, const hc_engine_options* opt, void** out) {
    return hc_guard([&] {
        const HostWeights w = weights_from_f64_opt(to_cfg(cfg), max_seq, emb, pos, layer_tensors, layer_extras, final_ln);
        *out = new Engine(w, opts_of(opt));
    });
}
int hc_tp_nccl_unique_id(uint8_t* out) {
    return hc_guard([&] {
        if (!out) throw InputError("null id buffer");
        nccl_unique_id(out);
    });
}
int hc_tp_create_nccl(const uint8_t* idc, const uint8_t* idk, int rank, int size, int device, void** tp) {
    return hc_guard([&] {
        if (!idc || !idk || !tp) throw InputError("null argument");
        *tp = make_nccl_group(idc, idk, rank, size, device).release();
    });
}
struct LocalGroupHolder {
    std::shared_ptr<LocalGroupState> g;
};
int hc_tp_create_local_group(int size, void** group) {
    return hc_guard([&] {
        if (!group) throw InputError("null argument");
        *group = new LocalGroupHolder{make_local_group(size)};
    });
}
int hc_tp_local_member(void* group, int rank, void** tp) {
    return hc_guard([&] {
        if (!group || !tp) throw InputError("null argument");
        *tp = local_group_member(static_cast<LocalGroupHolder*>(group)->g, rank);
    });
}
int hc_tp_create_emulated(int rank, int size, void** tp) {
    return hc_guard([&] {
        if (!tp) throw InputError("null argument");
        *tp = make_emulated_group(rank, size).release();
    });
}
int hc_tp_destroy(void* h, int is_group) {
    return hc_guard([&] {
        if (is_group)
            delete static_cast<LocalGroupHolder*>(h);
        else
            delete static_cast<TpGroup*>(h);
    });
}
int hc_engine_destroy(void* e) {
    return hc_guard([&] { delete eng(e); });
}
int hc_engine_prefill(void* e, int n, const char* const* ids, const int* offsets, const int* tokens) {
    return hc_guard([&] {
        if (n < 0) throw InputError("prefill: negative request count");
        if (n > 0 && (!ids || !offsets || (!tokens && offsets[n] > 0)))
            throw InputError("prefill: null ids / offsets / tokens");
        if (n > 0 && offsets[0] < 0) throw InputError("prefill: offsets[0] must be >= 0");
        std::vector<std::vector<int>> prompts(static_cast<size_t>(n));
        for (int r = 0; r < n; ++r) {
            if (offsets[r + 1] < offsets[r]) throw InputError("prefill: offsets must be non-decreasing");
            prompts[r].assign(tokens + offsets[r], tokens + offsets[r + 1]);
        }
        eng(e)->prefill(ids_of(n, ids), prompts);
    });
}
int hc_engine_admit_synthetic(void* e, int n, const char* const* ids, const int* lens, uint64_t seed) {
    return hc_guard([&] { eng(e)->admit_synthetic(ids_of(n, ids), std::vector<int>(lens, lens + n), seed); });
}

int hc_engine_set_minibatching(void* e, long act_max, long kv_max, const double* bundle5) {
    return hc_guard([&] {
        TimingBundle b{};
        if (bundle5) b = bundle_of(bundle5);
        eng(e)->set_minibatching(act_max, kv_max, b);
    });
}

int hc_engine_set_fused_recompute(void* e, int on, int* active) {
    return hc_guard([&] {
        const bool a = on < 0 ? eng(e)->fused_recompute() : eng(e)->set_fused_recompute(on != 0);
        if (active) *active = a ? 1 : 0;
    });
}

int hc_engine_fill_pools(void* e, uint64_t seed) {
    return hc_guard([&] { eng(e)->fill_pools(seed); });
}

int hc_engine_advance_synthetic(void* e, int n, const char* const* ids, int n_tokens) {
    return hc_guard([&] { eng(e)->advance_synthetic(ids_of(n, ids), n_tokens); });
}
int hc_engine_decode_step(void* e, int n, const char* const* ids, const int* tokens, uint16_t* x_out, float* logits,
                          int* argmax) {
    return hc_guard([&] {
        if (n < 0) throw InputError("decode_step: negative request count");
        if (n > 0 && (!ids || !tokens)) throw InputError("decode_step: null ids / tokens");
        eng(e)->decode_step(ids_of(n, ids), tokens, x_out, logits, argmax);
    });
}
int hc_engine_configure_cache(void* e, long kv_host, long kv_gpu, long act_host, long act_gpu, int kv_on_gpu, int mode,
                              long alloc_act_host, long alloc_kv_host, int host_layers, double recompute_ratio) {
    return hc_guard([&] {
        if (mode < 0 || mode > 3)
            throw InputError("engine mode must be 0 hybrid, 1 kv_only, 2 act_only, 3 token_recompute");
        HostAllocation a;
        a.act_host = alloc_act_host;
        a.kv_host = alloc_kv_host;
        eng(e)->configure_cache(PoolCaps{kv_host, kv_gpu, act_host, act_gpu}, kv_on_gpu != 0,
                                static_cast<CacheMode>(mode), a, host_layers, recompute_ratio);
    });
}
int hc_engine_forward_trace(void* e, const int* ids, int n, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                            uint16_t* out) {
    return hc_guard([&] { eng(e)->forward_trace(std::vector<int>(ids, ids + n), layer_inputs, k, v, out); });
}
int hc_engine_layer_forward(void* e, int layer, const uint16_t* x, int n, uint16_t* k, uint16_t* v, uint16_t* out) {
    return hc_guard([&] { eng(e)->layer_forward(layer, x, n, k, v, out); });
}
int hc_engine_free_request(void* e, const char* id) {
    return hc_guard([&] { eng(e)->free_request(sid(id)); });
}
int hc_engine_cache(void* e, void** cache) {
    return hc_guard([&] { *cache = &eng(e)->cache(); });
}
int hc_engine_read_block(void* e, int kind, int loc, int pbn, int layer, uint16_t* out) {
    return hc_guard([&] { eng(e)->read_block(kind_of(kind), loc_of(loc), pbn, layer, out); });
}
int hc_engine_read_weights(void* e, int layer, uint16_t* out) {
    return hc_guard([&] { eng(e)->read_weights(layer, out); });
}
int hc_engine_capture_inputs(void* e, int on) {
    return hc_guard([&] { eng(e)->set_capture_layer_inputs(on != 0); });
}
int hc_engine_captured_inputs(void* e, uint16_t* out, long count) {
    return hc_guard([&] {
        const auto& v = eng(e)->captured_layer_inputs();
        if (count < static_cast<long>(v.size())) throw InputError("captured_inputs: buffer too small");
        std::memcpy(out, v.data(), v.size() * 2);
    });
}
int hc_engine_last_stats(void* e, double* o) {
    return hc_guard([&] {
        const StepStats& s = eng(e)->last_stats();
        const double v[17] = {s.step_ms, s.h2d_bytes, s.d2h_bytes, s.recompute_tokens, s.recompute_ms,
                              s.attn_ms, s.gemm_ms, static_cast<double>(s.launches), s.copy_ms,
                              static_cast<double>(s.recompute_launches), s.store_ms,
                              static_cast<double>(s.minibatches), s.h2d_weights, s.h2d_kv, s.h2d_act,
                              s.d2h_kv, s.d2h_act};
        std::memcpy(o, v, sizeof v);
    });
}
int hc_engine_set_graphs(void* e, int on) {
    return hc_guard([&] { eng(e)->set_graphs(on != 0); });
}
int hc_engine_trace_json(void* e, char* buf, long len, long* needed) {
    return hc_guard([&] {
        const std::string& s = eng(e)->last_trace();
        if (needed) *needed = static_cast<long>(s.size() + 1);
        if (buf && len > 0) {
            const size_t k = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
            std::memcpy(buf, s.data(), k);
            buf[k] = '\0';
        }
    });
}
int hc_engine_set_profile(void* e, int on) {
    return hc_guard([&] { eng(e)->set_profile(on != 0); });
}
int hc_engine_time_kv_gen(void* e, int n_tokens, int reps, double* seconds) {
    return hc_guard([&] { *seconds = eng(e)->time_kv_gen(n_tokens, reps); });
}
int hc_engine_time_load_kv(void* e, int n_tokens, int reps, double* seconds) {
    return hc_guard([&] { *seconds = eng(e)->time_load_kv(n_tokens, reps); });
}

}  // extern "C"
