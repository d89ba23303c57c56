// The B200 decode engine for the KV-activation hybrid cache.
//
// One Engine owns one GPU's slice of the batch (requests never interact,
// SURVEY.md §8(e)): its HybridCache bookkeeping, its block pools and its
// pipeline. Pools (payload storage behind every pbn of cache.hpp):
//
//   KV / gpu    HBM      [L][kv_gpu_cap][2][H][tpb][hd]     resident
//   ACT / gpu   HBM      [L][act_gpu_cap][tpb][d]           resident
//   KV / host   pinned   [Lp][kv_host_cap][2][H][tpb][hd]   streamed per layer
//   ACT / host  pinned   [Lp][act_host_cap][tpb][d]         streamed per layer
//
// Lp = host_layers (default L). Lp < L folds the host pools' storage (logical
// layer l uses physical copy l % Lp) for hosts with less DRAM than the full
// cache; the bytes streamed per layer are unchanged.
//
// Decode step, per layer l (north-star (1)-(4)):
//   copy stream : [weights(l)] + KV/host runs + ACT/host runs -> slot l%2
//   compute     : act_append (ACT writer: new token's X -> its ACT slot,
//                 device + pinned host) -> recompute GEMM (tcgen05, ACT blocks
//                 -> K|V straight into paged layout) -> QKV GEMM -> kv_append
//                 (new token's K|V -> its KV slot, device + host) -> decode
//                 attention over the hybrid block table -> proj -> FFN1+relu
//                 -> FFN2 (= next layer's X)
//   copy(l+2) waits for compute(l) to release slot l%2 (double buffering,
//   sim.cpp:419-429's "2 units in flight").
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "host/cache.hpp"
#include "host/minibatch.hpp"
#include "host/model.hpp"
#include "kernels/kernels.hpp"
#include "tp.hpp"

namespace hc {

struct EngineOptions {
    int max_batch = 1;            // max requests per decode step
    int max_seq = 0;              // max context per request (0: weights.max_seq)
    int weights_on_device = 1;    // 0: weights in pinned host memory, streamed per layer
    long kv_host_cap = 0, kv_gpu_cap = 0, act_host_cap = 0, act_gpu_cap = 0;
    int kv_on_gpu = 0;
    int host_layers = 0;          // Lp (0 = num_layers)
    int weight_layers = 0;        // physical pinned weight layers (0 = num_layers; < L folds
                                  // layer l onto copy l % Lw — benchmark hosts with small DRAM)
    CacheMode mode = CacheMode::Hybrid;
    HostAllocation alloc{};       // hybrid-ratio setting (next_block_kind target)
    double recompute_ratio = 0.0;
    int scaled = 1;
    int max_prefill_tokens = 65536;
    int device = 0;
    int arch = kArchReference;    // decoder layer variant (host/model.hpp); from the weights when given
    TpGroup* tp = nullptr;        // head-sharded tensor parallelism (tp.hpp); nullptr = one GPU holds all heads
    // batch-partitioned ranks sharing ONE weight stream (streamed weights only):
    // rank g of N copies 1/N of every layer over its own host link and an
    // NVLink all-gather completes the layer, so each link carries 1/N of the
    // weights; nullptr = every rank streams whole layers
    TpGroup* weight_share = nullptr;
};

struct StepStats {
    double step_ms = 0;           // compute-stream time of the whole step
    double h2d_bytes = 0;         // bytes streamed host->device this step
    double d2h_bytes = 0;         // bytes stored device->host (mapped writes)
    double recompute_tokens = 0;  // ACT rows recomputed (incl. padding rows)
    double recompute_ms = 0;      // summed recompute GEMM time (when profiled)
    double attn_ms = 0;
    double gemm_ms = 0;           // QKV + proj + FFN GEMMs
    int launches = 0;             // kernels launched this step
    double copy_ms = 0;           // summed copy-stream time of the H2D streams (profiled)
    int recompute_launches = 0;
    double store_ms = 0;          // summed store-stream (D2H) time (profiled prefill)
    int minibatches = 1;          // (layer, mini-batch) units per layer of the last decode step
    // the h2d / d2h bytes by kind (the reference's traffic classes, sim.hpp:60-66)
    double h2d_weights = 0, h2d_kv = 0, h2d_act = 0, d2h_kv = 0, d2h_act = 0;
};

class Engine {
public:
    Engine(const HostWeights& w, const EngineOptions& o);
    // Draw DecoderWeights::generate(config, seed, max_seq) (+ rescale) layer by
    // layer straight into the engine's own memory (no full host copy).
    Engine(const ModelConfig& c, uint64_t seed, int max_seq, bool rescale, const EngineOptions& o);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Prefill (forward_prompt semantics, decoder.cpp:144-157) of new requests;
    // writes every layer's ACT / KV blocks chosen by the ratio policy.
    // Layer-outer pipeline: weights streamed once per layer, host blocks
    // stored by D2H copies on a store stream (last_stats(): step_ms = the
    // whole prefill, h2d = weights, d2h = stored blocks).
    void prefill(const std::vector<std::string>& ids, const std::vector<std::vector<int>>& prompts);
    // Admit requests with prompt_len tokens of bookkeeping only and fill their
    // blocks with a deterministic pattern (benchmark setup; no numerics).
    void admit_synthetic(const std::vector<std::string>& ids, const std::vector<int>& prompt_lens, uint64_t seed);
    // Mini-batched decode (paper §4.3.3; sim.cpp:258-358): staging slots hold
    // act_max ACT / kv_max KV blocks (+ one growth block per request); every
    // step packs its requests with form_minibatches (minibatch.cpp:36-83) on
    // pre-growth block counts, priced by `bundle`, and runs (layer,
    // mini-batch) units double-buffered. act_max = kv_max = 0 turns it off
    // (whole-batch steps, staging = the host pools).
    void set_minibatching(long act_max, long kv_max, const TimingBundle& bundle);
    // Recompute fused with decode attention (default on where supported: own
    // heads' width a multiple of 128): the recompute GEMM's epilogue reduces
    // each recomputed block to flash-decoding partials against the step's
    // queries instead of writing its K|V into the paged KV layout, so the
    // recomputed K|V never touch HBM. Off: the kKvPaged path (K|V stored,
    // attention reads them). Returns whether the fused path is in use.
    bool set_fused_recompute(bool on);
    bool fused_recompute() const;
    // Fill every pool slot with the deterministic pattern (benchmark setup:
    // slots that advance_synthetic later hands out then hold finite values).
    void fill_pools(uint64_t seed);
    // Grow each listed request by n_tokens through the allocator in decode
    // order (bookkeeping only; the slots keep the pool contents): places a
    // benchmark's timed steps at a later context without running the steps.
    void advance_synthetic(const std::vector<std::string>& ids, int n_tokens);

    // One decode step for the listed requests (generation_step semantics,
    // decoder.cpp:159-174, batched). Outputs are optional (nullptr = skip):
    // x_out [n x d] f16 bits, logits [n x V] fp32 (tied head x.E^T),
    // argmax [n].
    void decode_step(const std::vector<std::string>& ids, const int* tokens, uint16_t* x_out, float* logits,
                     int* argmax);
    void free_request(const std::string& id);
    // Token-recompute mode: tokens of the request kept as ids only (a
    // block-aligned prompt prefix, rebuilt through all layers every step).
    long recompute_prefix_len(const std::string& id) const;

    // Drop every request and re-create the block pools with new capacities /
    // ratio setting (weights and scratch stay): ratio sweeps on one engine.
    void configure_cache(const PoolCaps& caps, bool kv_on_gpu, CacheMode mode, const HostAllocation& alloc,
                         int host_layers, double recompute_ratio = 0.0);

    // forward_prompt (decoder.cpp:144-157) of one sequence on the GPU without
    // touching the cache: per-layer inputs X, K, V ([L][n][d]) and the output
    // [n][d], f16 bits. token_recompute_kv(ids, k) = (K, V)[k].
    void forward_trace(const std::vector<int>& ids, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                       uint16_t* out);
    // One layer of forward_prompt on caller-given input rows x [T x d]
    // (qkv_generate + attention_causal + project_ffn, decoder.cpp:150-153):
    // K, V [T x d] and the layer output [T x d]. Teacher-forced parity.
    void layer_forward(int layer, const uint16_t* x, int T, uint16_t* k, uint16_t* v, uint16_t* out);

    // Payload of one block at one layer (f16 bits; KV: [2][H][tpb][hd],
    // ACT: [tpb][d]) — for parity tests of the cache writers.
    void read_block(BlockKind kind, Location loc, int pbn, int layer, uint16_t* out);
    // Engine-held weights (f16 bits): layer >= 0 packed layer (model.hpp
    // layout), -1 embedding [V x d], -2 positional [max_seq x d], -3 final
    // LayerNorm gamma|beta [2d] (kArchOpt).
    void read_weights(int layer, uint16_t* out);
    // Decode-time layer inputs of the last step: [L][n][d] (debug / parity).
    void set_capture_layer_inputs(bool on) { capture_inputs_ = on; }
    const std::vector<uint16_t>& captured_layer_inputs() const { return captured_; }

    // Planner calibration (north-star (5)): time the recompute GEMM over
    // n ACT tokens and the host->device copy of n KV tokens on this engine's
    // streams; seconds per layer.
    double time_kv_gen(int n_tokens, int reps);
    double time_load_kv(int n_tokens, int reps);
    double time_load_bytes(size_t bytes, int reps);

    const HybridCache& cache() const { return *cache_; }
    HybridCache& cache() { return *cache_; }
    const ModelConfig& config() const { return cfg_; }
    const StepStats& last_stats() const { return stats_; }
    void set_profile(bool on) { profile_ = on; }
    // CUDA-graph replay of decode steps (default on; off with HC_DECODE_GRAPHS=0)
    void set_graphs(bool on) { graphs_ = on; }
    // {"events":[{name, track, start_us, end_us, iteration, layer, minibatch}]}
    // of the last profiled decode step — the reference's trace.json schema.
    const std::string& last_trace() const { return last_trace_; }
    cudaStream_t compute_stream() const { return s_compute_; }

private:
    struct Impl;
    void init(const ModelConfig& c, int max_seq, const uint16_t* emb, const uint16_t* pos, const uint16_t* final_ln,
              void (*fill_layer)(const void* ctx, int l, uint16_t* dst), const void* ctx);
    void run_layers(int T, int l0, int l1, const int* d_cu, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                    uint16_t* out, bool final_ln);
    std::unique_ptr<Impl> impl_;
    ModelConfig cfg_;
    EngineOptions opt_;
    std::unique_ptr<HybridCache> cache_;
    std::unique_ptr<BlockAssigner> assigner_;
    cudaStream_t s_compute_ = nullptr, s_copy_ = nullptr, s_store_ = nullptr, s_gather_ = nullptr;
    void alloc_staging();
    StepStats stats_{};
    bool profile_ = false;
    bool graphs_ = true;
    bool capture_inputs_ = false;
    std::string last_trace_;     // events of the last profiled step (JSON)
    long step_counter_ = 0;
    bool token_mode_ = false;                                     // CacheMode::TokenRecompute
    std::unordered_map<std::string, std::vector<int>> rc_ids_;    // recompute-only prompt prefixes
    int rc_prefix(int prompt_len) const;
    std::vector<uint16_t> captured_;
};

}  // namespace hc
