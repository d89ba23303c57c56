/*
 * hybridcache.h — C ABI of libhybridcache_b200.so, the B200-native (sm_100a)
 * KV-activation hybrid-caching decode path of arXiv 2501.01792.
 *
 * The reference ("hybridsim", /root/reference/proj) exposes a plain C++
 * library API; each entry point below names the reference
 * interface it replaces. Conventions:
 *   - every function returns int status: 0 ok, 1 InputError, 2 CapacityError,
 *     3 ConfigError, 4 CUDA/runtime error (errors.hpp:9-21); the message of
 *     the last failure on this thread is hc_last_error();
 *   - f16 tensors cross the boundary as uint16_t bit patterns, fp64 as double;
 *   - block kinds: 0 = KV, 1 = ACT; locations: 0 = host, 1 = gpu
 *     (cache.hpp:15-16);
 *   - matrices are row-major; reference-layout weights are [in x out]
 *     (A . W, model.hpp:38-45).
 * No CPU fallback exists: compute entry points fail (status 4) without a GPU.
 */
#ifndef HYBRIDCACHE_H
#define HYBRIDCACHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ library --- */
const char* hc_last_error(void);
int hc_abi_version(void);
int hc_device_count(void);
/* PCI bus id of a visible device (cudaDeviceGetPCIBusId), e.g. "0000:18:00.0". */
int hc_device_pci_bus_id(int device, char* buf, int len);
int hc_set_device(int device);

/* --------------------------------------------------------- model config ---
 * ModelConfig (model.hpp:15-36). ffn_dim 0 -> 4*hidden_dim. */
typedef struct hc_model_config {
    int num_layers;
    int hidden_dim;
    int num_heads;
    int ffn_dim;
    int vocab_size;
    int tokens_per_block;
    int bytes_per_scalar;
} hc_model_config;

/* ModelConfig::validate (model.cpp:8-17); fills ffn_dim in place. */
int hc_model_validate(hc_model_config* cfg);
/* ModelConfig::preset (model.cpp:37-43): "opt-6.7b" | "opt-13b" | "opt-30b" | "opt-66b". */
int hc_model_preset(const char* name, hc_model_config* out);

/* DecoderWeights::generate (model.cpp:94-117) + per-tensor rescale (rescale=1,
 * SURVEY.md §8(d)) + f16 rounding, in device layout: emb [V x d],
 * pos [max_seq x d], layers L x {Wqkv^T [3d x d], Wproj^T [d x d],
 * W1^T [f x d], W2^T [d x f]} (transposed, K-major). Any out may be NULL. */
int hc_generate_weights(const hc_model_config* cfg, uint64_t seed, int max_seq, int rescale, uint16_t* emb,
                        uint16_t* pos, uint16_t* layers);

/* ------------------------------------------------------ cache bookkeeping ---
 * HybridCache (cache.hpp:49-95, cache.cpp:35-166): bit-exact pbn / table
 * behaviour. Standalone handles, or the engine's own via hc_engine_cache. */
int hc_cache_create(int tokens_per_block, long kv_host, long kv_gpu, long act_host, long act_gpu, int kv_on_gpu,
                    void** out);
int hc_cache_destroy(void* cache);
int hc_cache_create_request(void* cache, const char* id, int prompt_len);   /* create_request  cache.cpp:66-74 */
int hc_cache_append_block(void* cache, const char* id, int kind, int* loc, int* pbn); /* append_block 79-107 */
int hc_cache_fill_token(void* cache, const char* id);                      /* fill_token      cache.cpp:109-117 */
int hc_cache_free_request(void* cache, const char* id);                    /* free_request    cache.cpp:123-132 */
int hc_cache_context_len(void* cache, const char* id, int* out);           /* BlockTable::context_len 12-16 */
int hc_cache_blocks_by_kind(void* cache, const char* id, long* act, long* kv); /* blocks_by_kind 18-27, 119-121 */
int hc_cache_free_blocks(void* cache, int kind, int loc, long* out);       /* free_blocks     cache.cpp:134-136 */
int hc_cache_capacity(void* cache, int kind, int loc, long* out);          /* capacity        cache.cpp:138-140 */
/* Block table of one request: up to cap entries; *n = entry count. */
int hc_cache_table(void* cache, const char* id, int* kinds, int* locs, int* pbns, int* filled, int cap, int* n);
/* dump_json().dump() (cache.cpp:149-166); *needed = bytes incl. NUL. */
int hc_cache_dump_json(void* cache, char* buf, long len, long* needed);
/* HybridCache::bytes_of (cache.cpp:142-147), per layer. */
int hc_bytes_of(int kind, int hidden_dim, int tokens_per_block, int bytes_per_scalar, uint64_t* out);

/* ----------------------------------------------------- ratio + planner ---
 * bundle5 = {kv_gen slope, kv_gen intercept, load_kv slope, load_kv intercept,
 *            t_load_w} (TimingBundle, timing.hpp:68-77)
 * mem4    = {m_host, s_weight, s_kv_block, s_act_block} (MemoryBudget, plan.hpp:27-32)
 * alloc6  = {act_host, kv_host, act_init, kv_init, act_remain, kv_remain} */
int hc_next_block_kind(long act_req, long kv_req, long act_host, long kv_host, int* kind); /* plan.cpp:154-164 */
int hc_fit_linear(const double* n_tokens, const double* seconds, int count, double* out4); /* timing.cpp:38-73 */
int hc_initial_cache_allocation(const double* bundle5, int tpb, long act_gpu, long* out2);  /* plan.cpp:53-69 */
int hc_alloc_remaining(const double* bundle5, const double* mem4, int tpb, long act_init, long kv_init,
                       long* out2);                                                         /* plan.cpp:71-104 */
int hc_plan_host_allocation(const double* bundle5, const double* mem4, int tpb, long act_gpu,
                            long* alloc6);                                                  /* plan.cpp:106-152 */
int hc_planned_times(const double* bundle5, int tpb, long act_host, long kv_host, long act_gpu,
                     double* out2);                                   /* planned_t_pcie / _computation 166-177 */
/* HBM residency (B200 extension, no reference counterpart): smallest ACT share
 * whose blocks fit hbm_bytes with KV and ACT placed on the GPU first.
 * out_share = r; out4 = {act_gpu, kv_gpu, act_host, kv_host} pool capacities. */
int hc_plan_hbm_residency(const hc_model_config* cfg, long requests, long blocks_per_request, double hbm_bytes,
                          double* out_share, long* out4);
/* Balanced three tiers (ACT in HBM, KV in HBM, KV streamed from pinned host)
 * minimising max(t_kv_gen, t_load_kv) per layer from a measured bundle5;
 * host_bytes bounds the pinned host tiers (0 = unbounded); weights_streamed:
 * the link also carries t_load_w per layer (weights left in pinned host);
 * out4 as above, out_times2 = predicted per-layer {t_comp, t_link} seconds. */
int hc_plan_hbm_tiers(const hc_model_config* cfg, long requests, long blocks_per_request, double hbm_bytes,
                      double host_bytes, const double* bundle5, int weights_streamed, double* out_share, long* out4,
                      double* out_times2);
/* Host-only plan minimising the predicted step (B200 extension of Alg. 1, whose
 * planned_t_pcie, plan.cpp:166-168, leaves the ACT blocks' own link time out):
 * x of N = requests * blocks_per_request host blocks as ACT minimising
 * max(t_load_w + t_load_kv(KV + ACT-equivalent tokens), t_kv_gen(x tpb)) per layer
 * within host_bytes (0 = unbounded). out2 = {act_host, kv_host} capacities
 * (+ one block per request of rounding slack), out_times2 = {t_comp, t_link}. */
int hc_plan_host_min_step(const hc_model_config* cfg, long requests, long blocks_per_request, double host_bytes,
                          const double* bundle5, double* out_share, long* out2, double* out_times2);
/* bundle_from_samples (timing.cpp:172-183) from MEASURED samples; out =
 * {kv slope, kv icept, kv r2, kv clamped, load slope, load icept, load r2,
 *  load clamped, t_load_w, s_weight_layer, s_weight_total} */
int hc_bundle_from_samples(const double* kv_n, const double* kv_s, int kv_count, const double* ld_n,
                           const double* ld_s, int ld_count, double link_bytes_per_s, const hc_model_config* cfg,
                           double* out11);
/* budget_for (plan.cpp:41-51) */
int hc_budget_for(double host_mem, const hc_model_config* cfg, double s_weight_total, double* mem4);
/* flop_count (flops.cpp:7-33); kind 0 KvGen 1 QkvGen 2 Attention 3 ProjFfn
 * 4 TokenRecomputeToLayerK 5 FullLayer */
int hc_flop_count(int kind, const hc_model_config* cfg, long n_tokens, int k, double* out);
/* weight_bytes (timing.cpp:118-127): out2 = {per_layer, total} */
int hc_weight_bytes(const hc_model_config* cfg, uint64_t* out2);

/* -------------------------------------------------- mini-batch packer ---
 * form_minibatches (minibatch.cpp:36-83): order[k] = request index in packing
 * order, batch_of[i] = mini-batch of request i. */
int hc_form_minibatches(int n, const char* const* ids, const long* act_blocks, const long* kv_blocks, long act_max,
                        long kv_max, const double* bundle5, int tpb, int* order, int* batch_of, int* n_batches);
/* brute_force_pack (minibatch.hpp:43-47; <= 10 requests): exhaustive search,
 * fewest mini-batches then smallest mean F_b; outputs as hc_form_minibatches. */
int hc_brute_force_pack(int n, const char* const* ids, const long* act_blocks, const long* kv_blocks, long act_max,
                        long kv_max, const double* bundle5, int tpb, int* order, int* batch_of, int* n_batches);
/* balance / cost_fb (minibatch.cpp:10-23): out2 = {balance, F_b} */
int hc_cost_fb(long act_mb, long kv_mb, const double* bundle5, int tpb, double* out2);
/* default_packer (sim.cpp:122-132): out2 = {act_max, kv_max} */
int hc_default_packer(double gpu_mem_bytes, const hc_model_config* cfg, long* out2);

/* -------------------------------------------------------------- engine ---
 * The decode path proper: prefill / decode-step calls over the hybrid cache
 * (forward_prompt decoder.cpp:144-157, generation_step 159-174, batched),
 * with the pools, streams and kernels of csrc/engine.hpp. */
typedef struct hc_engine_options {
    int max_batch;           /* requests per decode step */
    int max_seq;             /* max context (0: weights' max_seq) */
    int weights_on_device;   /* 0: weights in pinned host memory, streamed per layer */
    long kv_host_cap, kv_gpu_cap, act_host_cap, act_gpu_cap; /* PoolCaps (cache.hpp:40-45), blocks */
    int kv_on_gpu;
    int host_layers;         /* physical host-pool layer copies (0 = num_layers) */
    int mode;                /* 0 hybrid, 1 kv_only, 2 act_only, 3 token_recompute (SimMode, sim.hpp:21) */
    long alloc_act_host;     /* hybrid-ratio setting: HostAllocation target (plan.hpp:17-25) */
    long alloc_kv_host;
    int scaled;              /* 1/sqrt(head_dim) attention scale (decoder.hpp:28) */
    int max_prefill_tokens;  /* rows per prefill chunk (0: 65536) */
    int device;
    int weight_layers;       /* physical pinned weight layers (0 = num_layers) */
    double recompute_ratio;  /* mode 3 (token_recompute): share of each prompt kept as ids only */
    int arch;                /* 0 reference decoder (decoder.cpp: no bias/LN/residual); 1 OPT (pre-LN,
                              * biases, residuals, final LN; the ACT cache holds LN1(x)). Seeded engines
                              * draw the OPT extras; f64 engines take them from _create_from_f64_opt. */
    void* tp;                /* NULL, or a tensor-parallel rank handle (hc_tp_*): head-sharded variant */
    void* weight_share;      /* NULL, or a group handle (hc_tp_*) of batch-partitioned ranks that share
                              * ONE weight stream: each rank copies 1/N of every layer over its own host
                              * link and an NVLink all-gather completes it (streamed weights only; not
                              * with tp). Every rank must issue the same decode_step sequence. */
} hc_engine_options;

/* ------------------------------------------ tensor parallelism (optional) ---
 * Head-sharded variant of SURVEY.md §8(e): rank g of N owns heads
 * [gH/N, (g+1)H/N) (W_q|W_k|W_v columns, W_proj rows, an FFN slice, its heads'
 * K|V in every KV block) and the ACT/host blocks with pbn % N == g; per layer
 * two all-reduces (compute stream) and one ACT all-gather (copy stream).
 * Every rank is driven with the same request ids / tokens. No reference
 * counterpart (the reference is single-process). */
int hc_tp_nccl_unique_id(uint8_t* out128);
/* NCCL group (one process per GPU): two ids from rank 0, broadcast by the caller. */
int hc_tp_create_nccl(const uint8_t* id_compute128, const uint8_t* id_copy128, int rank, int size, int device,
                      void** tp);
/* In-process group (N engines, one host thread each; tests on one GPU). */
int hc_tp_create_local_group(int size, void** group);
int hc_tp_local_member(void* group, int rank, void** tp); /* owned by the group */
/* Timing stand-in for one rank of a size-N group on one GPU (collectives skipped). */
int hc_tp_create_emulated(int rank, int size, void** tp);
int hc_tp_destroy(void* handle, int is_group);

int hc_engine_create(const hc_model_config* cfg, uint64_t seed, int max_seq, int rescale,
                     const hc_engine_options* opt, void** out);
/* Engine over caller-supplied fp64 reference-layout weights: emb [V x d],
 * pos [max_seq x d], layer_tensors[6*l + {0 q,1 k,2 v,3 proj,4 ffn1,5 ffn2}]. */
int hc_engine_create_from_f64(const hc_model_config* cfg, int max_seq, const double* emb, const double* pos,
                              const double* const* layer_tensors, const hc_engine_options* opt, void** out);
/* Same for arch 1 (OPT): + layer_extras[10*l + {0 b_q,1 b_k,2 b_v,3 b_o [d],4 b_1 [f],5 b_2,6 gamma1,
 * 7 beta1,8 gamma2,9 beta2 [d]}] and final_ln = gamma_f | beta_f [2d]. No reference counterpart. */
int hc_engine_create_from_f64_opt(const hc_model_config* cfg, int max_seq, const double* emb, const double* pos,
                                  const double* const* layer_tensors, const double* const* layer_extras,
                                  const double* final_ln, const hc_engine_options* opt, void** out);
int hc_engine_destroy(void* engine);
/* Prefill n requests; prompt r = tokens[offsets[r] .. offsets[r+1]). */
int hc_engine_prefill(void* engine, int n, const char* const* ids, const int* offsets, const int* tokens);
/* Bookkeeping-only admission + pattern-filled pools (benchmark setup). */
int hc_engine_admit_synthetic(void* engine, int n, const char* const* ids, const int* prompt_lens, uint64_t seed);
/* Mini-batched decode (paper §4.3.3; sim.cpp:258-358; minibatch.cpp:36-83):
 * staging slots of act_max ACT / kv_max KV blocks; each step is packed by
 * form_minibatches on pre-growth block counts, priced by bundle5 = {kv_gen
 * slope, intercept, load_kv slope, intercept, t_load_w}, and run as (layer,
 * mini-batch) units. act_max = kv_max = 0: whole-batch steps. */
int hc_engine_set_minibatching(void* engine, long act_max, long kv_max, const double* bundle5);
/* Recompute fused with decode attention (default on when the heads' width is a
 * multiple of 128): the recompute GEMM (recompute_kv_from_activation,
 * decoder.cpp:123-129) reduces each recomputed block to flash-decoding partials
 * against the step's queries (attention_row, decoder.cpp:15-43) instead of
 * storing K|V in the paged layout. on = 0: K|V written (kKvPaged) and read back
 * by the attention; on < 0: query only. *active (may be NULL) = the path now in use. */
int hc_engine_set_fused_recompute(void* engine, int on, int* active);
/* Pattern-fill every pool slot (benchmark setup, before a real prefill). */
int hc_engine_fill_pools(void* engine, uint64_t seed);
/* Grow each request by n_tokens through the allocator in decode order
 * (sim.cpp:308-310), bookkeeping only (benchmark: timed steps at a later context). */
int hc_engine_advance_synthetic(void* engine, int n, const char* const* ids, int n_tokens);
/* One decode step; x_out [n x d] f16, logits [n x V] fp32, argmax [n]; any may be NULL. */
int hc_engine_decode_step(void* engine, int n, const char* const* ids, const int* tokens, uint16_t* x_out,
                          float* logits, int* argmax);
int hc_engine_free_request(void* engine, const char* id);
/* Drop all requests and rebuild the pools / ratio setting (weights kept). */
int hc_engine_configure_cache(void* engine, long kv_host, long kv_gpu, long act_host, long act_gpu, int kv_on_gpu,
                              int mode, long alloc_act_host, long alloc_kv_host, int host_layers,
                              double recompute_ratio);
/* forward_prompt (decoder.cpp:144-157) of one sequence without cache effects:
 * layer_inputs / k / v [L x n x d], out [n x d] (f16); any may be NULL.
 * token_recompute_kv(ids, layer) (decoder.cpp:131-142) = (k, v)[layer]. */
int hc_engine_forward_trace(void* engine, const int* ids, int n, uint16_t* layer_inputs, uint16_t* k, uint16_t* v,
                            uint16_t* out);
/* One layer of forward_prompt on given input rows x [n x d] (qkv_generate +
 * attention_causal + project_ffn, decoder.cpp:150-153): k, v, out [n x d]. */
int hc_engine_layer_forward(void* engine, int layer, const uint16_t* x, int n, uint16_t* k, uint16_t* v,
                            uint16_t* out);
/* Borrowed HybridCache handle of the engine (use with hc_cache_* read calls). */
int hc_engine_cache(void* engine, void** cache);
/* Payload of one block at one layer (KV [2][H][tpb][hd], ACT [tpb][d]). */
int hc_engine_read_block(void* engine, int kind, int loc, int pbn, int layer, uint16_t* out);
/* Engine-held weights (f16): layer >= 0 packed layer, -1 embedding [V x d],
 * -2 positional [max_seq x d]. */
int hc_engine_read_weights(void* engine, int layer, uint16_t* out);  /* -3: final LN (arch 1) */
int hc_engine_capture_inputs(void* engine, int on);
/* Decode-time layer inputs of the last step, [L][n][d] f16 (n = last batch). */
int hc_engine_captured_inputs(void* engine, uint16_t* out, long count);
/* out17 = {step_ms, h2d_bytes, d2h_bytes, recompute_rows, recompute_ms, attn_ms, gemm_ms, launches,
 *          copy_ms, recompute_launches, store_ms, minibatches, h2d_weights, h2d_kv, h2d_act, d2h_kv,
 *          d2h_act} of the last decode step or prefill (bytes by the reference's traffic classes,
 *          sim.hpp:60-66); the *_ms splits need hc_engine_set_profile(1). */
int hc_engine_last_stats(void* engine, double* out17);
/* Per-kernel CUDA-event timing of the next steps (small overhead). */
int hc_engine_set_profile(void* engine, int on);
/* Replay decode steps as CUDA graphs keyed by their launch structure (default on,
 * HC_DECODE_GRAPHS=0 disables; profiled steps and TP engines run eagerly). */
int hc_engine_set_graphs(void* engine, int on);
/* Events of the last profiled step in the reference's trace.json schema
 * {"events":[{name, track, start_us, end_us, iteration, layer, minibatch}]}
 * (SimEvent, sim.hpp:50-58; main.cpp:263-275). */
int hc_engine_trace_json(void* engine, char* buf, long len, long* needed);
/* Planner calibration on this engine: seconds per layer. */
int hc_engine_time_kv_gen(void* engine, int n_tokens, int reps, double* seconds);
int hc_engine_time_load_kv(void* engine, int n_tokens, int reps, double* seconds);

/* ------------------------------------------------------------- kernels ---
 * Single kernels of the path on host buffers (parity-test boundary). */
/* C = A . W, W passed transposed (Wt [N x K]); epi 0 f16, 1 relu f16, 3 fp32. */
int hc_gemm_f16(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, void* out, int bn);
/* Split-K weight-streaming GEMM (epi 0 / 1), fp32 partials reduced in a second kernel. */
int hc_gemm_f16_splitk(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, uint16_t* out, int bn,
                        int splits);
/* Weight-streaming decode GEMM (swap-AB, stream-K over `ctas` CTAs, 0 = one per SM; M <= 256):
 * C = A . W (+ bias) (+ res), relu for epi 1, fp32 for epi 3 — the M = batch projections of
 * qkv_generate / project_ffn (decoder.cpp:97-121); cut units are summed by a second, dependent kernel. */
int hc_gemm_f16_wstream(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, const uint16_t* bias,
                        const uint16_t* res, void* out, int ctas);
/* Device microseconds per launch of one decode GEMM (M x N x K, epi 0/1/3) over `reps` back-to-back
 * launches with W streamed from HBM; mode 0 tile kernel + split-K, 1 weight-streaming kernel. */
int hc_gemm_bench(int M, int N, int K, int epi, int mode, int reps, double* us_per_call);
/* recompute_kv_from_activation (decoder.cpp:123-129) into the paged layout. */
int hc_recompute_kv_paged(int n_blocks, int tpb, int d, int heads, const uint16_t* act_pool, const uint16_t* wkv_t,
                          const int* tiles, int n_tiles, uint16_t* kv_out, int bn);
/* attention_step over a hybrid block table (decoder.cpp:105-111). */
int hc_decode_attention(int B, int H, int hd, int tpb, const uint16_t* q, const uint16_t* region0, long n0,
                        const uint16_t* region1, long n1, const int* blk_ref, int max_blocks, const int* n_blocks,
                        const int* ctx_len, int scaled, int splits, uint16_t* out);
/* attention_causal (decoder.cpp:55-63) for n_req requests of P tokens. */
int hc_prefill_attention(int n_req, int P, int H, int hd, const uint16_t* qkv, int scaled, uint16_t* out);

#ifdef __cplusplus
}
#endif

#endif /* HYBRIDCACHE_H */
