// Hybrid-ratio planner (north-star (5)): the paper's cost model (Alg. 1,
// Eq. 8-11) fed by MEASURED B200 samples — recompute-GEMM seconds vs ACT
// tokens and host-link seconds vs KV tokens — instead of the reference's
// synthetic ones.
//
// Reference: timing.hpp:15-88 / timing.cpp:38-183 (fit, eval, invert,
// weight bytes, bundle), plan.hpp:17-65 / plan.cpp:41-177 (budget, two-step
// allocation, frontier polish), flops.cpp:7-37 (FLOP model).
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

#include "host/cache.hpp"
#include "host/model.hpp"

namespace hc {

struct Sample {
    double n_tokens = 0.0;
    double seconds = 0.0;
};

struct LinearTimeModel {
    double slope = 0.0;
    double intercept = 0.0;
    double r_squared = 0.0;
    bool intercept_clamped = false;
};

LinearTimeModel fit_linear(const std::vector<Sample>& samples);
double eval(const LinearTimeModel& m, double n_tokens);
long invert(const LinearTimeModel& m, double seconds);

struct WeightBytes {
    uint64_t per_layer = 0;
    uint64_t total = 0;
};
WeightBytes weight_bytes(const ModelConfig& c);

struct TimingBundle {
    LinearTimeModel t_kv_gen;   // seconds vs ACT tokens recomputed, per layer
    LinearTimeModel t_load_kv;  // seconds vs KV tokens loaded, per layer
    double t_load_w = 0.0;      // seconds per layer of weights over the host link
    uint64_t s_weight_layer = 0;
    uint64_t s_weight_total = 0;
};

TimingBundle bundle_from_samples(const std::vector<Sample>& kv_gen, const std::vector<Sample>& load_kv,
                                 double link_bytes_per_s, const ModelConfig& c);

struct MemoryBudget {
    double m_host = 0;
    double s_weight = 0;
    double s_kv_block = 0;   // all-layer footprint of one KV block
    double s_act_block = 0;  // all-layer footprint of one ACT block
};
MemoryBudget budget_for(double host_mem, const ModelConfig& c, const TimingBundle& b);

std::pair<long, long> initial_cache_allocation(const TimingBundle& b, int tpb, long act_gpu);
std::pair<long, long> alloc_remaining(const TimingBundle& b, const MemoryBudget& mem, int tpb, long act_init,
                                      long kv_init);
HostAllocation plan_host_allocation(const TimingBundle& b, const MemoryBudget& mem, int tpb, long act_gpu);
double planned_t_pcie(const TimingBundle& b, int tpb, const HostAllocation& a);
double planned_t_computation(const TimingBundle& b, int tpb, const HostAllocation& a, long act_gpu);

// HBM residency (B200 extension of Alg. 1; no reference counterpart): the
// blocks of `requests` x `blocks_per_request` context blocks placed on the GPU
// first (kv_on_gpu, cache.cpp:64-91) within `hbm_bytes`. With the cache in
// HBM there is no link time to hide recompute under, so every KV block that
// fits saves 4 d^2 tpb FLOPs per layer per step: the planned ACT share is the
// smallest one whose blocks fit (0 when all-KV fits). Each ACT block also
// needs a recompute slot (one layer of a KV block); blocks that do not fit
// stay in pinned host memory (KV, streamed through two staging slots).
struct HbmPlan {
    double act_share = 0;         // r: HostAllocation target act / (act + kv)
    long act_gpu = 0, kv_gpu = 0;  // pool capacities (blocks)
    long act_host = 0, kv_host = 0;
};
HbmPlan plan_hbm_residency(const ModelConfig& c, long requests, long blocks_per_request, double hbm_bytes);

// Balanced three-tier plan (B200 extension of Alg. 1's balance, Eq. 10): x ACT
// blocks in HBM (recomputed each step), y KV blocks in HBM, z KV blocks in
// pinned host memory streamed per layer. Over all x, y is the most KV that
// still fits next to x ACT blocks, their recompute slots and the staging slots
// of the z host blocks; the plan minimises the per-layer critical path
// max(t_kv_gen(x tpb), t_load_kv(z tpb)) from the MEASURED bundle — with
// weights resident the link is otherwise idle, so streaming some KV from host
// while the tensor cores recompute beats recomputing it. Capacities add one
// block of slack per request (ACT spill to host, KV host) for block-boundary
// rounding of the ratio. t_comp / t_link are the predicted per-layer times.
// host_bytes (> 0) bounds the pinned host memory of the host tiers (KV host
// blocks, all layers, plus the ACT spill blocks); 0 = unbounded.
// weights_streamed: the weights stay in pinned host memory and cross the link
// every layer (hbm_bytes then excludes only their two streaming slots), so the
// link side of the critical path is t_load_w + t_load_kv(z tpb): recompute is
// free up to the weight stream's time, KV blocks fill the remaining HBM.
struct HbmTierPlan : HbmPlan {
    double t_comp = 0, t_link = 0;
};
HbmTierPlan plan_hbm_tiers(const ModelConfig& c, long requests, long blocks_per_request, double hbm_bytes,
                           const TimingBundle& b, double host_bytes = 0, bool weights_streamed = false);

// Host-only plan minimising the predicted step (B200 extension of Alg. 1).
// Alg. 1's t_pcie (planned_t_pcie, plan.cpp:166-168) prices the weights and
// the KV host blocks only, but an ACT host block crosses the link too (d*2
// bytes per token against the KV block's 2*d*2). While recompute is cheap
// against the link — the B200 case: the recompute GEMM of a whole OPT-30B
// context takes a quarter of its ACT transfer — that term decides the ratio.
// Over x ACT blocks of the N = requests * blocks_per_request host blocks:
//   t_link(x) = t_load_w + t_load_kv((N - x) tpb + x tpb s_act / s_kv)
//   t_comp(x) = t_kv_gen(x tpb)
// minimise max(t_link, t_comp) per layer with the pinned host tiers
// ((N - x) KV + x ACT blocks, all layers, + one block of rounding slack per
// request of each kind for 0 < x < N) inside host_bytes (0 = unbounded).
struct HostStepPlan {
    double act_share = 0;  // r = x / N
    long act_host = 0, kv_host = 0;  // pool capacities (blocks)
    double t_comp = 0, t_link = 0;   // predicted per-layer seconds
};
HostStepPlan plan_host_min_step(const ModelConfig& c, long requests, long blocks_per_request, const TimingBundle& b,
                                double host_bytes = 0);

// FLOP model (flops.cpp:7-37); kinds: 0 KvGen, 1 QkvGen, 2 Attention,
// 3 ProjFfn, 4 TokenRecomputeToLayerK, 5 FullLayer.
double flop_count(int kind, const ModelConfig& c, long n_tokens, int k = 0);
double attention_step_flops(const ModelConfig& c, long ctx);

}  // namespace hc
