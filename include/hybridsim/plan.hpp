// hybridsim/plan.hpp — the hybrid-ratio planner (plan.hpp:10-65; paper Alg. 1
// + Eq. 8-10) and the per-block ratio rule, through the library's bit-exact
// restatement (hc_initial_cache_allocation, hc_alloc_remaining,
// hc_plan_host_allocation, hc_next_block_kind, hc_planned_times).
#pragma once
#include <utility>

#include <json.hpp>

#include "hybridsim/cache.hpp"
#include "hybridsim/timing.hpp"

namespace hybridsim {

struct GpuResidency {
    long act_gpu = 0;
};

struct HostAllocation {
    long act_host = 0;
    long kv_host = 0;
    long act_init = 0;
    long kv_init = 0;
    long act_remain = 0;
    long kv_remain = 0;

    nlohmann::json to_json() const {
        return nlohmann::json{{"act_host", act_host}, {"kv_host", kv_host},       {"act_init", act_init},
                              {"kv_init", kv_init},   {"act_remain", act_remain}, {"kv_remain", kv_remain}};
    }
    static HostAllocation from_json(const nlohmann::json& j) {
        return HostAllocation{j.at("act_host").get<long>(), j.at("kv_host").get<long>(), j.value("act_init", 0L),
                              j.value("kv_init", 0L), j.value("act_remain", 0L), j.value("kv_remain", 0L)};
    }
};

struct MemoryBudget {  // block sizes are all-layer footprints
    double m_host = 0;
    double s_weight = 0;
    double s_kv_block = 0;
    double s_act_block = 0;
};

namespace b200 {
inline void mem4(const MemoryBudget& m, double o[4]) {
    o[0] = m.m_host;
    o[1] = m.s_weight;
    o[2] = m.s_kv_block;
    o[3] = m.s_act_block;
}
}  // namespace b200

inline MemoryBudget budget_for(const HardwareProfile& profile, const ModelConfig& config, const TimingBundle& bundle) {
    hc_model_config c = config.to_c();
    double o[4];
    b200::check(hc_budget_for(profile.host_mem, &c, static_cast<double>(bundle.s_weight_total), o));
    return MemoryBudget{o[0], o[1], o[2], o[3]};
}

inline std::pair<long, long> initial_cache_allocation(const TimingBundle& bundle, int tokens_per_block,
                                                      GpuResidency act_gpu) {
    double b[5];
    bundle.to_c(b);
    long o[2];
    b200::check(hc_initial_cache_allocation(b, tokens_per_block, act_gpu.act_gpu, o));
    return {o[0], o[1]};
}

inline std::pair<long, long> alloc_remaining(const TimingBundle& bundle, const MemoryBudget& mem, int tokens_per_block,
                                             long act_init, long kv_init) {
    double b[5], m[4];
    bundle.to_c(b);
    b200::mem4(mem, m);
    long o[2];
    b200::check(hc_alloc_remaining(b, m, tokens_per_block, act_init, kv_init, o));
    return {o[0], o[1]};
}

inline HostAllocation plan_host_allocation(const TimingBundle& bundle, const MemoryBudget& mem, int tokens_per_block,
                                           GpuResidency act_gpu) {
    double b[5], m[4];
    bundle.to_c(b);
    b200::mem4(mem, m);
    long o[6];
    b200::check(hc_plan_host_allocation(b, m, tokens_per_block, act_gpu.act_gpu, o));
    return HostAllocation{o[0], o[1], o[2], o[3], o[4], o[5]};
}

inline BlockKind next_block_kind(long act_req, long kv_req, const HostAllocation& allocation) {
    int k = 0;
    b200::check(hc_next_block_kind(act_req, kv_req, allocation.act_host, allocation.kv_host, &k));
    return k ? BlockKind::ACT : BlockKind::KV;
}

namespace b200 {
inline std::pair<double, double> planned_times(const TimingBundle& bundle, int tpb, const HostAllocation& a,
                                               long act_gpu) {
    double b[5], o[2];
    bundle.to_c(b);
    check(hc_planned_times(b, tpb, a.act_host, a.kv_host, act_gpu, o));
    return {o[0], o[1]};
}
}  // namespace b200

inline double planned_t_pcie(const TimingBundle& bundle, int tokens_per_block, const HostAllocation& allocation) {
    return b200::planned_times(bundle, tokens_per_block, allocation, 0).first;
}

inline double planned_t_computation(const TimingBundle& bundle, int tokens_per_block,
                                    const HostAllocation& allocation, GpuResidency act_gpu) {
    return b200::planned_times(bundle, tokens_per_block, allocation, act_gpu.act_gpu).second;
}

}  // namespace hybridsim
