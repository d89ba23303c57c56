// hybridsim/minibatch.hpp — the mini-batch packer (minibatch.hpp:10-47; paper
// §4.3.3) through hc_form_minibatches / hc_brute_force_pack / hc_cost_fb.
// The B200 engine packs its own decode steps with the same function
// (hc_engine_set_minibatching).
#pragma once
#include <string>
#include <vector>

#include "hybridsim/timing.hpp"

namespace hybridsim {

struct RequestBlocks {
    std::string id;
    long act_blocks = 0;
    long kv_blocks = 0;
};

struct MiniBatch {
    std::vector<std::string> ids;
    long act_mb = 0;
    long kv_mb = 0;
};

struct PackerConfig {
    long act_max = 1;
    long kv_max = 1;
};

namespace b200 {
inline std::pair<double, double> balance_fb(long act_mb, long kv_mb, const TimingBundle& bundle, int tpb) {
    double b[5], o[2];
    bundle.to_c(b);
    check(hc_cost_fb(act_mb, kv_mb, b, tpb, o));
    return {o[0], o[1]};
}

using PackFn = int (*)(int, const char* const*, const long*, const long*, long, long, const double*, int, int*,
                       int*, int*);
inline std::vector<MiniBatch> pack(PackFn fn, const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                   const TimingBundle& bundle, int tpb) {
    const int n = static_cast<int>(requests.size());
    std::vector<const char*> ids;
    std::vector<long> a, k;
    for (const RequestBlocks& r : requests) {
        ids.push_back(r.id.c_str());
        a.push_back(r.act_blocks);
        k.push_back(r.kv_blocks);
    }
    std::vector<int> order(n), batch_of(n);
    int nb = 0;
    double b[5];
    bundle.to_c(b);
    check(fn(n, ids.data(), a.data(), k.data(), cfg.act_max, cfg.kv_max, b, tpb, order.data(), batch_of.data(), &nb));
    std::vector<MiniBatch> out(static_cast<size_t>(nb));
    for (int i = 0; i < n; ++i) {  // order lists requests mini-batch by mini-batch, in packing order
        const RequestBlocks& r = requests[static_cast<size_t>(order[i])];
        MiniBatch& mb = out[static_cast<size_t>(batch_of[order[i]])];
        mb.ids.push_back(r.id);
        mb.act_mb += r.act_blocks;
        mb.kv_mb += r.kv_blocks;
    }
    return out;
}
}  // namespace b200

inline double balance(long act_mb, long kv_mb, const TimingBundle& bundle, int tokens_per_block) {
    return b200::balance_fb(act_mb, kv_mb, bundle, tokens_per_block).first;
}

inline double cost_fb(long act_mb, long kv_mb, const TimingBundle& bundle, int tokens_per_block) {
    return b200::balance_fb(act_mb, kv_mb, bundle, tokens_per_block).second;
}

inline std::vector<MiniBatch> form_minibatches(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                               const TimingBundle& bundle, int tokens_per_block) {
    return b200::pack(hc_form_minibatches, requests, cfg, bundle, tokens_per_block);
}

inline std::vector<MiniBatch> brute_force_pack(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                               const TimingBundle& bundle, int tokens_per_block) {
    return b200::pack(hc_brute_force_pack, requests, cfg, bundle, tokens_per_block);
}

}  // namespace hybridsim
