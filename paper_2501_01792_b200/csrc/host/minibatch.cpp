#include "host/minibatch.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

#include "host/cache.hpp"
#include "host/errors.hpp"

namespace hc {

double balance(long act_mb, long kv_mb, const TimingBundle& b, int tpb) {
    if (act_mb < 0 || kv_mb < 0) throw InputError("balance: negative block count");
    const double recompute = eval(b.t_kv_gen, static_cast<double>(act_mb) * tpb);
    const double load = eval(b.t_load_kv, static_cast<double>(kv_mb) * tpb);
    if (recompute == 0.0 && load == 0.0) return 1.0;
    if (load == 0.0) return std::numeric_limits<double>::infinity();
    return recompute / load;
}

double cost_fb(long act_mb, long kv_mb, const TimingBundle& b, int tpb) {
    const double x = balance(act_mb, kv_mb, b, tpb);
    if (x == 0.0) return std::numeric_limits<double>::infinity();
    return std::max(x, 1.0 / x);
}

std::vector<MiniBatch> form_minibatches(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                        const TimingBundle& b, int tpb) {
    if (cfg.act_max < 1 || cfg.kv_max < 1) throw InputError("form_minibatches: capacities must be >= 1");
    for (const RequestBlocks& r : requests) {
        if (r.act_blocks < 0 || r.kv_blocks < 0)
            throw InputError("form_minibatches: negative block count for request " + r.id);
        if (r.act_blocks > cfg.act_max || r.kv_blocks > cfg.kv_max)
            throw InputError("request too large for GPU buffer capacities: " + r.id);
    }
    // largest first (ties by id), then repeated scans add every request that
    // fits and does not worsen the open batch's cost
    std::vector<size_t> idx(requests.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) {
        const long sx = requests[x].act_blocks + requests[x].kv_blocks;
        const long sy = requests[y].act_blocks + requests[y].kv_blocks;
        return sx != sy ? sx > sy : requests[x].id < requests[y].id;
    });
    std::vector<char> taken(idx.size(), 0);
    size_t left = idx.size();
    std::vector<MiniBatch> out;
    while (left) {
        MiniBatch mb;
        double cost = std::numeric_limits<double>::infinity();
        for (bool grew = true; grew;) {
            grew = false;
            for (size_t k = 0; k < idx.size(); ++k) {
                if (taken[k]) continue;
                const RequestBlocks& r = requests[idx[k]];
                if (mb.act_mb + r.act_blocks > cfg.act_max || mb.kv_mb + r.kv_blocks > cfg.kv_max) continue;
                const double c = cost_fb(mb.act_mb + r.act_blocks, mb.kv_mb + r.kv_blocks, b, tpb);
                if (!mb.ids.empty() && c > cost) continue;
                mb.ids.push_back(r.id);
                mb.act_mb += r.act_blocks;
                mb.kv_mb += r.kv_blocks;
                cost = c;
                taken[k] = 1;
                --left;
                grew = true;
            }
        }
        out.push_back(std::move(mb));
    }
    return out;
}

// Exhaustive partition search (the quality oracle for the greedy packer,
// minibatch.hpp:43-47): every assignment of requests to groups that respect
// the capacities, fewest groups first, then the smallest mean F_b. Groups are
// grown request by request; a branch is cut once it has more groups than the
// best complete partition.
std::vector<MiniBatch> brute_force_pack(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                        const TimingBundle& b, int tpb) {
    if (requests.size() > 10) throw InputError("brute_force_pack: refusing more than 10 requests");
    for (const RequestBlocks& r : requests)
        if (r.act_blocks < 0 || r.kv_blocks < 0 || r.act_blocks > cfg.act_max || r.kv_blocks > cfg.kv_max)
            throw InputError("request too large for GPU buffer capacities: " + r.id);
    if (requests.empty()) return {};
    const size_t n = requests.size();
    std::vector<int> group(n, -1), best;
    std::vector<long> ga, gk;  // per open group: ACT / KV blocks
    size_t best_groups = n + 1;
    double best_mean = std::numeric_limits<double>::infinity();
    auto mean_fb = [&] {
        double s = 0;
        for (size_t g = 0; g < ga.size(); ++g) s += cost_fb(ga[g], gk[g], b, tpb);
        return s / static_cast<double>(ga.size());
    };
    auto dfs = [&](auto&& self, size_t i) -> void {
        if (ga.size() > best_groups) return;
        if (i == n) {
            const double m = mean_fb();
            if (ga.size() < best_groups || m < best_mean) {
                best_groups = ga.size();
                best_mean = m;
                best = group;
            }
            return;
        }
        const RequestBlocks& r = requests[i];
        for (size_t g = 0; g < ga.size(); ++g) {
            if (ga[g] + r.act_blocks > cfg.act_max || gk[g] + r.kv_blocks > cfg.kv_max) continue;
            ga[g] += r.act_blocks;
            gk[g] += r.kv_blocks;
            group[i] = static_cast<int>(g);
            self(self, i + 1);
            ga[g] -= r.act_blocks;
            gk[g] -= r.kv_blocks;
        }
        ga.push_back(r.act_blocks);
        gk.push_back(r.kv_blocks);
        group[i] = static_cast<int>(ga.size()) - 1;
        self(self, i + 1);
        ga.pop_back();
        gk.pop_back();
        group[i] = -1;
    };
    dfs(dfs, 0);
    std::vector<MiniBatch> out(best_groups);
    for (size_t i = 0; i < n; ++i) {
        MiniBatch& mb = out[static_cast<size_t>(best[i])];
        mb.ids.push_back(requests[i].id);
        mb.act_mb += requests[i].act_blocks;
        mb.kv_mb += requests[i].kv_blocks;
    }
    return out;
}

PackerConfig default_packer(double gpu_mem_bytes, const ModelConfig& c) {
    const double kv = static_cast<double>(HybridCache::bytes_of(BlockKind::KV, c));
    const double act = static_cast<double>(HybridCache::bytes_of(BlockKind::ACT, c));
    PackerConfig p;
    p.kv_max = std::max(1L, static_cast<long>(std::floor(0.25 * gpu_mem_bytes / (2.0 * kv))));
    p.act_max = std::max(1L, static_cast<long>(std::floor(0.125 * gpu_mem_bytes / (2.0 * act))));
    return p;
}

}  // namespace hc
