#include "host/plan.hpp"

#include <cmath>
#include <cstdlib>
#include <set>
#include <tuple>

#include "host/errors.hpp"

namespace hc {

LinearTimeModel fit_linear(const std::vector<Sample>& s) {
    const size_t n = s.size();
    if (n < 2) throw InputError("fit_linear: need at least two samples");
    std::set<double> xs;
    for (const Sample& p : s) xs.insert(p.n_tokens);
    if (xs.size() < 2) throw InputError("fit_linear: need at least two distinct n_tokens values");
    // ordinary least squares around the means; negative intercept clamps to 0
    double sum_x = 0, sum_y = 0;
    for (const Sample& p : s) {
        sum_x += p.n_tokens;
        sum_y += p.seconds;
    }
    const double mean_x = sum_x / static_cast<double>(n), mean_y = sum_y / static_cast<double>(n);
    double cxx = 0, cxy = 0;
    for (const Sample& p : s) {
        cxx += (p.n_tokens - mean_x) * (p.n_tokens - mean_x);
        cxy += (p.n_tokens - mean_x) * (p.seconds - mean_y);
    }
    LinearTimeModel m;
    m.slope = cxy / cxx;
    m.intercept = mean_y - m.slope * mean_x;
    if (m.intercept < 0) {
        m.intercept = 0.0;
        m.intercept_clamped = true;
    }
    double res = 0, tot = 0;
    for (const Sample& p : s) {
        const double f = m.slope * p.n_tokens + m.intercept;
        res += (p.seconds - f) * (p.seconds - f);
        tot += (p.seconds - mean_y) * (p.seconds - mean_y);
    }
    m.r_squared = tot == 0.0 ? (res == 0.0 ? 1.0 : 0.0) : 1.0 - res / tot;
    return m;
}

double eval(const LinearTimeModel& m, double n) {
    if (n < 0) throw InputError("eval: negative token count");
    return m.slope * n + m.intercept;
}

long invert(const LinearTimeModel& m, double seconds) {
    if (m.slope <= 0) throw InputError("invert: model is not invertible (slope <= 0)");
    if (seconds < 0) throw InputError("invert: negative time budget");
    long n = static_cast<long>(std::floor((seconds - m.intercept) / m.slope));
    if (n < 0) return 0;
    while (n > 0 && eval(m, static_cast<double>(n)) > seconds) --n;  // never overshoot
    return n;
}

WeightBytes weight_bytes(const ModelConfig& c) {
    const uint64_t d = c.hidden_dim, f = c.ffn_dim, bps = c.bytes_per_scalar;
    WeightBytes w;
    w.per_layer = (4 * d * d + 2 * d * f) * bps;
    w.total = w.per_layer * static_cast<uint64_t>(c.num_layers) + static_cast<uint64_t>(c.vocab_size) * d * bps;
    return w;
}

TimingBundle bundle_from_samples(const std::vector<Sample>& kv_gen, const std::vector<Sample>& load_kv,
                                 double link_bytes_per_s, const ModelConfig& c) {
    if (link_bytes_per_s <= 0) throw InputError("bundle_from_samples: link bandwidth must be positive");
    TimingBundle b;
    b.t_kv_gen = fit_linear(kv_gen);
    b.t_load_kv = fit_linear(load_kv);
    const WeightBytes w = weight_bytes(c);
    b.s_weight_layer = w.per_layer;
    b.s_weight_total = w.total;
    b.t_load_w = static_cast<double>(w.per_layer) / link_bytes_per_s;
    return b;
}

MemoryBudget budget_for(double host_mem, const ModelConfig& c, const TimingBundle& b) {
    MemoryBudget m;
    m.m_host = host_mem;
    m.s_weight = static_cast<double>(b.s_weight_total);
    m.s_kv_block = static_cast<double>(HybridCache::bytes_of(BlockKind::KV, c)) * c.num_layers;
    m.s_act_block = static_cast<double>(HybridCache::bytes_of(BlockKind::ACT, c)) * c.num_layers;
    return m;
}

namespace {
// largest n with n * block <= avail, settled exactly after the division
long blocks_fitting(double avail, double block) {
    if (avail <= 0 || block <= 0) return 0;
    long n = static_cast<long>(std::floor(avail / block));
    while (n > 0 && static_cast<double>(n) * block > avail) --n;
    while (static_cast<double>(n + 1) * block <= avail) ++n;
    return n;
}
}  // namespace

std::pair<long, long> initial_cache_allocation(const TimingBundle& b, int tpb, long act_gpu) {
    if (tpb < 1) throw InputError("initial_cache_allocation: bad block size");
    if (act_gpu < 0) throw InputError("initial_cache_allocation: negative ACT_GPU");
    // idle link time left after the GPU-resident ACT recompute
    const double slack = b.t_load_w - eval(b.t_kv_gen, static_cast<double>(act_gpu) * tpb);
    if (slack >= 0) {
        if (b.t_kv_gen.slope > 0) return {invert(b.t_kv_gen, slack) / tpb, 0};
        return {0, 0};
    }
    if (b.t_load_kv.slope > 0) return {0, invert(b.t_load_kv, -slack) / tpb};
    return {0, 0};
}

std::pair<long, long> alloc_remaining(const TimingBundle& b, const MemoryBudget& mem, int tpb, long act_init,
                                      long kv_init) {
    if (mem.s_kv_block <= 0 || mem.s_act_block <= 0)
        throw InputError("alloc_remaining: block sizes must be positive");
    const double used = mem.s_act_block * static_cast<double>(act_init) + mem.s_kv_block * static_cast<double>(kv_init);
    const double left = mem.m_host - mem.s_weight - used;
    if (left < 0) throw CapacityError("alloc_remaining: host memory cannot hold weights plus initial blocks");
    const double bt = static_cast<double>(tpb);
    const double act_s = b.t_kv_gen.slope * bt, kv_s = b.t_load_kv.slope * bt;
    const double act_i = b.t_kv_gen.intercept, kv_i = b.t_load_kv.intercept;
    // balance: act_i + act_s*x == kv_i + kv_s*y  with  s_act*x + s_kv*y == left
    const double denom = act_s * mem.s_kv_block + kv_s * mem.s_act_block;
    if (denom <= 0) return {0, static_cast<long>(std::floor(left / mem.s_kv_block))};
    const double x = (kv_s * left + mem.s_kv_block * (kv_i - act_i)) / denom;
    if (x < 0) return {0, blocks_fitting(left, mem.s_kv_block)};
    const double y = (left - mem.s_act_block * x) / mem.s_kv_block;
    if (y < 0) return {blocks_fitting(left, mem.s_act_block), 0};
    const long xi = static_cast<long>(std::floor(x + 1e-9 * (1.0 + std::abs(x))));
    return {xi, blocks_fitting(left - mem.s_act_block * static_cast<double>(xi), mem.s_kv_block)};
}

double planned_t_pcie(const TimingBundle& b, int tpb, const HostAllocation& a) {
    return b.t_load_w + eval(b.t_load_kv, static_cast<double>(a.kv_host) * tpb);
}

double planned_t_computation(const TimingBundle& b, int tpb, const HostAllocation& a, long act_gpu) {
    return eval(b.t_kv_gen, static_cast<double>(a.act_host + act_gpu) * tpb);
}

HostAllocation plan_host_allocation(const TimingBundle& b, const MemoryBudget& mem, int tpb, long act_gpu) {
    HostAllocation a;
    std::tie(a.act_init, a.kv_init) = initial_cache_allocation(b, tpb, act_gpu);
    std::tie(a.act_remain, a.kv_remain) = alloc_remaining(b, mem, tpb, a.act_init, a.kv_init);
    a.act_host = a.act_init + a.act_remain;
    a.kv_host = a.kv_init + a.kv_remain;

    // exact discrete minimiser of |t_pcie - t_comp| on the memory frontier;
    // the signed gap decreases strictly with the ACT count -> binary search
    const double avail = mem.m_host - mem.s_weight;
    auto kv_on_frontier = [&](long x) { return blocks_fitting(avail - mem.s_act_block * static_cast<double>(x), mem.s_kv_block); };
    auto gap = [&](long x) {
        HostAllocation c = a;
        c.act_host = x;
        c.kv_host = kv_on_frontier(x);
        return planned_t_pcie(b, tpb, c) - planned_t_computation(b, tpb, c, act_gpu);
    };
    const long x_max = blocks_fitting(avail, mem.s_act_block);
    long best;
    if (gap(0) <= 0) {
        best = 0;
    } else if (gap(x_max) >= 0) {
        best = x_max;
    } else {
        long lo = 0, hi = x_max;
        while (hi - lo > 1) {
            const long mid = lo + (hi - lo) / 2;
            if (gap(mid) > 0)
                lo = mid;
            else
                hi = mid;
        }
        best = std::abs(gap(lo)) <= std::abs(gap(hi)) ? lo : hi;
    }
    a.act_host = best;
    a.kv_host = kv_on_frontier(best);
    a.act_remain = a.act_host - a.act_init;
    a.kv_remain = a.kv_host - a.kv_init;
    return a;
}

double flop_count(int kind, const ModelConfig& c, long n_tokens, int k) {
    if (n_tokens < 0) throw InputError("flop_count: negative token count");
    const double n = static_cast<double>(n_tokens), d = c.hidden_dim, f = c.ffn_dim;
    switch (kind) {
        case 0: return 2.0 * (2.0 * n * d * d);                    // K,V from activations
        case 1: return 2.0 * (3.0 * n * d * d);                    // Q,K,V
        case 2: return 2.0 * d * n * (n + 1.0);                    // causal attention
        case 3: return 2.0 * (n * d * d + 2.0 * n * d * f);        // proj + FFN
        case 5: return flop_count(1, c, n_tokens) + flop_count(2, c, n_tokens) + flop_count(3, c, n_tokens);
        case 4:
            if (k < 0 || k >= c.num_layers) throw InputError("flop_count: layer index out of range");
            return static_cast<double>(k) * flop_count(5, c, n_tokens) + flop_count(1, c, n_tokens);
    }
    throw InputError("flop_count: unknown op kind");
}

double attention_step_flops(const ModelConfig& c, long ctx) {
    return 4.0 * static_cast<double>(c.hidden_dim) * static_cast<double>(ctx);
}

HbmPlan plan_hbm_residency(const ModelConfig& c, long requests, long blocks_per_request, double hbm_bytes) {
    if (requests < 1 || blocks_per_request < 1) throw InputError("plan_hbm_residency: empty workload");
    if (hbm_bytes <= 0) throw InputError("plan_hbm_residency: no device memory");
    const double L = c.num_layers;
    const double kv_one = static_cast<double>(HybridCache::bytes_of(BlockKind::KV, c));
    const double kv_all = kv_one * L, act_all = static_cast<double>(HybridCache::bytes_of(BlockKind::ACT, c)) * L;
    const long N = requests * blocks_per_request;
    HbmPlan p;
    // x ACT blocks (+ x recompute slots) and N - x KV blocks within hbm_bytes
    const double x_exact = (N * kv_all - hbm_bytes) / (kv_all - act_all - kv_one);
    const long x_fit = x_exact <= 0 ? 0 : static_cast<long>(std::ceil(x_exact));
    p.act_share = x_fit == 0 ? 0.0 : std::min(1.0, static_cast<double>(x_fit + requests) / N);
    const double r = p.act_share;
    // per-kind capacities with one block of slack per request (block-boundary rounding)
    const long act_need = r <= 0 ? 0 : (r >= 1 ? N : requests * (static_cast<long>(std::ceil(r * blocks_per_request)) + 1));
    const long kv_need = r >= 1 ? 0 : (r <= 0 ? N : requests * (static_cast<long>(std::ceil((1 - r) * blocks_per_request)) + 1));
    const long act_gpu = static_cast<long>(
        std::min<double>(act_need, std::floor(hbm_bytes / (act_all + kv_one))));
    const double room = hbm_bytes - act_gpu * (act_all + kv_one) - 2.0 * kv_need * kv_one;
    const long kv_gpu = static_cast<long>(std::max(0.0, std::min<double>(kv_need, std::floor(room / (kv_all - 2 * kv_one)))));
    p.act_gpu = act_gpu;
    p.act_host = act_need - act_gpu;
    p.kv_gpu = kv_gpu;
    p.kv_host = kv_need - kv_gpu;
    return p;
}

HbmTierPlan plan_hbm_tiers(const ModelConfig& c, long requests, long blocks_per_request, double hbm_bytes,
                           const TimingBundle& b, double host_bytes, bool weights_streamed) {
    if (requests < 1 || blocks_per_request < 1) throw InputError("plan_hbm_tiers: empty workload");
    if (hbm_bytes <= 0) throw InputError("plan_hbm_tiers: no device memory");
    if (host_bytes < 0) throw InputError("plan_hbm_tiers: negative host budget");
    const double L = c.num_layers, tpb = c.tokens_per_block, B = static_cast<double>(requests);
    const double kv_one = static_cast<double>(HybridCache::bytes_of(BlockKind::KV, c));
    const double act_one = static_cast<double>(HybridCache::bytes_of(BlockKind::ACT, c));
    const double kv_all = kv_one * L, act_all = act_one * L;
    const long N = requests * blocks_per_request;
    auto t_comp = [&](long x) { return x > 0 ? eval(b.t_kv_gen, static_cast<double>(x) * tpb) : 0.0; };
    const double t_w = weights_streamed ? b.t_load_w : 0.0;
    auto t_link = [&](long z) { return t_w + (z > 0 ? eval(b.t_load_kv, static_cast<double>(z) * tpb) : 0.0); };
    HbmTierPlan best;
    double best_t = -1;
    for (long x = 0; x <= N; ++x) {
        // x ACT/gpu blocks + recompute slots (x + B spill), KV staging for z + B host blocks,
        // ACT staging for the B spill blocks, y KV/gpu blocks
        const double rhs = hbm_bytes - x * (act_all + kv_one) - B * kv_one - 2.0 * (N - x + B) * kv_one -
                           2.0 * B * act_one;
        if (rhs < 0) break;  // rhs falls with x: an ACT block (all layers) outweighs the staging slot it saves
        const long y = std::min<long>(N - x, static_cast<long>(std::floor(rhs / (kv_all - 2 * kv_one))));
        const long z = N - x - std::max<long>(y, 0);
        if (host_bytes > 0) {  // pinned host tiers: KV host blocks (+ slack) and the ACT spill blocks
            const double slack = x > 0 && x < N ? B : 0.0;
            if ((z + slack) * kv_all + slack * act_all > host_bytes) continue;
        }
        const double t = std::max(t_comp(x), t_link(z));
        if (best_t < 0 || t < best_t) {
            best_t = t;
            best.act_share = static_cast<double>(x) / N;
            best.act_gpu = x;
            best.act_host = x > 0 && x < N ? requests : 0;
            best.kv_gpu = std::max<long>(y, 0);
            best.kv_host = z + (x > 0 && x < N ? requests : 0);  // slack only where the ratio rounds
            best.t_comp = t_comp(x);
            best.t_link = t_link(z);
        }
    }
    if (best_t < 0)
        throw CapacityError("plan_hbm_tiers: device and host memory cannot hold the workload and its staging");
    return best;
}

HostStepPlan plan_host_min_step(const ModelConfig& c, long requests, long blocks_per_request, const TimingBundle& b,
                                double host_bytes) {
    if (requests < 1 || blocks_per_request < 1) throw InputError("plan_host_min_step: empty workload");
    if (host_bytes < 0) throw InputError("plan_host_min_step: negative host budget");
    const double L = c.num_layers, tpb = c.tokens_per_block, B = static_cast<double>(requests);
    const double kv_one = static_cast<double>(HybridCache::bytes_of(BlockKind::KV, c));
    const double act_one = static_cast<double>(HybridCache::bytes_of(BlockKind::ACT, c));
    const double ratio = act_one / kv_one;  // link cost of an ACT token in KV tokens
    const long N = requests * blocks_per_request;
    HostStepPlan best;
    double best_t = -1;
    for (long x = 0; x <= N; ++x) {
        const double slack = x > 0 && x < N ? B : 0.0;
        if (host_bytes > 0 && ((N - x + slack) * kv_one + (x + slack) * act_one) * L > host_bytes) continue;
        const double tc = x > 0 ? eval(b.t_kv_gen, static_cast<double>(x) * tpb) : 0.0;
        const double tl = b.t_load_w + eval(b.t_load_kv, (static_cast<double>(N - x) + x * ratio) * tpb);
        const double t = std::max(tc, tl);
        if (best_t < 0 || t < best_t) {
            best_t = t;
            best.act_share = static_cast<double>(x) / N;
            best.act_host = x + static_cast<long>(slack);
            best.kv_host = N - x + static_cast<long>(slack);
            best.t_comp = tc;
            best.t_link = tl;
        }
    }
    if (best_t < 0) throw CapacityError("plan_host_min_step: pinned host memory cannot hold the workload");
    return best;
}

}  // namespace hc
