// hybridsim/timing.hpp — the planner's timing models (timing.hpp:10-86):
// fit_linear and bundle_from_samples run in the library (hc_fit_linear,
// hc_bundle_from_samples: the same OLS the B200 engine's measured samples go
// through); the analytic sample synthesis of the reference's simulator
// (timing.cpp:75-103) is restated here for callers that calibrate from a
// HardwareProfile instead of measuring.
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

#include <json.hpp>

#include "hybridsim/flops.hpp"
#include "hybridsim/rng.hpp"

namespace hybridsim {

struct HardwareProfile {
    double pcie_bandwidth = 25e9;
    double gpu_throughput = 82.6e12;
    double gpu_efficiency = 0.35;
    double host_mem = 882e9;
    double gpu_mem = 24e9;
    double noise_std = 0.0;

    double effective_flops() const { return gpu_throughput * gpu_efficiency; }
    void validate() const {
        if (!(pcie_bandwidth > 0 && gpu_throughput > 0 && gpu_efficiency > 0 && host_mem > 0 && gpu_mem > 0))
            throw InputError("HardwareProfile: all rates and capacities must be positive");
        if (gpu_efficiency > 1.0) throw InputError("HardwareProfile: gpu_efficiency must be <= 1");
        if (noise_std < 0) throw InputError("HardwareProfile: noise_std must be >= 0");
    }
    static HardwareProfile from_json(const nlohmann::json& j) {
        HardwareProfile p;
        for (auto [k, f] : {std::pair<const char*, double*>{"pcie_bandwidth", &p.pcie_bandwidth},
                            {"gpu_throughput", &p.gpu_throughput}, {"gpu_efficiency", &p.gpu_efficiency},
                            {"host_mem", &p.host_mem}, {"gpu_mem", &p.gpu_mem}, {"noise_std", &p.noise_std}})
            if (j.contains(k)) *f = j.at(k).get<double>();
        p.validate();
        return p;
    }
    nlohmann::json to_json() const {
        return nlohmann::json{{"pcie_bandwidth", pcie_bandwidth}, {"gpu_throughput", gpu_throughput},
                              {"gpu_efficiency", gpu_efficiency}, {"host_mem", host_mem},
                              {"gpu_mem", gpu_mem}, {"noise_std", noise_std}};
    }
};

struct LinearTimeModel {  // seconds(n) = slope * n + intercept
    double slope = 0.0;
    double intercept = 0.0;
    double r_squared = 0.0;
    bool intercept_clamped = false;
};

struct Sample {
    double n_tokens = 0.0;
    double seconds = 0.0;
};

inline LinearTimeModel fit_linear(const std::vector<Sample>& samples) {
    std::vector<double> n, s;
    for (const Sample& x : samples) {
        n.push_back(x.n_tokens);
        s.push_back(x.seconds);
    }
    double o[4];
    b200::check(hc_fit_linear(n.data(), s.data(), static_cast<int>(n.size()), o));
    return LinearTimeModel{o[0], o[1], o[2], o[3] != 0.0};
}

enum class SampleKind { KvGen, LoadKv };

// analytic time of n tokens (recompute FLOPs at the effective rate, or one
// layer's K|V bytes over the link), times (1 + eps), eps ~ N(0, noise_std)
// from the (seed, kind) stream; n log-spaced over [lo, hi]
inline std::vector<Sample> synthesize_samples(const HardwareProfile& profile, const ModelConfig& config,
                                              SampleKind kind, int n_points, std::uint64_t seed,
                                              double lo_tokens = 64.0, double hi_tokens = 65536.0) {
    profile.validate();
    if (n_points < 2) throw InputError("synthesize_samples: n_points must be >= 2");
    SplitMix64 rng(mix_seed(seed, kind == SampleKind::KvGen ? 0x6b76 : 0x6c64));
    const double kv_bytes_per_token = 2.0 * config.hidden_dim * config.bytes_per_scalar;
    std::vector<Sample> out;
    for (int i = 0; i < n_points; ++i) {
        const double n = std::floor(lo_tokens * std::pow(hi_tokens / lo_tokens, static_cast<double>(i) / (n_points - 1)));
        double t = kind == SampleKind::KvGen
                       ? flop_count(FlopKind::KvGen, config, static_cast<long>(n)) / profile.effective_flops()
                       : n * kv_bytes_per_token / profile.pcie_bandwidth;
        t *= 1.0 + rng.normal(0.0, profile.noise_std);
        out.push_back(Sample{n, t});
    }
    return out;
}

inline double eval(const LinearTimeModel& m, double n_tokens) {
    if (n_tokens < 0) throw InputError("eval: negative token count");
    return m.slope * n_tokens + m.intercept;
}

inline long invert(const LinearTimeModel& m, double seconds) {  // largest n with eval(n) <= seconds
    if (m.slope <= 0) throw InputError("invert: model is not invertible (slope <= 0)");
    if (seconds < 0) throw InputError("invert: negative time budget");
    long n = static_cast<long>(std::floor((seconds - m.intercept) / m.slope));
    if (n < 0) return 0;
    while (n > 0 && eval(m, static_cast<double>(n)) > seconds) --n;
    return n;
}

struct WeightBytes {
    std::uint64_t per_layer = 0;
    std::uint64_t total = 0;
};

inline WeightBytes weight_bytes(const ModelConfig& config) {
    hc_model_config c = config.to_c();
    std::uint64_t o[2];
    b200::check(hc_weight_bytes(&c, o));
    return WeightBytes{o[0], o[1]};
}

struct TimingBundle {
    LinearTimeModel t_kv_gen;
    LinearTimeModel t_load_kv;
    double t_load_w = 0.0;
    std::uint64_t s_weight_layer = 0;
    std::uint64_t s_weight_total = 0;

    nlohmann::json to_json() const {
        auto m = [](const LinearTimeModel& x) {
            return nlohmann::json{{"slope", x.slope}, {"intercept", x.intercept}, {"r2", x.r_squared},
                                  {"intercept_clamped", x.intercept_clamped}};
        };
        return nlohmann::json{{"kv_gen", m(t_kv_gen)}, {"load_kv", m(t_load_kv)}, {"t_load_w", t_load_w},
                              {"s_weight_layer", s_weight_layer}, {"s_weight_total", s_weight_total}};
    }
    static TimingBundle from_json(const nlohmann::json& j) {
        auto m = [](const nlohmann::json& x) {
            return LinearTimeModel{x.at("slope").get<double>(), x.at("intercept").get<double>(),
                                   x.value("r2", 0.0), x.value("intercept_clamped", false)};
        };
        TimingBundle b;
        b.t_kv_gen = m(j.at("kv_gen"));
        b.t_load_kv = m(j.at("load_kv"));
        b.t_load_w = j.at("t_load_w").get<double>();
        b.s_weight_layer = j.at("s_weight_layer").get<std::uint64_t>();
        b.s_weight_total = j.value("s_weight_total", std::uint64_t{0});
        return b;
    }
    // {kv slope, kv intercept, load slope, load intercept, t_load_w} (hybridcache.h bundle5)
    void to_c(double out5[5]) const {
        out5[0] = t_kv_gen.slope;
        out5[1] = t_kv_gen.intercept;
        out5[2] = t_load_kv.slope;
        out5[3] = t_load_kv.intercept;
        out5[4] = t_load_w;
    }
};

inline TimingBundle bundle_from_samples(const std::vector<Sample>& kv_gen, const std::vector<Sample>& load_kv,
                                        const HardwareProfile& profile, const ModelConfig& config) {
    std::vector<double> kn, ks, ln, ls;
    for (const Sample& x : kv_gen) {
        kn.push_back(x.n_tokens);
        ks.push_back(x.seconds);
    }
    for (const Sample& x : load_kv) {
        ln.push_back(x.n_tokens);
        ls.push_back(x.seconds);
    }
    hc_model_config c = config.to_c();
    double o[11];
    b200::check(hc_bundle_from_samples(kn.data(), ks.data(), static_cast<int>(kn.size()), ln.data(), ls.data(),
                                       static_cast<int>(ln.size()), profile.pcie_bandwidth, &c, o));
    TimingBundle b;
    b.t_kv_gen = LinearTimeModel{o[0], o[1], o[2], o[3] != 0.0};
    b.t_load_kv = LinearTimeModel{o[4], o[5], o[6], o[7] != 0.0};
    b.t_load_w = o[8];
    b.s_weight_layer = static_cast<std::uint64_t>(o[9]);
    b.s_weight_total = static_cast<std::uint64_t>(o[10]);
    return b;
}

inline TimingBundle calibrate(const HardwareProfile& profile, const ModelConfig& config, std::uint64_t seed,
                              int n_points = 16) {
    return bundle_from_samples(synthesize_samples(profile, config, SampleKind::KvGen, n_points, seed),
                               synthesize_samples(profile, config, SampleKind::LoadKv, n_points, seed), profile,
                               config);
}

}  // namespace hybridsim
