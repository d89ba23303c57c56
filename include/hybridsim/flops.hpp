// hybridsim/flops.hpp — flop_count (flops.hpp:8-24) through hc_flop_count.
#pragma once
#include "hybridsim/model.hpp"

namespace hybridsim {

enum class FlopKind { KvGen, QkvGen, Attention, ProjFfn, TokenRecomputeToLayerK, FullLayer };

inline double flop_count(FlopKind kind, const ModelConfig& config, long n_tokens, int k = 0) {
    hc_model_config c = config.to_c();
    double v = 0.0;
    b200::check(hc_flop_count(static_cast<int>(kind), &c, n_tokens, k, &v));
    return v;
}

// one decode query over ctx_len cached tokens (flops.cpp:35-37): 4 d ctx
inline double attention_step_flops(const ModelConfig& config, long ctx_len) {
    return 4.0 * config.hidden_dim * static_cast<double>(ctx_len);
}

}  // namespace hybridsim
