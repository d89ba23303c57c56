// hybridsim/model.hpp — ModelConfig (model.hpp:15-36) over the C ABI:
// validate / preset run the library's checks (hc_model_validate,
// hc_model_preset), so errors and presets are the reference's.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <json.hpp>

#include "hybridsim/errors.hpp"

namespace hybridsim {

struct ModelConfig {
    std::string name = "custom";
    int num_layers = 1;
    int hidden_dim = 64;
    int num_heads = 1;
    int ffn_dim = 0;  // 0: 4 * hidden_dim (filled by validate)
    int vocab_size = 256;
    int tokens_per_block = 16;
    int bytes_per_scalar = 2;
    std::uint64_t seed = 0;

    int head_dim() const { return hidden_dim / num_heads; }

    hc_model_config to_c() const {
        return hc_model_config{num_layers, hidden_dim, num_heads, ffn_dim, vocab_size, tokens_per_block,
                               bytes_per_scalar};
    }
    void validate() {
        hc_model_config c = to_c();
        b200::check(hc_model_validate(&c));
        ffn_dim = c.ffn_dim;
    }
    static ModelConfig preset(const std::string& name) {
        hc_model_config c{};
        b200::check(hc_model_preset(name.c_str(), &c));
        ModelConfig m;
        m.name = name;
        m.num_layers = c.num_layers;
        m.hidden_dim = c.hidden_dim;
        m.num_heads = c.num_heads;
        m.ffn_dim = c.ffn_dim;
        m.vocab_size = c.vocab_size;
        m.tokens_per_block = c.tokens_per_block;
        m.bytes_per_scalar = c.bytes_per_scalar;
        return m;
    }
    static const std::vector<std::string>& preset_names() {
        static const std::vector<std::string> n = {"opt-6.7b", "opt-13b", "opt-30b", "opt-66b"};
        return n;
    }
    static ModelConfig from_json(const nlohmann::json& j) {
        ModelConfig c = j.contains("preset") ? preset(j.at("preset").get<std::string>()) : ModelConfig{};
        auto take = [&](const char* k, auto& field) {
            if (j.contains(k)) field = j.at(k).get<std::decay_t<decltype(field)>>();
        };
        take("name", c.name);
        take("num_layers", c.num_layers);
        take("hidden_dim", c.hidden_dim);
        take("num_heads", c.num_heads);
        take("ffn_dim", c.ffn_dim);
        take("vocab_size", c.vocab_size);
        take("tokens_per_block", c.tokens_per_block);
        take("bytes_per_scalar", c.bytes_per_scalar);
        take("seed", c.seed);
        c.validate();
        return c;
    }
    nlohmann::json to_json() const {
        return nlohmann::json{{"name", name},         {"num_layers", num_layers},
                              {"hidden_dim", hidden_dim}, {"num_heads", num_heads},
                              {"ffn_dim", ffn_dim},   {"vocab_size", vocab_size},
                              {"tokens_per_block", tokens_per_block},
                              {"bytes_per_scalar", bytes_per_scalar}, {"seed", seed}};
    }
};

}  // namespace hybridsim
