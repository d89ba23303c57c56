// Model configuration and synthetic weights (reference: model.hpp:15-58,
// model.cpp:8-117, rng.hpp:10-49).
//
// Weights are drawn exactly as the reference draws them (one SplitMix64
// stream per tensor, U(-0.1, 0.1), identical tags), then rescaled per tensor
// (the reference init has no LayerNorm / residual and blows
// up ~10x per layer) and rounded to bf16. Device layout is transposed
// ([out][in], K-major) for the tcgen05 GEMM:
//   layer l: Wqkv^T [3d x d] | Wproj^T [d x d] | W1^T [f x d] | W2^T [d x f]
// packed contiguously so one copy streams a whole layer.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace hc {

struct ModelConfig {
    std::string name = "custom";
    int num_layers = 1;
    int hidden_dim = 64;
    int num_heads = 1;
    int ffn_dim = 0;  // 0 -> 4 * hidden_dim
    int vocab_size = 256;
    int tokens_per_block = 16;
    int bytes_per_scalar = 2;
    uint64_t seed = 0;

    int head_dim() const { return hidden_dim / num_heads; }
    void validate();  // throws InputError; fills ffn_dim default
    static ModelConfig preset(const std::string& name);
};

// SplitMix64 (rng.hpp:10-43): counter based, draw i uses seed + (i+1)*golden.
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    static uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    uint64_t next() { return mix(state += 0x9e3779b97f4a7c15ULL); }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
};

uint64_t mix_seed(uint64_t seed, uint64_t tag);

// fp64 -> fp32 (RNE) -> bf16 (RNE) bits.
uint16_t to_bf16(double x);
double from_bf16(uint16_t b);

// Per-tensor rescale factors (index: 0 q,1 k,2 v,3 proj,4 ffn1,5 ffn2).
void rescale_factors(const ModelConfig& c, double out[6]);

// Host copy of the bf16 weights in device layout.
struct HostWeights {
    ModelConfig config;
    int max_seq = 0;
    std::vector<uint16_t> embedding;   // [vocab x d] (also the tied LM head, K-major)
    std::vector<uint16_t> positional;  // [max_seq x d]
    std::vector<uint16_t> layers;      // L x layer_elems(), packed as documented above
    size_t layer_elems() const;
    uint16_t* layer(int l) { return layers.data() + static_cast<size_t>(l) * layer_elems(); }
    const uint16_t* layer(int l) const { return layers.data() + static_cast<size_t>(l) * layer_elems(); }
};

// Offsets (elements) of each matrix inside a packed layer.
struct LayerOffsets {
    size_t wqkv, wproj, w1, w2, total;
    static LayerOffsets of(const ModelConfig& c);
};

// DecoderWeights::generate (model.cpp:94-117) + rescale + bf16 + transpose.
// rescale=false keeps the raw U(-0.1, 0.1) draws (parity with the unmodified
// reference init at toy depth).
HostWeights generate_weights(const ModelConfig& config, uint64_t seed, int max_seq, bool rescale = true);

// Streaming pieces of generate_weights (so multi-GB models can be drawn
// straight into pinned / staging memory): one packed layer, or the two tables.
void generate_layer(const ModelConfig& config, uint64_t seed, int layer, bool rescale, uint16_t* dst);
void generate_tables(const ModelConfig& config, uint64_t seed, int max_seq, uint16_t* emb, uint16_t* pos);

// Build from externally supplied fp64 tensors in the reference layout
// ([in x out], row-major): emb [V x d], pos [S x d], per layer q,k,v,proj
// [d x d], ffn1 [d x f], ffn2 [f x d].
HostWeights weights_from_f64(const ModelConfig& config, int max_seq, const double* emb, const double* pos,
                             const double* const* layer_tensors /* L*6 pointers */);

}  // namespace hc
