// A reference-style C++ caller of the B200 path through the C ABI only
// (include/hybridcache.h): what a hybridsim client (verify.cpp / sim.cpp
// style) looks like when it links libhybridcache_b200.so.
// Status codes are rethrown as the reference's exception types
// (errors.hpp:9-21). Builds with plain g++ (no CUDA headers):
//
//   g++ -std=c++17 -Iinclude examples/decode_demo.cpp -Lpaper_2501_01792_b200
//       -lhybridcache_b200 -Wl,-rpath,'$ORIGIN/../paper_2501_01792_b200' -o examples/decode_demo
//   (one line; __graft_entry__.build() does it)
//
// Run: prints the block table and greedy tokens, exits 0 ("decode_demo ok");
// without a GPU it exits 3 after the library reports status 4 for the first
// compute call (no CPU fallback).
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "hybridcache.h"

namespace hybridsim {
struct InputError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
}  // namespace hybridsim

struct CudaUnavailable : std::runtime_error {
    using std::runtime_error::runtime_error;
};

static void hc_check(int rc) {
    if (rc == 0) return;
    const std::string msg = hc_last_error();
    if (rc == 1) throw hybridsim::InputError(msg);
    if (rc == 2) throw hybridsim::CapacityError(msg);
    if (rc == 3) throw hybridsim::ConfigError(msg);
    throw CudaUnavailable(msg);
}

int main() {
    try {
        // a small OPT-like shape: 2 layers, d 256, 2 heads (hd 128), 16-token blocks
        hc_model_config cfg{};
        cfg.num_layers = 2;
        cfg.hidden_dim = 256;
        cfg.num_heads = 2;
        cfg.ffn_dim = 512;
        cfg.vocab_size = 512;
        cfg.tokens_per_block = 16;
        cfg.bytes_per_scalar = 2;
        hc_check(hc_model_validate(&cfg));

        hc_engine_options o{};
        o.max_batch = 2;
        o.weights_on_device = 0;  // weights streamed from pinned host memory per layer
        o.kv_host_cap = 8;
        o.act_host_cap = 8;
        o.act_gpu_cap = 1;
        o.mode = 0;               // hybrid
        o.alloc_act_host = 1;     // KV:ACT = 1:1 (next_block_kind target, plan.cpp:154-164)
        o.alloc_kv_host = 1;
        o.scaled = 1;
        void* eng = nullptr;
        hc_check(hc_engine_create(&cfg, 42, 64, 1, &o, &eng));  // DecoderWeights::generate(cfg, 42, 64)

        const char* ids[2] = {"r0", "r1"};
        std::vector<int> tokens;
        for (int t = 0; t < 37 + 20; ++t) tokens.push_back((t * 131 + 7) % cfg.vocab_size);
        const int offsets[3] = {0, 37, 57};
        hc_check(hc_engine_prefill(eng, 2, ids, offsets, tokens.data()));  // forward_prompt + ACT/KV writers

        int next[2] = {tokens[36], tokens[56]};
        for (int step = 0; step < 4; ++step) {  // generation_step, batched, greedy
            int argmax[2];
            hc_check(hc_engine_decode_step(eng, 2, ids, next, nullptr, nullptr, argmax));
            std::printf("step %d: tokens %d %d\n", step, argmax[0], argmax[1]);
            next[0] = argmax[0];
            next[1] = argmax[1];
        }
        void* cache = nullptr;
        hc_check(hc_engine_cache(eng, &cache));  // HybridCache (borrowed)
        long need = 0;
        hc_check(hc_cache_dump_json(cache, nullptr, 0, &need));
        std::vector<char> buf(static_cast<size_t>(need));
        hc_check(hc_cache_dump_json(cache, buf.data(), need, &need));
        std::printf("%s\n", buf.data());

        // the reference's error behaviour: an unknown request is an InputError
        try {
            const char* bad[1] = {"nope"};
            int t = 1;
            hc_check(hc_engine_decode_step(eng, 1, bad, &t, nullptr, nullptr, nullptr));
            std::printf("expected InputError\n");
            return 1;
        } catch (const hybridsim::InputError&) {
        }
        hc_check(hc_engine_destroy(eng));
        std::printf("decode_demo ok\n");
        return 0;
    } catch (const CudaUnavailable& e) {
        std::fprintf(stderr, "no CUDA device: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
