// Mini-batch packer (paper §4.3.3; reference minibatch.hpp:10-47,
// minibatch.cpp:10-83; default capacities sim.cpp:122-132): greedy bin
// packing of requests into GPU-buffer-sized mini-batches minimising
// F_b = max(b, 1/b), b = predicted recompute time / predicted load time.
// Bit-exact with the reference (same visiting order and tie rules).
#pragma once
#include <string>
#include <vector>

#include "host/plan.hpp"

namespace hc {

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
    long act_max = 1;  // ACT blocks one staging buffer holds
    long kv_max = 1;   // KV blocks one staging buffer holds
};

double balance(long act_mb, long kv_mb, const TimingBundle& b, int tpb);
double cost_fb(long act_mb, long kv_mb, const TimingBundle& b, int tpb);
std::vector<MiniBatch> form_minibatches(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                        const TimingBundle& b, int tpb);
// Exhaustive search (<= 10 requests): fewest mini-batches, then the smallest
// mean F_b — the packer's quality oracle.
std::vector<MiniBatch> brute_force_pack(const std::vector<RequestBlocks>& requests, const PackerConfig& cfg,
                                        const TimingBundle& b, int tpb);
// Staging capacities from a GPU memory size: 1/4 for KV, 1/8 for ACT, halved
// for double buffering (sim.cpp:122-132).
PackerConfig default_packer(double gpu_mem_bytes, const ModelConfig& c);

}  // namespace hc
