// Hybrid cache block tables — the "cache layout descriptors" of the engine
// API (reference: cache.hpp:15-95, cache.cpp:35-166; bit-exact behaviour).
//
// Four (kind x location) pools of physical block numbers (pbn) with LIFO free
// lists that hand out pbn 0 first; per request an ordered block table where
// only the last entry may be partially filled. ACT blocks prefer the GPU pool
// until it drains; KV blocks go to host unless kv_on_gpu. A failed append
// leaves the table untouched (CapacityError).
//
// Unlike the reference ("blocks are records, not buffers", cache.hpp:47-48)
// each pbn here names real storage: the engine maps (kind, location, pbn) to
// an HBM or pinned-host block (engine.hpp).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "host/model.hpp"

namespace hc {

enum class BlockKind : int { KV = 0, ACT = 1 };
enum class Location : int { HostMem = 0, GpuMem = 1 };

const char* to_string(BlockKind k);
const char* to_string(Location l);

struct BlockTableEntry {
    BlockKind kind;
    Location location;
    int pbn = -1;
    int filled_tokens = 0;
};

struct BlockTable {
    std::string request_id;
    int prompt_len = 0;
    std::vector<BlockTableEntry> entries;
    int context_len() const;
    std::pair<long, long> blocks_by_kind() const;  // (act, kv)
};

struct PoolCaps {
    long kv_host = 0;
    long kv_gpu = 0;
    long act_host = 0;
    long act_gpu = 0;
};

class HybridCache {
public:
    HybridCache(int tokens_per_block, PoolCaps caps, bool kv_on_gpu = false);

    BlockTable& create_request(const std::string& id, int prompt_len);
    const BlockTableEntry& append_block(const std::string& id, BlockKind kind);
    void fill_token(const std::string& id);
    std::pair<long, long> blocks_by_kind(const std::string& id) const;
    void free_request(const std::string& id);
    const BlockTable& table(const std::string& id) const;
    const std::vector<std::string>& request_order() const { return order_; }
    bool has_request(const std::string& id) const { return tables_.count(id) != 0; }

    long free_blocks(BlockKind kind, Location loc) const;
    long capacity(BlockKind kind, Location loc) const;
    int tokens_per_block() const { return tpb_; }
    bool kv_on_gpu() const { return kv_on_gpu_; }

    // Per-layer payload bytes of one block (cache.cpp:142-147).
    static uint64_t bytes_of(BlockKind kind, const ModelConfig& config);

    // Same document as the reference's dump_json().dump(): compact, keys sorted.
    std::string dump_json() const;

private:
    struct Pool {
        long cap = 0;
        std::vector<int> free_stack;  // back() is handed out next
    };
    static int slot(BlockKind k, Location l) { return static_cast<int>(k) * 2 + static_cast<int>(l); }
    BlockTable& mut(const std::string& id);

    int tpb_;
    bool kv_on_gpu_;
    Pool pools_[4];
    std::unordered_map<std::string, BlockTable> tables_;
    std::vector<std::string> order_;
};

// The simulator's per-token growth rule (sim.cpp:150-220): at each block
// boundary pick the kind by the ratio policy (hybrid), or force KV / ACT;
// token_recompute keeps a token-level share as ids only. Reproduces the
// reference's block tables bit-exactly when driven in the same call order.
enum class CacheMode : int { Hybrid = 0, KvOnly = 1, ActOnly = 2, TokenRecompute = 3 };

struct HostAllocation {
    long act_host = 0, kv_host = 0;
    long act_init = 0, kv_init = 0;
    long act_remain = 0, kv_remain = 0;
};

BlockKind next_block_kind(long act_req, long kv_req, const HostAllocation& allocation);

// Byte-neutral pool conversion of forced modes (sim.cpp:150-167).
void mode_allocation(CacheMode mode, HostAllocation& alloc, long& act_gpu);

struct TokenSlot {
    bool stored = false;   // false: token-recompute token (no cache payload)
    BlockTableEntry entry{};
    int token_index = 0;   // row inside the block
    bool new_block = false;
};

class BlockAssigner {
public:
    BlockAssigner(HybridCache& cache, CacheMode mode, const HostAllocation& alloc, double recompute_ratio = 0.0);
    void add_request(const std::string& id, int prompt_len);
    TokenSlot add_token(const std::string& id);
    // Dry run of add_token over a batch (no mutation): throws CapacityError if
    // the new blocks the batch would append do not fit the free pools, so a
    // batched decode step either grows every context or none (the reference's
    // per-token append leaves the table untouched on failure, cache.cpp:91, 98).
    void check_batch_capacity(const std::vector<std::string>& ids) const;
    long recompute_tokens(const std::string& id) const;
    CacheMode mode() const { return mode_; }
    const HostAllocation& allocation() const { return alloc_; }

private:
    HybridCache& cache_;
    CacheMode mode_;
    HostAllocation alloc_;
    double ratio_;
    std::unordered_map<std::string, long> rc_;
};

}  // namespace hc
