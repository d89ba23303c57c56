// hybridsim/cache.hpp — HybridCache and its block tables (cache.hpp:15-95)
// over the library's bit-exact bookkeeping (hc_cache_*). The wrapper keeps a
// read-only mirror of every table, refreshed after each mutation, so table()
// and append_block() can hand out references with the reference's lifetime
// rules (valid until the next mutation of that request).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <json.hpp>

#include "hybridsim/model.hpp"

namespace hybridsim {

enum class BlockKind { KV, ACT };
enum class Location { HostMem, GpuMem };

inline const char* to_string(BlockKind k) { return k == BlockKind::KV ? "KV" : "ACT"; }
inline const char* to_string(Location l) { return l == Location::HostMem ? "host" : "gpu"; }

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

    int context_len() const {
        int n = 0;
        for (const auto& e : entries) n += e.filled_tokens;
        return n;
    }
    std::pair<long, long> blocks_by_kind() const {  // (act, kv)
        long a = 0;
        for (const auto& e : entries) a += e.kind == BlockKind::ACT;
        return {a, static_cast<long>(entries.size()) - a};
    }
};

struct PoolCaps {
    long kv_host = 0;
    long kv_gpu = 0;
    long act_host = 0;
    long act_gpu = 0;
};

class HybridCache {
public:
    HybridCache(int tokens_per_block, PoolCaps caps, bool kv_on_gpu = false) : tpb_(tokens_per_block) {
        b200::check(hc_cache_create(tokens_per_block, caps.kv_host, caps.kv_gpu, caps.act_host, caps.act_gpu,
                                    kv_on_gpu ? 1 : 0, &h_));
    }
    HybridCache(const HybridCache&) = delete;
    HybridCache& operator=(const HybridCache&) = delete;
    HybridCache(HybridCache&& o) noexcept : h_(o.h_), tpb_(o.tpb_), tables_(std::move(o.tables_)),
                                            order_(std::move(o.order_)) {
        o.h_ = nullptr;
    }
    ~HybridCache() {
        if (h_) hc_cache_destroy(h_);
    }

    BlockTable& create_request(const std::string& id, int prompt_len) {
        b200::check(hc_cache_create_request(h_, id.c_str(), prompt_len));
        order_.push_back(id);
        BlockTable& t = tables_[id];
        t = BlockTable{id, prompt_len, {}};
        return t;
    }
    const BlockTableEntry& append_block(const std::string& id, BlockKind kind) {
        int loc = 0, pbn = 0;
        b200::check(hc_cache_append_block(h_, id.c_str(), kind == BlockKind::ACT ? 1 : 0, &loc, &pbn));
        BlockTable& t = tables_.at(id);
        t.entries.push_back(BlockTableEntry{kind, loc ? Location::GpuMem : Location::HostMem, pbn, 0});
        return t.entries.back();
    }
    void fill_token(const std::string& id) {
        b200::check(hc_cache_fill_token(h_, id.c_str()));
        tables_.at(id).entries.back().filled_tokens += 1;
    }
    std::pair<long, long> blocks_by_kind(const std::string& id) const {
        long a = 0, k = 0;
        b200::check(hc_cache_blocks_by_kind(h_, id.c_str(), &a, &k));
        return {a, k};
    }
    void free_request(const std::string& id) {
        b200::check(hc_cache_free_request(h_, id.c_str()));
        tables_.erase(id);
        for (auto it = order_.begin(); it != order_.end(); ++it)
            if (*it == id) {
                order_.erase(it);
                break;
            }
    }
    const BlockTable& table(const std::string& id) const {
        int n = 0;
        b200::check(hc_cache_table(h_, id.c_str(), nullptr, nullptr, nullptr, nullptr, 0, &n));  // InputError if unknown
        return tables_.at(id);
    }
    const std::vector<std::string>& request_order() const { return order_; }
    long free_blocks(BlockKind kind, Location loc) const {
        long n = 0;
        b200::check(hc_cache_free_blocks(h_, kind == BlockKind::ACT ? 1 : 0, loc == Location::GpuMem ? 1 : 0, &n));
        return n;
    }
    long capacity(BlockKind kind, Location loc) const {
        long n = 0;
        b200::check(hc_cache_capacity(h_, kind == BlockKind::ACT ? 1 : 0, loc == Location::GpuMem ? 1 : 0, &n));
        return n;
    }
    int tokens_per_block() const { return tpb_; }

    static std::uint64_t bytes_of(BlockKind kind, const ModelConfig& config) {
        std::uint64_t v = 0;
        b200::check(hc_bytes_of(kind == BlockKind::ACT ? 1 : 0, config.hidden_dim, config.tokens_per_block,
                                config.bytes_per_scalar, &v));
        return v;
    }
    nlohmann::json dump_json() const {
        long need = 0;
        b200::check(hc_cache_dump_json(h_, nullptr, 0, &need));
        std::string s(static_cast<size_t>(need), '\0');
        b200::check(hc_cache_dump_json(h_, s.data(), need, &need));
        s.resize(s.find('\0') == std::string::npos ? s.size() : s.find('\0'));
        return nlohmann::json::parse(s);
    }
    void* handle() const { return h_; }

private:
    void* h_ = nullptr;
    int tpb_;
    std::unordered_map<std::string, BlockTable> tables_;
    std::vector<std::string> order_;
};

}  // namespace hybridsim
