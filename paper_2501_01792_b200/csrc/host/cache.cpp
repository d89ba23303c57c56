#include "host/cache.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "host/errors.hpp"

namespace hc {

const char* to_string(BlockKind k) { return k == BlockKind::ACT ? "ACT" : "KV"; }
const char* to_string(Location l) { return l == Location::GpuMem ? "gpu" : "host"; }

int BlockTable::context_len() const {
    int n = 0;
    for (const auto& e : entries) n += e.filled_tokens;
    return n;
}

std::pair<long, long> BlockTable::blocks_by_kind() const {
    const long act = std::count_if(entries.begin(), entries.end(),
                                   [](const BlockTableEntry& e) { return e.kind == BlockKind::ACT; });
    return {act, static_cast<long>(entries.size()) - act};
}

HybridCache::HybridCache(int tokens_per_block, PoolCaps caps, bool kv_on_gpu)
    : tpb_(tokens_per_block), kv_on_gpu_(kv_on_gpu) {
    if (tokens_per_block < 1) throw InputError("HybridCache: tokens_per_block must be >= 1");
    const long c[4] = {caps.kv_host, caps.kv_gpu, caps.act_host, caps.act_gpu};
    for (int i = 0; i < 4; ++i) {
        if (c[i] < 0) throw InputError("HybridCache: negative pool capacity");
        pools_[i].cap = c[i];
        pools_[i].free_stack.resize(static_cast<size_t>(c[i]));
        for (long b = 0; b < c[i]; ++b) pools_[i].free_stack[static_cast<size_t>(b)] = static_cast<int>(c[i] - 1 - b);
    }
}

BlockTable& HybridCache::mut(const std::string& id) {
    auto it = tables_.find(id);
    if (it == tables_.end()) throw InputError("unknown request id: " + id);
    return it->second;
}

const BlockTable& HybridCache::table(const std::string& id) const {
    auto it = tables_.find(id);
    if (it == tables_.end()) throw InputError("unknown request id: " + id);
    return it->second;
}

BlockTable& HybridCache::create_request(const std::string& id, int prompt_len) {
    if (prompt_len < 0) throw InputError("create_request: negative prompt length");
    if (tables_.count(id)) throw InputError("duplicate request id: " + id);
    BlockTable& t = tables_[id];
    t.request_id = id;
    t.prompt_len = prompt_len;
    order_.push_back(id);
    return t;
}

const BlockTableEntry& HybridCache::append_block(const std::string& id, BlockKind kind) {
    BlockTable& t = mut(id);
    if (!t.entries.empty() && t.entries.back().filled_tokens < tpb_)
        throw InputError("append_block: last block not yet full");
    const bool gpu_first = kind == BlockKind::ACT || kv_on_gpu_;
    Location loc;
    if (gpu_first && !pools_[slot(kind, Location::GpuMem)].free_stack.empty())
        loc = Location::GpuMem;
    else if (!pools_[slot(kind, Location::HostMem)].free_stack.empty())
        loc = Location::HostMem;
    else
        throw CapacityError(std::string("append_block: ") + to_string(kind) + " pools exhausted");
    Pool& p = pools_[slot(kind, loc)];
    const int pbn = p.free_stack.back();
    p.free_stack.pop_back();
    t.entries.push_back(BlockTableEntry{kind, loc, pbn, 0});
    return t.entries.back();
}

void HybridCache::fill_token(const std::string& id) {
    BlockTable& t = mut(id);
    if (t.entries.empty()) throw InputError("fill_token: no blocks; append_block first");
    if (t.entries.back().filled_tokens >= tpb_) throw InputError("fill_token: last block full; append_block first");
    ++t.entries.back().filled_tokens;
}

std::pair<long, long> HybridCache::blocks_by_kind(const std::string& id) const { return table(id).blocks_by_kind(); }

void HybridCache::free_request(const std::string& id) {
    BlockTable& t = mut(id);
    for (const auto& e : t.entries) pools_[slot(e.kind, e.location)].free_stack.push_back(e.pbn);
    tables_.erase(id);
    order_.erase(std::find(order_.begin(), order_.end(), id));
}

long HybridCache::free_blocks(BlockKind kind, Location loc) const {
    return static_cast<long>(pools_[slot(kind, loc)].free_stack.size());
}

long HybridCache::capacity(BlockKind kind, Location loc) const { return pools_[slot(kind, loc)].cap; }

uint64_t HybridCache::bytes_of(BlockKind kind, const ModelConfig& c) {
    const uint64_t row = static_cast<uint64_t>(c.hidden_dim) * static_cast<uint64_t>(c.bytes_per_scalar);
    return static_cast<uint64_t>(c.tokens_per_block) * row * (kind == BlockKind::KV ? 2u : 1u);
}

namespace {
void json_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char ch : s) {
        switch (ch) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            default:
                if (ch < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", ch);
                    out += buf;
                } else {
                    out += static_cast<char>(ch);
                }
        }
    }
    out += '"';
}
}  // namespace

std::string HybridCache::dump_json() const {
    // keys in lexicographic order, as nlohmann::json (std::map) dumps them
    std::string o = "{\"requests\":[";
    bool first_req = true;
    for (const std::string& id : order_) {
        const BlockTable& t = table(id);
        if (!first_req) o += ',';
        first_req = false;
        o += "{\"context_len\":" + std::to_string(t.context_len()) + ",\"entries\":[";
        for (size_t i = 0; i < t.entries.size(); ++i) {
            const auto& e = t.entries[i];
            if (i) o += ',';
            o += "{\"filled\":" + std::to_string(e.filled_tokens) + ",\"kind\":\"" + to_string(e.kind) +
                 "\",\"location\":\"" + to_string(e.location) + "\",\"pbn\":" + std::to_string(e.pbn) + "}";
        }
        o += "],\"id\":";
        json_string(o, t.request_id);
        o += ",\"prompt_len\":" + std::to_string(t.prompt_len) + "}";
    }
    o += "],\"tokens_per_block\":" + std::to_string(tpb_) + "}";
    return o;
}

// ---------------------------------------------------------------------------

BlockKind next_block_kind(long act_req, long kv_req, const HostAllocation& a) {
    if (a.act_host + a.kv_host <= 0) throw InputError("next_block_kind: allocation has no blocks");
    if (act_req < 0 || kv_req < 0) throw InputError("next_block_kind: negative block count");
    // keep the request's ACT share closest to the host allocation's; ties -> ACT
    const double target = static_cast<double>(a.act_host) / static_cast<double>(a.act_host + a.kv_host);
    const double n = static_cast<double>(act_req + kv_req + 1);
    const double if_act = std::abs(static_cast<double>(act_req + 1) / n - target);
    const double if_kv = std::abs(static_cast<double>(act_req) / n - target);
    return if_act <= if_kv ? BlockKind::ACT : BlockKind::KV;
}

void mode_allocation(CacheMode mode, HostAllocation& a, long& act_gpu) {
    switch (mode) {
        case CacheMode::Hybrid: break;
        case CacheMode::KvOnly:
        case CacheMode::TokenRecompute:
            a.kv_host += a.act_host / 2;  // one KV block = two ACT blocks of bytes
            a.act_host = 0;
            act_gpu = 0;
            break;
        case CacheMode::ActOnly:
            a.act_host += 2 * a.kv_host;
            a.kv_host = 0;
            break;
    }
}

BlockAssigner::BlockAssigner(HybridCache& cache, CacheMode mode, const HostAllocation& alloc, double recompute_ratio)
    : cache_(cache), mode_(mode), alloc_(alloc), ratio_(recompute_ratio) {
    if (mode == CacheMode::TokenRecompute && (recompute_ratio < 0.0 || recompute_ratio > 1.0))
        throw ConfigError("recompute_ratio must lie in [0, 1]");
}

void BlockAssigner::add_request(const std::string& id, int prompt_len) {
    cache_.create_request(id, prompt_len);
    rc_[id] = 0;
}

long BlockAssigner::recompute_tokens(const std::string& id) const {
    auto it = rc_.find(id);
    return it == rc_.end() ? 0 : it->second;
}

void BlockAssigner::check_batch_capacity(const std::vector<std::string>& ids) const {
    long act = 0, kv = 0;
    for (const std::string& id : ids) {
        if (mode_ == CacheMode::TokenRecompute) {  // the same rule as add_token, without the update
            const auto it = rc_.find(id);
            const long rc = it == rc_.end() ? 0 : it->second;
            const double total = static_cast<double>(rc + cache_.table(id).context_len() + 1);
            if (std::abs(static_cast<double>(rc + 1) / total - ratio_) <=
                std::abs(static_cast<double>(rc) / total - ratio_))
                continue;
        }
        const BlockTable& t = cache_.table(id);
        if (t.context_len() % cache_.tokens_per_block() != 0) continue;
        BlockKind kind = BlockKind::KV;
        if (mode_ == CacheMode::Hybrid) {
            const auto [a, k] = t.blocks_by_kind();
            kind = next_block_kind(a, k, alloc_);
        } else if (mode_ == CacheMode::ActOnly) {
            kind = BlockKind::ACT;
        }
        ++(kind == BlockKind::ACT ? act : kv);
    }
    const long act_free =
        cache_.free_blocks(BlockKind::ACT, Location::GpuMem) + cache_.free_blocks(BlockKind::ACT, Location::HostMem);
    const long kv_free = cache_.free_blocks(BlockKind::KV, Location::HostMem) +
                         (cache_.kv_on_gpu() ? cache_.free_blocks(BlockKind::KV, Location::GpuMem) : 0);
    if (act > act_free)
        throw CapacityError("append_block: ACT pools exhausted (the step needs " + std::to_string(act) + " blocks, " +
                            std::to_string(act_free) + " free)");
    if (kv > kv_free)
        throw CapacityError("append_block: KV pools exhausted (the step needs " + std::to_string(kv) + " blocks, " +
                            std::to_string(kv_free) + " free)");
}

TokenSlot BlockAssigner::add_token(const std::string& id) {
    TokenSlot s;
    if (mode_ == CacheMode::TokenRecompute) {
        long& rc = rc_[id];
        const double total = static_cast<double>(rc + cache_.table(id).context_len() + 1);
        const double with_rc = std::abs(static_cast<double>(rc + 1) / total - ratio_);
        const double without = std::abs(static_cast<double>(rc) / total - ratio_);
        if (with_rc <= without) {
            ++rc;
            return s;  // kept as a token id only
        }
    }
    const BlockTable& t = cache_.table(id);
    if (t.context_len() % cache_.tokens_per_block() == 0) {
        BlockKind kind = BlockKind::KV;
        if (mode_ == CacheMode::Hybrid) {
            const auto [a, k] = t.blocks_by_kind();
            kind = next_block_kind(a, k, alloc_);
        } else if (mode_ == CacheMode::ActOnly) {
            kind = BlockKind::ACT;
        }
        cache_.append_block(id, kind);
        s.new_block = true;
    }
    cache_.fill_token(id);
    s.stored = true;
    s.entry = cache_.table(id).entries.back();
    s.token_index = s.entry.filled_tokens - 1;
    return s;
}

}  // namespace hc
