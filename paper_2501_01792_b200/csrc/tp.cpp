#include "tp.hpp"

#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "host/errors.hpp"

namespace hc {

// ------------------------------------------------------------------ NCCL ---
namespace {

// the subset of nccl.h this file needs (ABI-stable since NCCL 2.0)
using ncclComm_t = void*;
struct ncclUniqueId {
    char internal[128];
};
enum { kNcclSum = 0, kNcclFloat32 = 7, kNcclFloat16 = 6 };
struct NcclApi {
    int (*get_unique_id)(ncclUniqueId*) = nullptr;
    int (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(int) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        // HC_NCCL_LIB names a specific libnccl; otherwise reuse the copy a host
        // framework (torch) already loaded (RTLD_NOLOAD), else the system one.
        // Loading ours first would shadow torch's same-soname NCCL for a later
        // `import torch` — the Python API therefore imports torch first.
        void* h = nullptr;
        if (const char* p = std::getenv("HC_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.all_gather || !api.comm_destroy)
            err = "libnccl.so.2 lacks a required symbol";
    });
    if (!err.empty()) throw ConfigError(err);
    return api;
}

void nccl_check(int rc, const char* what) {
    if (rc != 0) {
        const char* s = nccl().error_string ? nccl().error_string(rc) : "?";
        throw std::runtime_error(std::string(what) + ": NCCL error " + std::to_string(rc) + " (" + s + ")");
    }
}

class NcclChannel final : public TpGroup {
public:
    NcclChannel(const uint8_t id[128], int rank, int size, TpGroup* copy) : rank_(rank), size_(size), copy_(copy) {
        ncclUniqueId u;
        std::memcpy(u.internal, id, 128);
        nccl_check(nccl().comm_init_rank(&comm_, size, u, rank), "ncclCommInitRank");
    }
    ~NcclChannel() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void all_reduce_sum(float* buf, size_t n, cudaStream_t st) override {
        if (size_ > 1 && n) nccl_check(nccl().all_reduce(buf, buf, n, kNcclFloat32, kNcclSum, comm_, st), "ncclAllReduce");
    }
    void all_gather(const f16* send, f16* recv, size_t n, cudaStream_t st) override {
        if (!n) return;
        if (size_ == 1) {
            if (send != recv) HC_CUDA(cudaMemcpyAsync(recv, send, n * 2, cudaMemcpyDeviceToDevice, st));
            return;
        }
        nccl_check(nccl().all_gather(send, recv, n, kNcclFloat16, comm_, st), "ncclAllGather");
    }
    TpGroup* copy_channel() override { return copy_ ? copy_ : this; }

private:
    ncclComm_t comm_ = nullptr;
    int rank_, size_;
    TpGroup* copy_;
};

class NcclGroup final : public TpGroup {
public:
    NcclGroup(const uint8_t idc[128], const uint8_t idk[128], int rank, int size)
        : copy_(idk, rank, size, nullptr), compute_(idc, rank, size, &copy_) {}
    int rank() const override { return compute_.rank(); }
    int size() const override { return compute_.size(); }
    void all_reduce_sum(float* buf, size_t n, cudaStream_t st) override { compute_.all_reduce_sum(buf, n, st); }
    void all_gather(const f16* s, f16* r, size_t n, cudaStream_t st) override { compute_.all_gather(s, r, n, st); }
    TpGroup* copy_channel() override { return &copy_; }

private:
    NcclChannel copy_;
    NcclChannel compute_;
};

}  // namespace

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(out, u.internal, 128);
}

std::unique_ptr<TpGroup> make_nccl_group(const uint8_t idc[128], const uint8_t idk[128], int rank, int size,
                                         int device) {
    if (size < 1 || rank < 0 || rank >= size) throw InputError("tensor parallel: bad rank / size");
    HC_CUDA(cudaSetDevice(device));
    return std::make_unique<NcclGroup>(idc, idk, rank, size);
}

// ------------------------------------------------------------- Emulated ---
namespace {
class EmulatedRank final : public TpGroup {
public:
    EmulatedRank(int rank, int size) : rank_(rank), size_(size) {}
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void all_reduce_sum(float*, size_t, cudaStream_t) override {}
    void all_gather(const f16*, f16*, size_t, cudaStream_t) override {}
    TpGroup* copy_channel() override { return this; }

private:
    int rank_, size_;
};
}  // namespace

std::unique_ptr<TpGroup> make_emulated_group(int rank, int size) {
    if (size < 1 || rank < 0 || rank >= size) throw InputError("tensor parallel: bad rank / size");
    return std::make_unique<EmulatedRank>(rank, size);
}

// ----------------------------------------------------------- LocalGroup ---
// Host-thread rendezvous: every collective is (post pointers, barrier, each
// rank pulls what it needs with peer copies into its own memory, barrier).
namespace {
struct Rendezvous {
    explicit Rendezvous(int n) : n(n), ptr(n, nullptr), dev(n, 0) {}
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<const void*> ptr;
    std::vector<int> dev;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long gen = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

class LocalMember final : public TpGroup {
public:
    LocalMember(Rendezvous* s, int rank, LocalMember* copy) : s_(s), rank_(rank), copy_(copy) {}
    ~LocalMember() override {
        if (tmp_) cudaFree(tmp_);
    }
    int rank() const override { return rank_; }
    int size() const override { return s_->n; }
    void all_reduce_sum(float* buf, size_t n, cudaStream_t st) override {
        if (!n) return;
        const int N = s_->n;
        post(buf, st);
        ensure_tmp(n * N);
        for (int j = 0; j < N; ++j)
            HC_CUDA(cudaMemcpyPeerAsync(tmp_ + j * n, dev_, s_->ptr[j], s_->dev[j], n * 4, st));
        HC_CUDA(cudaStreamSynchronize(st));
        s_->barrier();  // every rank has read every buffer
        sum_rows_f32(tmp_, N, n, buf, st);
        HC_CUDA(cudaStreamSynchronize(st));
        s_->barrier();
    }
    void all_gather(const f16* send, f16* recv, size_t n, cudaStream_t st) override {
        if (!n) return;
        post(send, st);
        for (int j = 0; j < s_->n; ++j) {
            f16* dst = recv + j * n;
            if (dst != s_->ptr[j] || s_->dev[j] != dev_)
                HC_CUDA(cudaMemcpyPeerAsync(dst, dev_, s_->ptr[j], s_->dev[j], n * 2, st));
        }
        HC_CUDA(cudaStreamSynchronize(st));
        s_->barrier();
    }
    TpGroup* copy_channel() override { return copy_ ? static_cast<TpGroup*>(copy_) : this; }

private:
    void post(const void* p, cudaStream_t st) {
        HC_CUDA(cudaGetDevice(&dev_));
        HC_CUDA(cudaStreamSynchronize(st));
        {
            std::lock_guard<std::mutex> lk(s_->mu);
            s_->ptr[rank_] = p;
            s_->dev[rank_] = dev_;
        }
        s_->barrier();  // every rank posted
    }
    void ensure_tmp(size_t elems) {
        if (elems <= tmp_elems_) return;
        if (tmp_) cudaFree(tmp_);
        HC_CUDA(cudaMalloc(&tmp_, elems * 4));
        tmp_elems_ = elems;
    }
    Rendezvous* s_;
    int rank_;
    LocalMember* copy_;
    int dev_ = 0;
    float* tmp_ = nullptr;
    size_t tmp_elems_ = 0;
};
}  // namespace

// owns both channels' rendezvous and every member
class LocalGroupState {
public:
    explicit LocalGroupState(int n) : compute(n), copy(n), members(n), copies(n) {}
    Rendezvous compute, copy;
    std::vector<std::unique_ptr<LocalMember>> members, copies;
    std::mutex mu;
};

std::shared_ptr<LocalGroupState> make_local_group(int size) {
    if (size < 1) throw InputError("tensor parallel: group size must be >= 1");
    return std::make_shared<LocalGroupState>(size);
}

TpGroup* local_group_member(const std::shared_ptr<LocalGroupState>& g, int rank) {
    if (!g || rank < 0 || rank >= g->compute.n) throw InputError("tensor parallel: bad local rank");
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->members[rank]) {
        g->copies[rank] = std::make_unique<LocalMember>(&g->copy, rank, nullptr);
        g->members[rank] = std::make_unique<LocalMember>(&g->compute, rank, g->copies[rank].get());
    }
    return g->members[rank].get();
}

}  // namespace hc
