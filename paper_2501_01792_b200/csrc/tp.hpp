// Tensor-parallel group of the optional head-sharded variant (SURVEY.md
// §8(e)): rank g of N owns heads [g H/N, (g+1) H/N) — their W_q|W_k|W_v
// columns, W_proj rows, a 1/N slice of the FFN, and the K|V of its heads in
// every KV block — plus the ACT blocks whose pbn % N == g. Per layer it
// needs two all-reduces of the [rows x d] partial sums (after proj and after
// FFN2) on the compute stream and one all-gather of the streamed ACT blocks
// on the copy stream, so every rank streams 1/N of the weights, 1/N of the
// KV bytes and 1/N of the ACT bytes over its own host link.
//
// Two implementations:
//   NcclGroup  — one process per GPU; NCCL (dlopen'ed libnccl.so.2, the copy
//                torch already loaded) with one communicator per stream so
//                the compute-stream and copy-stream collectives never
//                interleave differently across ranks. NVLink / NVSwitch.
//   LocalGroup — N ranks as N engines in ONE process (any devices, e.g. all
//                on one GPU), each driven by its own host thread: host
//                barriers + device copies. Tests the sharded arithmetic
//                without a multi-GPU box; not a performance path.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

#include "kernels/kernels.hpp"

namespace hc {

class TpGroup {
public:
    virtual ~TpGroup() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // buf[0..n) <- sum over ranks of buf[0..n)   (fp32: the partial sums of the
    // row-sharded W_proj / W2 GEMMs, reduced before bias + residual are added)
    virtual void all_reduce_sum(float* buf, size_t n, cudaStream_t st) = 0;
    // recv[r*n .. (r+1)*n) <- rank r's send[0..n)   (in-place when send == recv + rank*n)
    virtual void all_gather(const f16* send, f16* recv, size_t n, cudaStream_t st) = 0;
    // distinct collective channel for the copy stream (same group, own ordering)
    virtual TpGroup* copy_channel() = 0;
};

// NCCL: ids are ncclUniqueId bytes (128) created by rank 0 (nccl_unique_id)
// and broadcast by the caller (e.g. torch.distributed); two ids, one per channel.
void nccl_unique_id(uint8_t out[128]);
std::unique_ptr<TpGroup> make_nccl_group(const uint8_t id_compute[128], const uint8_t id_copy[128], int rank, int size,
                                         int device);

// Timing stand-in for ONE rank of an N-rank group on a single GPU: every
// shard shape, stream and byte count of rank `rank`, collectives skipped
// (outputs are not meaningful). bench.py --tp-emulate uses it to time a
// rank's step where only one GPU is available; NVLink time is modelled.
std::unique_ptr<TpGroup> make_emulated_group(int rank, int size);

// LocalGroup: make_local_group(N) returns the shared state; member(r) the rank-r
// handle (owned by the group).
class LocalGroupState;
std::shared_ptr<LocalGroupState> make_local_group(int size);
TpGroup* local_group_member(const std::shared_ptr<LocalGroupState>& g, int rank);

}  // namespace hc
