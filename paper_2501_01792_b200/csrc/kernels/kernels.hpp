// Host-side launch API for every CUDA kernel of the hybrid-cache decode path.
// No torch types; plain device pointers + a stream.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace hc {

using f16 = __half;

// ---------------------------------------------------------------- GEMM ----
struct GemmCall {
    int epi = 0;                 // gemm::Epi
    const f16* A = nullptr;     // [a_rows x K], row stride lda (elements)
    long long lda = 0;
    int a_rows = 0;              // rows addressable by TMA (OOB rows read as 0)
    const f16* B = nullptr;     // [N x K] (weights transposed), row stride ldb
    long long ldb = 0;
    int M = 0, N = 0, K = 0;     // logical problem (rows >= M are not stored)
    const int* m_tile_rows = nullptr;  // device array of explicit tile first rows
    int num_m_tiles = 0;               // used with m_tile_rows
    void* out = nullptr;
    long long ldc = 0;
    int tpb = 0, d = 0, hd = 0, blk_off = 0;  // kKvPaged
    int bn = 0;                  // 0 = heuristic
    int max_ctas = 0;            // 0 = all SMs
    int group_m = 0;             // rasterisation group (0 = default 16)
    int l2_hint = -1;            // gemm::kL2* bits; -1 = by shape (large-M GEMMs keep the A slab in L2)
    float* ws = nullptr;         // split-K workspace (fp32); null disables split-K
    size_t ws_floats = 0;
    int splits = 0;              // 0 = planner (pick_split), else forced split count
    // f16 epilogue operands (kStore / kRelu / kKvPaged): C += bias[n] + res[m*ldr + n]
    // before relu (OPT linear biases and residual connections)
    const f16* bias = nullptr;
    const f16* res = nullptr;
    long long ldr = 0;
    // kAttnPart (recompute fused with decode attention; gemm.cuh attn_part_tile):
    // B = [Wk | Wv]^T with the V rows from v_row; N = 2 * heads * hd; blk_info
    // per (M tile, block slot) = request << 8 | valid tokens (-1: skip); q rows
    // by request (ld ldq, head h at column h * hd); partial records into part
    const int* blk_info = nullptr;
    const f16* q = nullptr;
    long long ldq = 0;
    float qscale = 1.f;
    float* part = nullptr;
    // weight-streaming kernel: launch with programmatic stream serialisation
    // (only when the previous operation on the stream is a kernel)
    int pdl = 0;
};
// the decode GEMMs' workspace (split-K / stream-K fp32 partials): with ws and
// neither splits nor bn forced, M <= 256 kStore / kRelu / kF32 GEMMs run the
// weight-streaming kernel (wstream.cuh), which needs wstream_ws_floats(M)
struct GemmScratch {
    float* ws = nullptr;
    size_t floats = 0;
    int pdl = 0;  // GemmCall::pdl for the weight-streaming kernel
};
// fp32 partial slots the weight-streaming GEMM uses at batch M (0: M > 256)
size_t wstream_ws_floats(int M);
// the weight-streaming GEMM when c qualifies (returns false otherwise)
bool run_wstream(const GemmCall& c, cudaStream_t st);
// out[m][n] = f16(epi(sum_s ws[s][m][n] + bias[n] + res[m*ldr + n])) — the
// split-K finish (relu, bias, res optional)
void splitk_reduce(const float* ws, int splits, int M, int N, f16* out, bool relu, cudaStream_t st,
                   const f16* bias = nullptr, const f16* res = nullptr, long long ldr = 0);
void run_gemm(const GemmCall& c, cudaStream_t st);
void run_gemm_tiled(const GemmCall& c, cudaStream_t st);  // run_gemm without the weight-streaming dispatch
int num_sms();

// ----------------------------------------------------------- attention ----
// Decode attention over the hybrid block table (north-star (3)).
// For request b: blocks blk_ref[b*max_blocks + i], i < n_blocks[b], each a
// packed (region << 28 | index) into one of 4 region base pointers; the last
// block holds ctx_len[b] - (n_blocks[b]-1)*tpb tokens. Block layout:
// [K|V][head][tpb][hd] f16. q: [B x d] (row stride ldq), out: [B x d].
struct AttnCall {
    const f16* q = nullptr;
    long long ldq = 0;
    f16* out = nullptr;
    const int* blk_ref = nullptr;
    const int* n_blocks = nullptr;
    const int* ctx_len = nullptr;
    int max_blocks = 0;
    const f16* region[16] = {};
    int B = 0, H = 0, hd = 0, tpb = 0;
    float scale = 1.f;
    // split-K workspace (fp32): [B*H*splits*(hd+2)]; nullptr -> no split
    float* work = nullptr;
    int splits = 1;
    // refs of region part_region are blocks whose K|V the fused recompute
    // (GemmCall kAttnPart) already reduced to flash-decoding partials: the
    // block's tpb / min(tpb, 32) records per head are merged instead of K|V
    const float* part = nullptr;
    int part_region = -1;
    // every block ref of the call is in part_region (no K|V-cached block, no
    // token-recompute block): the records-only kernel runs
    int records_only = 0;
};
void decode_attention(const AttnCall& c, cudaStream_t st);
// the (head_dim, tokens_per_block) pairs decode_attention is instantiated for
bool decode_attention_supported(int hd, int tpb);
int attention_splits(int B, int H, int max_ctx, int tpb);

// Causal prefill attention over ragged requests: request r owns rows
// [cu[r], cu[r+1]) of qkv [rows x 3d] (Q|K|V per row); out [rows x d].
// cu is a device array of n_req+1 offsets; max_len = max request length.
// rows = rows of qkv (bounds of the tcgen05 path's TMA map). head_dim 64 and 128
// run on tcgen05/TMEM (prefill_attention_tc.cu); the mma.sync kernel
// (prefill_attention.cu) only under HC_PREFILL_TC=0.
void prefill_attention(const f16* qkv, f16* out, const int* cu, int n_req, int max_len, int H, int hd,
                       float scale, cudaStream_t st, long long rows);

// --------------------------------------------------------------- misc ----
// X[i] = E[ids[i]] + Pos[pos[i]]   (decoder.cpp:65-95), f16 out
void embed(const f16* E, const f16* Pos, const int* ids, const int* pos, int n, int d, f16* X,
           long long ldx, cudaStream_t st);

// Token-slot writes of the new decode token (activation-cache writer / KV
// append, north-star (1)). Block refs are packed (region << 28 | index) into
// region[] (device pools, staging buffers, or mapped pinned-host pools).
// For request b:
//   act_append: X[b] -> ACT block row slot_tok[b] of dev_ref[b] and of
//               host_ref[b] (either may be -1 = skip). ACT layout [tpb][d].
//   kv_append:  K|V columns of qkv[b] -> KV block token slot (layout
//               [K|V][head][tpb][hd]) of dev_ref[b] / host_ref[b].
struct AppendCall {
    const f16* src = nullptr;      // act: X [B x d]; kv: qkv [B x 3d] (K at +d, V at +2d)
    long long ld = 0;
    const int* dev_ref = nullptr;
    const int* host_ref = nullptr;
    const int* tok = nullptr;
    f16* region[16] = {};
    int B = 0, d = 0, H = 0, hd = 0, tpb = 0;
};
void act_append(const AppendCall& c, cudaStream_t st);
void kv_append(const AppendCall& c, cudaStream_t st);

// Prefill scatter of whole blocks: block i takes rows [src_row[i],
// src_row[i] + n_tok[i]) of src and writes them to block dst_ref[i].
struct BlockScatter {
    const f16* src = nullptr;      // act: X rows [d]; kv: qkv rows [3d]
    long long ld = 0;
    const int* src_row = nullptr;
    const int* n_tok = nullptr;
    const int* dst_ref = nullptr;
    f16* region[16] = {};
    int n_blocks = 0, d = 0, H = 0, hd = 0, tpb = 0;
};
void scatter_act_blocks(const BlockScatter& c, cudaStream_t st);
void scatter_kv_blocks(const BlockScatter& c, cudaStream_t st);

// y[r] = (x[r] - mean_r) / sqrt(var_r + eps) * gamma + beta over rows r < n of
// width d (kArchOpt LayerNorms); f16 in/out, fp32 statistics.
void layernorm_rows(const f16* x, long long ldx, const f16* gamma, const f16* beta, f16* y, long long ldy, int n,
                    int d, float eps, cudaStream_t st);

// out[i] = sum_j src[j*n + i] for i < n, j < parts (in-process all-reduce)
void sum_rows_f32(const float* src, int parts, size_t n, float* out, cudaStream_t st);
// out[m][n] = f16(sum[m][n] + bias[n] + res[m*ldr + n]) (bias / res optional):
// the finish of a tensor-parallel all-reduce (W_proj, W2 partial sums)
void add_bias_residual(const float* sum, const f16* bias, const f16* res, long long ldr, int M, int N, f16* out,
                       cudaStream_t st);
// fp32 split-K finish: out[m][n] = sum_s ws[s][m][n]
void splitk_reduce_f32(const float* ws, int splits, int M, int N, float* out, cudaStream_t st);

// argmax over each row of fp32 logits [B x V]
void argmax_rows(const float* logits, int B, int V, int* out, cudaStream_t st);

// DecoderWeights::generate draws on the GPU (bit-exact with host/model.cpp):
// U(-0.1, 0.1) stream `seed`, times scale (if apply_scale), -> f16 bits;
// transposed: dst[c*rows + r] = value(r, c) of the reference's [rows x cols].
void gen_weights_transposed(uint16_t* dst, int rows, int cols, uint64_t seed, double scale, bool apply_scale,
                            cudaStream_t st);
void gen_weights_plain(uint16_t* dst, size_t n, uint64_t seed, cudaStream_t st);

// fill a f16 buffer with a deterministic hash pattern in [-a, a]
void fill_pattern(f16* dst, size_t n, uint64_t seed, float amp, cudaStream_t st);

inline int pack_ref(int region, int index) { return (region << 28) | index; }

}  // namespace hc
