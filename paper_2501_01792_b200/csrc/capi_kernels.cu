// Kernel-level C-ABI entry points (include/hybridcache.h, "kernel" section).
// Each takes HOST buffers, stages them to the device, runs one kernel of the
// path and copies the result back — the boundary the parity tests drive.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "kernels/gemm.cuh"
#include "kernels/kernels.hpp"

using namespace hc;

namespace {

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t count) : n(count) {
        if (count) HC_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    DevBuf(const T* host, size_t count) : DevBuf(count) {
        if (count) HC_CUDA(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void to_host(T* host) const {
        if (n) HC_CUDA(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

extern "C" {

// C[M x N] = A[M x K] . W  with W given transposed as Wt[N x K] (f16 bits).
// epi: 0 f16, 1 relu f16, 3 fp32 (out sized accordingly). bn: 0 = auto.
int hc_gemm_f16(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, void* out,
                 int bn) {
    return hc_guard([&] {
        if (epi != gemm::kStore && epi != gemm::kRelu && epi != gemm::kF32)
            throw hc_input_error("hc_gemm_f16: epi must be 0, 1 or 3");
        DevBuf<uint16_t> a(A, size_t(M) * K), w(Wt, size_t(N) * K);
        const size_t out_bytes = size_t(M) * N * (epi == gemm::kF32 ? 4 : 2);
        DevBuf<uint8_t> o(out_bytes);
        GemmCall c;
        c.epi = epi;
        c.A = reinterpret_cast<const f16*>(a.p);
        c.lda = K;
        c.a_rows = M;
        c.B = reinterpret_cast<const f16*>(w.p);
        c.ldb = K;
        c.M = M;
        c.N = N;
        c.K = K;
        c.out = o.p;
        c.ldc = N;
        c.bn = bn;
        run_gemm(c, nullptr);
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(static_cast<uint8_t*>(out));
    });
}

// Split-K variant of hc_gemm_f16 (epi 0 / 1): fp32 partials over `splits`
// K ranges reduced by splitk_reduce — the weight-streaming decode GEMMs.
int hc_gemm_f16_splitk(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, uint16_t* out, int bn,
                        int splits) {
    return hc_guard([&] {
        if (epi != gemm::kStore && epi != gemm::kRelu) throw hc_input_error("hc_gemm_f16_splitk: epi must be 0 or 1");
        if (splits < 1) throw hc_input_error("hc_gemm_f16_splitk: splits must be >= 1");
        DevBuf<uint16_t> a(A, size_t(M) * K), w(Wt, size_t(N) * K), o(size_t(M) * N);
        DevBuf<float> ws(size_t(splits) * M * N);
        GemmCall c;
        c.epi = epi;
        c.A = reinterpret_cast<const f16*>(a.p);
        c.lda = K;
        c.a_rows = M;
        c.B = reinterpret_cast<const f16*>(w.p);
        c.ldb = K;
        c.M = M;
        c.N = N;
        c.K = K;
        c.out = o.p;
        c.ldc = N;
        c.bn = bn;
        c.ws = ws.p;
        c.ws_floats = ws.n;
        c.splits = splits;
        run_gemm(c, nullptr);
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(out);
    });
}

// The weight-streaming decode GEMM (wstream.cuh: swap-AB, stream-K over
// `ctas` CTAs, 0 = one per SM) with the f16 epilogue operands of the OPT
// projections: C = A . W (+ bias[n]) (+ res[m][n]) (relu for epi 1); epi 3 fp32.
int hc_gemm_f16_wstream(int epi, int M, int N, int K, const uint16_t* A, const uint16_t* Wt, const uint16_t* bias,
                        const uint16_t* res, void* out, int ctas) {
    return hc_guard([&] {
        if (epi != gemm::kStore && epi != gemm::kRelu && epi != gemm::kF32)
            throw hc_input_error("hc_gemm_f16_wstream: epi must be 0, 1 or 3");
        if (M < 1 || M > 256 || N < 16 || N % 16 || K < 8 || K % 8)
            throw hc_input_error("hc_gemm_f16_wstream: needs 1 <= M <= 256, N % 16 == 0, K % 8 == 0");
        if (epi == gemm::kF32 && (bias || res)) throw hc_input_error("hc_gemm_f16_wstream: fp32 output takes no bias / res");
        DevBuf<uint16_t> a(A, size_t(M) * K), w(Wt, size_t(N) * K);
        DevBuf<uint16_t> b(bias, bias ? size_t(N) : 0), r(res, res ? size_t(M) * N : 0);
        const size_t out_bytes = size_t(M) * N * (epi == gemm::kF32 ? 4 : 2);
        DevBuf<uint8_t> o(out_bytes);
        DevBuf<float> ws(wstream_ws_floats(M));
        GemmCall c;
        c.epi = epi;
        c.A = reinterpret_cast<const f16*>(a.p);
        c.lda = K;
        c.a_rows = M;
        c.B = reinterpret_cast<const f16*>(w.p);
        c.ldb = K;
        c.M = M;
        c.N = N;
        c.K = K;
        c.out = o.p;
        c.ldc = N;
        c.bias = bias ? reinterpret_cast<const f16*>(b.p) : nullptr;
        c.res = res ? reinterpret_cast<const f16*>(r.p) : nullptr;
        c.ldr = N;
        c.ws = ws.p;
        c.ws_floats = ws.n;
        c.max_ctas = ctas;
        if (!run_wstream(c, nullptr)) throw hc_input_error("hc_gemm_f16_wstream: shape not supported (or HC_WSTREAM=0)");
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(static_cast<uint8_t*>(out));
    });
}

// Device time of one decode GEMM C[M x N] = A . W (W [N x K]) per launch, over
// `reps` back-to-back launches cycling through enough copies of W that none is
// L2-resident (weights stream from HBM as in a decode step). mode 0: the tile
// kernel with split-K + reduce (the planner's pick), 1: the weight-streaming
// kernel (wstream.cuh), 2: the same launched programmatically dependent (its
// weight prefetch overlaps the previous launch's tail). Measurement helper (scripts/decode_gemm_bench.py).
int hc_gemm_bench(int M, int N, int K, int epi, int mode, int reps, double* us_per_call) {
    return hc_guard([&] {
        if (M < 1 || N < 16 || K < 64 || reps < 1 || !us_per_call) throw hc_input_error("hc_gemm_bench: bad shape");
        const size_t wbytes = size_t(N) * K * 2;
        const int copies = std::max<int>(2, static_cast<int>((512ull << 20) / wbytes) + 1);
        DevBuf<uint16_t> a(size_t(M) * K), w(size_t(N) * K * copies), o(size_t(M) * N * 2);
        HC_CUDA(cudaMemset(a.p, 0x11, a.n * 2));
        HC_CUDA(cudaMemset(w.p, 0x11, w.n * 2));
        const size_t wsf = std::max(size_t(16) * M * N, wstream_ws_floats(M));
        DevBuf<float> ws(wsf);
        GemmCall c;
        c.epi = epi;
        c.A = reinterpret_cast<const f16*>(a.p);
        c.lda = K;
        c.a_rows = M;
        c.ldb = K;
        c.M = M;
        c.N = N;
        c.K = K;
        c.out = o.p;
        c.ldc = N;
        c.ws = ws.p;
        c.ws_floats = ws.n;
        auto launch = [&](int i) {
            c.B = reinterpret_cast<const f16*>(w.p) + size_t(i % copies) * N * K;
            c.pdl = mode == 2;
            if (mode >= 1) {
                if (!run_wstream(c, nullptr)) throw hc_input_error("hc_gemm_bench: wstream does not take this shape");
            } else {
                GemmCall t = c;
                t.splits = 0;
                run_gemm_tiled(t, nullptr);
            }
        };
        for (int i = 0; i < 3; ++i) launch(i);
        cudaEvent_t e0, e1;
        HC_CUDA(cudaEventCreate(&e0));
        HC_CUDA(cudaEventCreate(&e1));
        HC_CUDA(cudaEventRecord(e0, nullptr));
        for (int i = 0; i < reps; ++i) launch(i);
        HC_CUDA(cudaEventRecord(e1, nullptr));
        HC_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        HC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        HC_CUDA(cudaGetLastError());
        *us_per_call = ms * 1e3 / reps;
    });
}

// Recompute K|V of the ACT-cached blocks straight into the paged KV layout
// (north-star (2); recompute_kv_from_activation, decoder.cpp:123-129).
//   act_pool  [n_blocks x tpb x d]        ACT block payloads (f16 bits)
//   wkv_t     [2d x d]                     [W_K | W_V] transposed
//   tiles     [n_tiles]                    first pool row of each 128-row tile
//   kv_out    [n_blocks x 2 x H x tpb x hd] K|V blocks (f16 bits)
int hc_recompute_kv_paged(int n_blocks, int tpb, int d, int heads, const uint16_t* act_pool,
                          const uint16_t* wkv_t, const int* tiles, int n_tiles, uint16_t* kv_out, int bn) {
    return hc_guard([&] {
        if (d % heads) throw hc_input_error("hc_recompute_kv_paged: d % heads != 0");
        const size_t rows = size_t(n_blocks) * tpb;
        DevBuf<uint16_t> a(act_pool, rows * d), w(wkv_t, size_t(2) * d * d);
        DevBuf<int> t(tiles, n_tiles);
        DevBuf<uint16_t> o(size_t(n_blocks) * 2 * d * tpb);
        HC_CUDA(cudaMemset(o.p, 0, o.n * 2));
        GemmCall c;
        c.epi = gemm::kKvPaged;
        c.A = reinterpret_cast<const f16*>(a.p);
        c.lda = d;
        c.a_rows = static_cast<int>(rows);
        c.B = reinterpret_cast<const f16*>(w.p);
        c.ldb = d;
        c.M = static_cast<int>(rows);
        c.N = 2 * d;
        c.K = d;
        c.m_tile_rows = t.p;
        c.num_m_tiles = n_tiles;
        c.out = o.p;
        c.tpb = tpb;
        c.d = d;
        c.hd = d / heads;
        c.blk_off = 0;
        c.bn = bn;
        run_gemm(c, nullptr);
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(kv_out);
    });
}

// Decode attention over a hybrid block table (north-star (3)).
//   q [B x d]; region0 / region1: two block pools [n0|n1 x 2 x H x tpb x hd]
//   blk_ref [B x max_blocks] packed (region << 28 | index); n_blocks, ctx_len [B]
int hc_decode_attention(int B, int H, int hd, int tpb, const uint16_t* q, const uint16_t* region0,
                        long n0, const uint16_t* region1, long n1, const int* blk_ref, int max_blocks,
                        const int* n_blocks, const int* ctx_len, int scaled, int splits, uint16_t* out) {
    return hc_guard([&] {
        const int d = H * hd;
        const size_t blk = size_t(2) * d * tpb;
        DevBuf<uint16_t> dq(q, size_t(B) * d), r0(region0, n0 * blk), r1(region1, n1 * blk);
        DevBuf<int> dref(blk_ref, size_t(B) * max_blocks), dnb(n_blocks, B), dctx(ctx_len, B);
        DevBuf<uint16_t> o(size_t(B) * d);
        int max_ctx = 0;
        for (int b = 0; b < B; ++b) max_ctx = ctx_len[b] > max_ctx ? ctx_len[b] : max_ctx;
        if (splits <= 0) splits = attention_splits(B, H, max_ctx, tpb);
        DevBuf<float> work(size_t(B) * H * splits * (hd + 2));
        AttnCall c;
        c.q = reinterpret_cast<const f16*>(dq.p);
        c.ldq = d;
        c.out = reinterpret_cast<f16*>(o.p);
        c.blk_ref = dref.p;
        c.n_blocks = dnb.p;
        c.ctx_len = dctx.p;
        c.max_blocks = max_blocks;
        c.region[0] = reinterpret_cast<const f16*>(r0.p);
        c.region[1] = reinterpret_cast<const f16*>(r1.p);
        c.B = B;
        c.H = H;
        c.hd = hd;
        c.tpb = tpb;
        c.scale = scaled ? 1.0f / std::sqrt(static_cast<float>(hd)) : 1.0f;
        c.work = work.p;
        c.splits = splits;
        decode_attention(c, nullptr);
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(out);
    });
}

// Causal prefill attention over qkv rows [n_req*P x 3d] -> out [n_req*P x d].
int hc_prefill_attention(int n_req, int P, int H, int hd, const uint16_t* qkv, int scaled, uint16_t* out) {
    return hc_guard([&] {
        const int d = H * hd;
        DevBuf<uint16_t> dq(qkv, size_t(n_req) * P * 3 * d), o(size_t(n_req) * P * d);
        std::vector<int> cu(n_req + 1);
        for (int r = 0; r <= n_req; ++r) cu[r] = r * P;
        DevBuf<int> dcu(cu.data(), cu.size());
        prefill_attention(reinterpret_cast<const f16*>(dq.p), reinterpret_cast<f16*>(o.p), dcu.p, n_req, P, H, hd,
                          scaled ? 1.0f / std::sqrt(static_cast<float>(hd)) : 1.0f, nullptr,
                          static_cast<long long>(n_req) * P);
        HC_CUDA(cudaGetLastError());
        HC_CUDA(cudaDeviceSynchronize());
        o.to_host(out);
    });
}

}  // extern "C"
