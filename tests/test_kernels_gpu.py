"""Kernel parity on the B200 through the C ABI (fp64 numpy reference on the
same bf16-rounded inputs). Tolerance: max|got-ref| / max|ref| <= 1e-2 for bf16
outputs (north_star: 'max relative error <= 1e-2'), 1e-4 for fp32 outputs."""
import numpy as np
import pytest

import hybridsim_oracle as O

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def rel(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def rand_bits(rng, shape, scale=1.0):
    from paper_2501_01792_b200.kernels import f32_to_f16_bits
    return f32_to_f16_bits(rng.uniform(-scale, scale, size=shape))


def f64(bits):
    from paper_2501_01792_b200.kernels import f16_bits_to_f32
    return f16_bits_to_f32(bits).astype(np.float64)


@pytest.mark.parametrize("M,N,K,bn", [
    (128, 128, 64, 0), (128, 256, 128, 256), (64, 768, 768, 0), (300, 512, 320, 128),
    (130, 96, 200, 32), (128, 7168 // 8, 1024, 64), (1024, 1024, 512, 256), (2048, 512, 7168 // 4, 0),
])
def test_gemm_f16_store(native, M, N, K, bn):
    from paper_2501_01792_b200.kernels import gemm_f16
    rng = np.random.default_rng(M * 7 + N + K)
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    ref = f64(a) @ f64(wt).T
    got = f64(gemm_f16(a, wt, 0, bn))
    assert rel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("bn", [32, 64, 128, 256])
def test_gemm_relu_and_f32(native, bn):
    from paper_2501_01792_b200.kernels import gemm_f16
    rng = np.random.default_rng(bn)
    M, N, K = 200, 512, 384
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    ref = f64(a) @ f64(wt).T
    got = f64(gemm_f16(a, wt, 1, bn))
    assert rel(got, np.maximum(ref, 0)) <= TOL_BF16
    assert (got >= 0).all()
    got32 = gemm_f16(a, wt, 3, bn).astype(np.float64)
    assert rel(got32, ref) <= 1e-4


@pytest.mark.parametrize("d,heads,nb,tpb", [(256, 2, 20, 16), (768, 12, 9, 16), (1024, 8, 33, 8)])
def test_recompute_kv_paged(native, d, heads, nb, tpb):
    """recompute_kv_from_activation (decoder.cpp:123-129) into paged blocks."""
    from paper_2501_01792_b200.kernels import recompute_kv_paged
    rng = np.random.default_rng(d + nb)
    act = rand_bits(rng, (nb, tpb, d))
    wk = rand_bits(rng, (d, d), 1.0 / np.sqrt(d))   # [in x out] as in the reference
    wv = rand_bits(rng, (d, d), 1.0 / np.sqrt(d))
    wkv_t = np.concatenate([wk.T, wv.T], axis=0)      # [2d x d]
    rows = nb * tpb
    tiles = np.arange(0, rows, 128, dtype=np.int32)
    got = f64(recompute_kv_paged(act, wkv_t, heads, tiles))
    a = f64(act).reshape(rows, d)
    k, v = O.recompute_kv_from_activation(a, 0, O.DecoderWeights(
        O.ModelConfig(num_layers=1, hidden_dim=d, num_heads=heads).validate(), 1, None, None,
        [{"w_k": f64(wk), "w_v": f64(wv)}]))
    hd = d // heads
    ref = np.stack([k.reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3),
                    v.reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3)], axis=1)
    assert got.shape == ref.shape
    assert rel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("nb,d,heads", [(300, 512, 4), (560, 256, 2), (1100, 256, 2)])
def test_recompute_kv_paged_many_groups(native, nb, d, heads):
    """The 1-SM recompute over 38 / 70 / 138 M tiles: several rasterisation
    groups including a partial last one, every tile exactly once."""
    from paper_2501_01792_b200.kernels import recompute_kv_paged
    rng = np.random.default_rng(nb + d)
    tpb = 16
    hd = d // heads
    act = rand_bits(rng, (nb, tpb, d))
    wkv = rand_bits(rng, (2 * d, d), 1.0 / np.sqrt(d))
    tiles = np.arange(0, nb * tpb, 128, dtype=np.int32)
    got = f64(recompute_kv_paged(act, wkv, heads, tiles, bn=256))
    x = f64(act).reshape(nb * tpb, d)
    kv = x @ f64(wkv).T
    k, v = kv[:, :d], kv[:, d:]
    ref = np.stack([k.reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3),
                    v.reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3)], axis=1)
    assert rel(got, ref) <= TOL_BF16


def test_recompute_kv_paged_tile_subset(native):
    """Only listed 128-row tiles are recomputed; other blocks stay untouched."""
    from paper_2501_01792_b200.kernels import recompute_kv_paged
    rng = np.random.default_rng(5)
    d, heads, nb, tpb = 256, 2, 32, 16
    act = rand_bits(rng, (nb, tpb, d))
    wkv_t = rand_bits(rng, (2 * d, d), 1.0 / 16)
    got = recompute_kv_paged(act, wkv_t, heads, np.array([256], np.int32))
    touched = np.abs(f64(got)).reshape(nb, -1).max(axis=1) > 0
    assert touched[16:24].all() and not touched[:16].any() and not touched[24:].any()


def _attention_case(rng, B, H, hd, tpb, ctxs, n0=64, n1=64):
    d = H * hd
    q = rand_bits(rng, (B, d))
    r0 = rand_bits(rng, (n0, 2, H, tpb, hd))
    r1 = rand_bits(rng, (n1, 2, H, tpb, hd))
    max_blocks = max((c + tpb - 1) // tpb for c in ctxs)
    refs = np.full((B, max_blocks), -1, np.int32)
    nbk = np.zeros(B, np.int32)
    want = np.zeros((B, d))
    pools = [f64(r0), f64(r1)]
    for b, c in enumerate(ctxs):
        n = (c + tpb - 1) // tpb
        nbk[b] = n
        ks, vs = [], []
        for i in range(n):
            region = int(rng.integers(0, 2))
            idx = int(rng.integers(0, (n0, n1)[region]))
            refs[b, i] = (region << 28) | idx
            blk = pools[region][idx]                       # [2, H, tpb, hd]
            ks.append(blk[0].transpose(1, 0, 2).reshape(tpb, d))
            vs.append(blk[1].transpose(1, 0, 2).reshape(tpb, d))
        K = np.concatenate(ks)[:c]
        V = np.concatenate(vs)[:c]
        want[b] = O.attention_rows(f64(q)[b:b + 1], K, V, [c], H, True)[0]
    return q, r0, r1, refs, nbk, np.asarray(ctxs, np.int32), want


@pytest.mark.parametrize("B,H,hd,tpb,ctxs,splits", [
    (4, 2, 128, 16, [1, 17, 33, 160], 1),
    (4, 12, 64, 16, [129, 144, 150, 160], 0),
    (3, 4, 128, 8, [5, 64, 200], 2),
    (2, 2, 64, 32, [31, 400], 4),
    (16, 8, 128, 16, [1152] * 16, 0),
])
def test_decode_attention_hybrid_table(native, B, H, hd, tpb, ctxs, splits):
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(B * 100 + H)
    q, r0, r1, refs, nbk, cl, want = _attention_case(rng, B, H, hd, tpb, ctxs)
    got = f64(decode_attention(q, r0, r1, refs, nbk, cl, H, True, splits))
    assert rel(got, want) <= TOL_BF16


def test_decode_attention_single_token_returns_v(native):
    """test_decoder.cpp:102-107: a one-token context returns that V row."""
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(1)
    q, r0, r1, refs, nbk, cl, want = _attention_case(rng, 2, 2, 128, 16, [1, 1])
    got = decode_attention(q, r0, r1, refs, nbk, cl, 2, True, 1)
    for b in range(2):
        idx = refs[b, 0] & 0x0FFFFFFF
        pool = (r0, r1)[refs[b, 0] >> 28]
        v = pool[idx, 1, :, 0, :].reshape(-1)
        assert np.array_equal(got[b], v)


@pytest.mark.parametrize("splits", [1, 2])
def test_decode_attention_ignores_unfilled_slots(native, splits):
    """Unfilled token slots of a partial last block may hold any bits (a block
    staged in HBM and copied out whole): NaN there must not reach the output
    (0 * NaN = NaN, so they are excluded, not zero-weighted)."""
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(7)
    B, H, hd, tpb = 3, 2, 128, 16
    ctxs = [5, 17, 40]
    d = H * hd
    q = rand_bits(rng, (B, d))
    nb = [(c + tpb - 1) // tpb for c in ctxs]
    r0 = rand_bits(rng, (sum(nb), 2, H, tpb, hd))
    r1 = rand_bits(rng, (1, 2, H, tpb, hd))
    refs = np.full((B, max(nb)), -1, np.int32)
    want = np.zeros((B, d))
    k0 = 0
    for b, c in enumerate(ctxs):
        refs[b, :nb[b]] = np.arange(k0, k0 + nb[b])
        last = k0 + nb[b] - 1
        r0[last, :, :, c - (nb[b] - 1) * tpb:, :] = 0x7FC0  # NaN in every unfilled slot
        blk = f64(r0[k0:k0 + nb[b]])
        K = blk[:, 0].transpose(0, 2, 1, 3).reshape(-1, d)[:c]
        V = blk[:, 1].transpose(0, 2, 1, 3).reshape(-1, d)[:c]
        want[b] = O.attention_rows(f64(q)[b:b + 1], K, V, [c], H, True)[0]
        k0 += nb[b]
    got = f64(decode_attention(q, r0, r1, refs, np.asarray(nb, np.int32), np.asarray(ctxs, np.int32), H, True,
                               splits))
    assert np.isfinite(got).all()
    assert rel(got, want) <= TOL_BF16


@pytest.mark.parametrize("n_req,P,H,hd", [(2, 37, 2, 128), (3, 130, 4, 64), (1, 256, 8, 128), (2, 1, 2, 128),
                                          (2, 64, 2, 64), (1, 321, 2, 128), (1, 640, 2, 128),
                                          (3, 1000, 2, 128), (2, 129, 3, 128), (1, 640, 2, 64),
                                          (3, 1000, 4, 64), (2, 257, 12, 64)])
def test_prefill_attention_causal(native, n_req, P, H, hd):
    from paper_2501_01792_b200.kernels import prefill_attention
    rng = np.random.default_rng(P)
    d = H * hd
    qkv = rand_bits(rng, (n_req * P, 3 * d))
    got = f64(prefill_attention(qkv, n_req, P, H))
    x = f64(qkv)
    for r in range(n_req):
        sl = slice(r * P, (r + 1) * P)
        want = O.attention_rows(x[sl, :d], x[sl, d:2 * d], x[sl, 2 * d:], list(range(1, P + 1)), H, True)
        assert rel(got[sl], want) <= TOL_BF16


@pytest.mark.parametrize("M,N,K", [(1024, 512, 512), (1100, 768, 320), (2560, 1024, 1024), (4096, 256, 7168 // 4)])
@pytest.mark.parametrize("epi", [0, 1, 3])
def test_gemm_cta_pair(native, M, N, K, epi):
    """Large-M GEMMs run on the CTA-pair (cta_group::2, 256x256) kernel."""
    from paper_2501_01792_b200.kernels import gemm_f16
    rng = np.random.default_rng(M + N + epi)
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    ref = f64(a) @ f64(wt).T
    if epi == 1:
        ref = np.maximum(ref, 0)
    got = gemm_f16(a, wt, epi, 0).astype(np.float64) if epi == 3 else f64(gemm_f16(a, wt, epi, 0))
    assert rel(got, ref) <= (1e-4 if epi == 3 else TOL_BF16)


@pytest.mark.parametrize("nb,tpb,d,heads", [(100, 16, 512, 4), (129, 16, 1024, 8), (64, 8, 256, 2)])
def test_recompute_kv_paged_cta_pair(native, nb, tpb, d, heads):
    """Paged recompute on the pair kernel, odd tile counts (tail tile repeated)."""
    from paper_2501_01792_b200.kernels import recompute_kv_paged
    rng = np.random.default_rng(nb + d)
    act = rand_bits(rng, (nb, tpb, d))
    wkv_t = rand_bits(rng, (2 * d, d), 1.0 / np.sqrt(d))
    rows = nb * tpb
    tiles = np.arange(0, rows, 128, dtype=np.int32)
    got = f64(recompute_kv_paged(act, wkv_t, heads, tiles))
    a = f64(act).reshape(rows, d)
    kv = a @ f64(wkv_t).T
    hd = d // heads
    ref = np.stack([kv[:, :d].reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3),
                    kv[:, d:].reshape(nb, tpb, heads, hd).transpose(0, 2, 1, 3)], axis=1)
    assert rel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("M,N,K,bn,splits,epi", [
    (128, 512, 2048, 128, 4, 0), (64, 768, 3072, 64, 3, 1), (100, 1024, 4096, 256, 8, 0), (128, 256, 448, 128, 2, 1),
    (128, 384, 1000, 64, 5, 0),
])
def test_gemm_splitk(native, M, N, K, bn, splits, epi):
    """Split-K decode GEMM: fp32 partials over K ranges + reduce == the full GEMM."""
    from paper_2501_01792_b200.kernels import gemm_f16_splitk
    rng = np.random.default_rng(K + splits)
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    ref = f64(a) @ f64(wt).T
    if epi == 1:
        ref = np.maximum(ref, 0)
    got = f64(gemm_f16_splitk(a, wt, splits, epi, bn))
    assert rel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("scaled", [True, False])
def test_decode_attention_unscaled_matches_oracle(native, scaled):
    """attention_step(q, kv, heads, scaled) with scaled=false (decoder.hpp:28,
    test_decoder.cpp:124-135): the raw q.k scores, no 1/sqrt(hd)."""
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(11)
    B, H, hd, tpb = 3, 4, 64, 16
    q, r0, r1, refs, nbk, cl, _ = _attention_case(rng, B, H, hd, tpb, [7, 40, 130])
    q = f32_bits(f64(q) * 0.25)  # keep the unscaled scores in a sane range
    want = np.zeros((B, H * hd))
    pools = [f64(r0), f64(r1)]
    for b, c in enumerate(cl):
        ks, vs = [], []
        for i in range(nbk[b]):
            blk = pools[refs[b, i] >> 28][refs[b, i] & 0x0FFFFFFF]
            ks.append(blk[0].transpose(1, 0, 2).reshape(tpb, -1))
            vs.append(blk[1].transpose(1, 0, 2).reshape(tpb, -1))
        want[b] = O.attention_rows(f64(q)[b:b + 1], np.concatenate(ks)[:c], np.concatenate(vs)[:c], [int(c)], H,
                                   scaled)[0]
    got = f64(decode_attention(q, r0, r1, refs, nbk, cl, H, scaled, 1))
    assert rel(got, want) <= TOL_BF16


def f32_bits(x):
    from paper_2501_01792_b200.kernels import f32_to_f16_bits
    return f32_to_f16_bits(x)


@pytest.mark.parametrize("splits", [1, 3])
def test_decode_attention_identical_rows_return_shared_v(native, splits):
    """test_decoder.cpp:109-122: every context token with the same K row and the
    same V row -> the output is that V row (softmax weights sum to 1; the fp32
    result rounds back to the fp16 V value)."""
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(12)
    B, H, hd, tpb, nb = 2, 2, 128, 16, 5
    q = rand_bits(rng, (B, H * hd))
    krow, vrow = rand_bits(rng, (H, hd)), rand_bits(rng, (H, hd))
    r0 = np.zeros((nb, 2, H, tpb, hd), np.uint16)
    r0[:, 0] = krow[None, :, None, :]
    r0[:, 1] = vrow[None, :, None, :]
    r1 = r0[:1].copy()
    refs = np.tile(np.arange(nb, dtype=np.int32), (B, 1))
    refs[1, 2] = (1 << 28)  # a block of the second region
    cl = np.array([nb * tpb, nb * tpb - 7], np.int32)
    got = decode_attention(q, r0, r1, refs, np.full(B, nb, np.int32), cl, H, True, splits)
    for b in range(B):
        assert np.abs(f64(got[b]) - f64(vrow.reshape(-1))).max() <= 2 ** -10 * np.abs(f64(vrow)).max()


@pytest.mark.parametrize("scaled", [True, False])
def test_decode_attention_stays_in_v_envelope(native, scaled):
    """test_decoder.cpp:140-162: each output column lies inside [min, max] of
    that column of V over the context (a convex combination), up to one fp16
    rounding of the output, over random heads / widths / context lengths."""
    from paper_2501_01792_b200.kernels import decode_attention
    rng = np.random.default_rng(13)
    for trial in range(12):
        H = int(rng.integers(1, 5))
        hd = int(rng.choice([64, 128]))
        tpb = int(rng.choice([8, 16, 32]))
        ctxs = [int(c) for c in rng.integers(1, 200, 3)]
        q, r0, r1, refs, nbk, cl, _ = _attention_case(rng, 3, H, hd, tpb, ctxs, n0=40, n1=40)
        got = f64(decode_attention(q, r0, r1, refs, nbk, cl, H, scaled, int(rng.integers(0, 3))))
        pools = [f64(r0), f64(r1)]
        for b, c in enumerate(ctxs):
            vs = [pools[refs[b, i] >> 28][refs[b, i] & 0x0FFFFFFF][1].transpose(1, 0, 2).reshape(tpb, -1)
                  for i in range(nbk[b])]
            V = np.concatenate(vs)[:c]
            lo, hi = V.min(axis=0), V.max(axis=0)
            ulp = 2.0 ** -10 * np.maximum(np.abs(lo), np.abs(hi))
            assert (got[b] >= lo - ulp).all() and (got[b] <= hi + ulp).all(), (trial, b)


def test_recompute_fault_injection_is_caught(native):
    """Negative control (verify.cpp:49-50, test_decoder.cpp:299-302): W_K[0,0]
    += 0.5 in the recompute path must make the recomputed-K comparison fail
    the 1e-2 bar, while the clean weights pass it. (The reference checks the
    end-to-end output at 1e-10 in fp64; through the decoder that fault moves
    the output by 1e-10..7e-4 — below any 16-bit bar — so the control sits at
    the recompute boundary the north star's K/V tolerance applies to.)"""
    from paper_2501_01792_b200.kernels import recompute_kv_paged
    rng = np.random.default_rng(14)
    nb, tpb, d, H = 16, 16, 256, 2
    act = rand_bits(rng, (nb, tpb, d), 0.1)
    w_k = rng.uniform(-0.1, 0.1, (d, d)) * 10 * np.sqrt(3 / d)
    w_v = rng.uniform(-0.1, 0.1, (d, d)) * 10 * np.sqrt(3 / d)
    wkv_t = f32_bits(np.concatenate([w_k.T, w_v.T]))
    X = f64(act).reshape(-1, d)
    want_k = X @ f64(wkv_t[:d]).T
    faulted = f64(wkv_t).copy()
    faulted[0, 0] += 0.5  # W_K[0][0] (row 0 of W_K^T is output column 0)
    for w, caught in ((wkv_t, False), (f32_bits(faulted), True)):
        got = f64(recompute_kv_paged(act, w, H, np.array([0, 128], np.int32)))
        k = got[:, 0].transpose(0, 2, 1, 3).reshape(-1, d)
        assert (rel(k, want_k) > TOL_BF16) == caught


@pytest.mark.parametrize("M,N,K,epi,ctas", [
    (1, 256, 64, 0, 0), (4, 768, 256, 0, 0), (16, 512, 1000, 1, 0), (33, 1536, 4096, 0, 0),
    (64, 12288, 4096, 0, 0), (64, 4096, 16384, 0, 0), (100, 2048, 2048, 1, 0), (128, 21504, 7168, 0, 0),
    (128, 7168, 28672, 0, 0), (200, 1024, 512, 0, 0), (256, 640, 1088, 1, 0), (128, 50272, 1024, 3, 0),
    (64, 2048, 4096, 0, 7), (48, 1024, 8192, 1, 3), (128, 1280, 640, 0, 148), (8, 272, 136, 3, 5),
])
def test_gemm_wstream(native, M, N, K, epi, ctas):
    """Weight-streaming decode GEMM (swap-AB, stream-K, cut units summed by
    the dependent reduce kernel): equals the fp64 product for every batch width
    MP 16..256, ragged N / K (OOB boxes), units cut across 1..148 CTAs, relu /
    fp32 epilogues."""
    from paper_2501_01792_b200.kernels import gemm_f16_wstream
    rng = np.random.default_rng(M * 31 + N + K + ctas)
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    ref = f64(a) @ f64(wt).T
    if epi == 3:
        got = gemm_f16_wstream(a, wt, 3, ctas=ctas).astype(np.float64)
        assert rel(got, ref) <= 1e-4
        return
    if epi == 1:
        ref = np.maximum(ref, 0)
    got = f64(gemm_f16_wstream(a, wt, epi, ctas=ctas))
    assert rel(got, ref) <= TOL_BF16


@pytest.mark.parametrize("M,N,K,relu", [(64, 768, 512, False), (128, 1024, 3000, True), (5, 4096, 256, False)])
def test_gemm_wstream_bias_residual(native, M, N, K, relu):
    """The OPT projections' epilogue: C = relu?(A . W + bias[n] + res[m][n])."""
    from paper_2501_01792_b200.kernels import gemm_f16_wstream
    rng = np.random.default_rng(N + K)
    a = rand_bits(rng, (M, K))
    wt = rand_bits(rng, (N, K), 1.0 / np.sqrt(K))
    bias = rand_bits(rng, (N,), 0.5)
    res = rand_bits(rng, (M, N))
    ref = f64(a) @ f64(wt).T + f64(bias)[None, :] + f64(res)
    if relu:
        ref = np.maximum(ref, 0)
    got = f64(gemm_f16_wstream(a, wt, 1 if relu else 0, bias, res, ctas=37))
    assert rel(got, ref) <= TOL_BF16
