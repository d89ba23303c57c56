#include "host/model.hpp"

#include <cmath>
#include <cstring>
#include <string>
#include <thread>

#include "host/errors.hpp"

namespace hc {

void ModelConfig::validate() {
    if (ffn_dim == 0) ffn_dim = 4 * hidden_dim;
    if (num_layers < 1 || hidden_dim < 1 || num_heads < 1 || vocab_size < 1 || tokens_per_block < 1 ||
        bytes_per_scalar < 1)
        throw InputError("ModelConfig: all counts must be >= 1");
    if (hidden_dim % num_heads != 0) throw InputError("ModelConfig: hidden_dim must be divisible by num_heads");
    if (ffn_dim < hidden_dim) throw InputError("ModelConfig: ffn_dim must be >= hidden_dim");
}

ModelConfig ModelConfig::preset(const std::string& name) {
    // public OPT shapes (model.cpp:37-43); vocab 50272, 16-token blocks, fp16 bytes
    struct P {
        const char* n;
        int l, d, h;
    };
    static const P table[] = {{"opt-6.7b", 32, 4096, 32},
                              {"opt-13b", 40, 5120, 40},
                              {"opt-30b", 48, 7168, 56},
                              {"opt-66b", 64, 9216, 72}};
    for (const P& p : table) {
        if (name == p.n) {
            ModelConfig c;
            c.name = name;
            c.num_layers = p.l;
            c.hidden_dim = p.d;
            c.num_heads = p.h;
            c.ffn_dim = 4 * p.d;
            c.vocab_size = 50272;
            return c;
        }
    }
    throw InputError("unknown model preset: " + name);
}

uint64_t mix_seed(uint64_t seed, uint64_t tag) {
    SplitMix64 r(seed ^ (0x9e3779b97f4a7c15ULL * (tag + 1)));
    return r.next();
}

uint16_t to_f16(double x) {
    // fp64 -> fp32 (RNE, the C++ conversion) -> IEEE binary16 (RNE), with
    // subnormals, overflow to inf and quiet NaNs — what __float2half_rn does
    const float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t sign = (u >> 16) & 0x8000u;
    const int exp = static_cast<int>((u >> 23) & 0xffu);
    uint32_t mant = u & 0x7fffffu;
    if (exp == 0xff) return static_cast<uint16_t>(sign | 0x7c00u | (mant ? 0x200u | (mant >> 13) : 0u));
    const int e = exp - 127 + 15;
    if (e >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
    if (e <= 0) {  // binary16 subnormal (or zero)
        if (e < -10) return static_cast<uint16_t>(sign);
        mant |= 0x800000u;
        const int shift = 14 - e;
        uint32_t h = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1u), half = 1u << (shift - 1);
        if (rem > half || (rem == half && (h & 1u))) ++h;
        return static_cast<uint16_t>(sign | h);
    }
    uint32_t h = (static_cast<uint32_t>(e) << 10) | (mant >> 13);
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;  // a carry into the exponent is exact (up to inf)
    return static_cast<uint16_t>(sign | h);
}

double from_f16(uint16_t b) {
    const int exp = (b >> 10) & 0x1f, mant = b & 0x3ff;
    const double s = (b & 0x8000) ? -1.0 : 1.0;
    if (exp == 0x1f) return mant ? std::nan("") : s * INFINITY;
    if (exp == 0) return s * std::ldexp(static_cast<double>(mant), -24);
    return s * std::ldexp(static_cast<double>(mant | 0x400), exp - 25);
}

void rescale_factors(const ModelConfig& c, double out[6]) {
    const double d = c.hidden_dim, f = c.ffn_dim;
    const double s_attn = 10.0 * std::sqrt(3.0 / d);
    out[0] = out[1] = out[2] = out[3] = s_attn;
    out[4] = 10.0 * std::sqrt(3.0 * std::sqrt(2.0) / d);
    out[5] = 10.0 * std::sqrt(3.0 * std::sqrt(2.0) / f);
}

LayerOffsets LayerOffsets::of(const ModelConfig& c, int arch, int tp) {
    if (tp < 1 || c.num_heads % tp || c.ffn_dim % tp) throw InputError("tensor parallel size must divide heads and ffn_dim");
    const size_t d = c.hidden_dim, f = c.ffn_dim, dg = d / tp, fg = f / tp;
    LayerOffsets o;
    o.wqkv = 0;
    o.wproj = 3 * dg * d;
    o.w1 = o.wproj + d * dg;
    o.w2 = o.w1 + fg * d;
    o.total = o.w2 + d * fg;
    if (arch == kArchOpt) {
        o.bqkv = o.total;
        o.bproj = o.bqkv + 3 * dg;
        o.b1 = o.bproj + d;
        o.b2 = o.b1 + fg;
        o.ln1g = o.b2 + d;
        o.ln1b = o.ln1g + d;
        o.ln2g = o.ln1b + d;
        o.ln2b = o.ln2g + d;
        o.total = o.ln2b + d;
    } else if (arch != kArchReference) {
        throw InputError("unknown model arch: " + std::to_string(arch));
    }
    return o;
}

size_t HostWeights::layer_elems() const { return LayerOffsets::of(config, arch).total; }

namespace {

// Draw a rows x cols U(-0.1, 0.1) matrix from stream `seed` (model.cpp:82-87)
// and store scale * value transposed into dst[cols x rows] as f16. The
// counter-based generator lets threads split the draw sequence.
void draw_transposed(uint16_t* dst, int rows, int cols, uint64_t seed, double scale) {
    const size_t n = static_cast<size_t>(rows) * cols;
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = static_cast<int>(std::min<size_t>(hw ? hw : 4, std::max<size_t>(1, n / (1 << 20))));
    auto work = [&](size_t r0, size_t r1) {
        for (size_t r = r0; r < r1; ++r) {
            for (int c = 0; c < cols; ++c) {
                const size_t i = r * cols + c;
                const uint64_t z = SplitMix64::mix(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
                const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
                const double v = -0.1 + (0.1 - -0.1) * u;
                dst[static_cast<size_t>(c) * rows + r] = to_f16(v * scale);
            }
        }
    };
    if (nt <= 1) {
        work(0, rows);
        return;
    }
    std::vector<std::thread> ts;
    for (int t = 0; t < nt; ++t)
        ts.emplace_back(work, static_cast<size_t>(rows) * t / nt, static_cast<size_t>(rows) * (t + 1) / nt);
    for (auto& t : ts) t.join();
}

// Same draw without transposition (embedding / positional tables).
void draw_plain(uint16_t* dst, int rows, int cols, uint64_t seed) {
    const size_t n = static_cast<size_t>(rows) * cols;
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = static_cast<int>(std::min<size_t>(hw ? hw : 4, std::max<size_t>(1, n / (1 << 20))));
    auto work = [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            const uint64_t z = SplitMix64::mix(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
            const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
            dst[i] = to_f16(-0.1 + (0.1 - -0.1) * u);
        }
    };
    std::vector<std::thread> ts;
    for (int t = 0; t < nt; ++t) ts.emplace_back(work, n * t / nt, n * (t + 1) / nt);
    for (auto& t : ts) t.join();
}

}  // namespace

void generate_tables(const ModelConfig& c, uint64_t seed, int max_seq, uint16_t* emb, uint16_t* pos) {
    draw_plain(emb, c.vocab_size, c.hidden_dim, mix_seed(seed, 0));
    draw_plain(pos, max_seq, c.hidden_dim, mix_seed(seed, 1));
}

void generate_layer(const ModelConfig& c, uint64_t seed, int l, bool rescale, uint16_t* L) {
    const int d = c.hidden_dim, f = c.ffn_dim;
    double fac[6];
    rescale_factors(c, fac);
    if (!rescale)
        for (double& x : fac) x = 1.0;
    const LayerOffsets off = LayerOffsets::of(c);
    const uint64_t base = 100 + static_cast<uint64_t>(l) * 8;  // model.cpp:90, 106-113
    // Wq, Wk, Wv [d x d] -> rows [0,d), [d,2d), [2d,3d) of Wqkv^T
    for (int k = 0; k < 3; ++k)
        draw_transposed(L + off.wqkv + static_cast<size_t>(k) * d * d, d, d, mix_seed(seed, base + k), fac[k]);
    draw_transposed(L + off.wproj, d, d, mix_seed(seed, base + 3), fac[3]);
    draw_transposed(L + off.w1, d, f, mix_seed(seed, base + 4), fac[4]);
    draw_transposed(L + off.w2, f, d, mix_seed(seed, base + 5), fac[5]);
}

namespace {
// n draws of stream `seed`; entries in blocks [k*blk, (k+1)*blk) with k even get +1
// (LayerNorm gammas), the others stay raw (betas / biases when blk == 0)
void draw_vec(uint16_t* dst, size_t n, uint64_t seed, size_t blk) {
    for (size_t i = 0; i < n; ++i) {
        const uint64_t z = SplitMix64::mix(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
        const double u = -0.1 + (0.1 - -0.1) * (static_cast<double>(z >> 11) * 0x1.0p-53);
        dst[i] = to_f16(blk && (i / blk) % 2 == 0 ? 1.0 + u : u);
    }
}
}  // namespace

void generate_layer_extras(const ModelConfig& c, uint64_t seed, int l, uint16_t* L) {
    const size_t d = c.hidden_dim, f = c.ffn_dim;
    const LayerOffsets off = LayerOffsets::of(c, kArchOpt);
    const uint64_t base = 100 + static_cast<uint64_t>(l) * 8;
    draw_vec(L + off.bqkv, 5 * d + f, mix_seed(seed, base + 6), 0);  // b_qkv | b_o | b_1 | b_2 (contiguous)
    draw_vec(L + off.ln1g, 4 * d, mix_seed(seed, base + 7), d);      // g1 | b1 | g2 | b2
}

void generate_final_ln(const ModelConfig& c, uint64_t seed, uint16_t* dst) {
    draw_vec(dst, 2 * static_cast<size_t>(c.hidden_dim), mix_seed(seed, 2), c.hidden_dim);
}

HostWeights generate_weights(const ModelConfig& config, uint64_t seed, int max_seq, bool rescale) {
    ModelConfig c = config;
    c.validate();
    if (max_seq < 1) throw InputError("DecoderWeights: max_seq must be >= 1");
    HostWeights w;
    w.config = c;
    w.max_seq = max_seq;
    w.embedding.resize(static_cast<size_t>(c.vocab_size) * c.hidden_dim);
    w.positional.resize(static_cast<size_t>(max_seq) * c.hidden_dim);
    generate_tables(c, seed, max_seq, w.embedding.data(), w.positional.data());
    w.layers.resize(LayerOffsets::of(c).total * c.num_layers);
    for (int l = 0; l < c.num_layers; ++l) generate_layer(c, seed, l, rescale, w.layer(l));
    return w;
}

HostWeights weights_from_f64(const ModelConfig& config, int max_seq, const double* emb, const double* pos,
                             const double* const* layer_tensors) {
    ModelConfig c = config;
    c.validate();
    HostWeights w;
    w.config = c;
    w.max_seq = max_seq;
    const int d = c.hidden_dim, f = c.ffn_dim;
    w.embedding.resize(static_cast<size_t>(c.vocab_size) * d);
    w.positional.resize(static_cast<size_t>(max_seq) * d);
    for (size_t i = 0; i < w.embedding.size(); ++i) w.embedding[i] = to_f16(emb[i]);
    for (size_t i = 0; i < w.positional.size(); ++i) w.positional[i] = to_f16(pos[i]);
    const LayerOffsets off = LayerOffsets::of(c);
    w.layers.resize(off.total * c.num_layers);
    auto put_t = [](uint16_t* dst, const double* src, int rows, int cols) {
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < cols; ++k) dst[static_cast<size_t>(k) * rows + r] = to_f16(src[static_cast<size_t>(r) * cols + k]);
    };
    for (int l = 0; l < c.num_layers; ++l) {
        uint16_t* L = w.layer(l);
        const double* const* t = layer_tensors + 6 * l;
        for (int k = 0; k < 3; ++k) put_t(L + off.wqkv + static_cast<size_t>(k) * d * d, t[k], d, d);
        put_t(L + off.wproj, t[3], d, d);
        put_t(L + off.w1, t[4], d, f);
        put_t(L + off.w2, t[5], f, d);
    }
    return w;
}

HostWeights weights_from_f64_opt(const ModelConfig& config, int max_seq, const double* emb, const double* pos,
                                 const double* const* layer_tensors, const double* const* layer_extras,
                                 const double* final_ln) {
    if (!layer_extras || !final_ln) throw InputError("opt arch needs layer extras and the final LayerNorm");
    HostWeights ref = weights_from_f64(config, max_seq, emb, pos, layer_tensors);
    HostWeights w;
    w.config = ref.config;
    w.arch = kArchOpt;
    w.max_seq = max_seq;
    w.embedding = std::move(ref.embedding);
    w.positional = std::move(ref.positional);
    const LayerOffsets r = LayerOffsets::of(w.config), o = LayerOffsets::of(w.config, kArchOpt);
    const size_t d = w.config.hidden_dim, f = w.config.ffn_dim;
    w.layers.resize(o.total * w.config.num_layers);
    for (int l = 0; l < w.config.num_layers; ++l) {
        uint16_t* L = w.layer(l);
        std::memcpy(L, ref.layers.data() + r.total * l, r.total * 2);
        const double* const* e = layer_extras + 10 * l;
        const size_t dst[10] = {o.bqkv, o.bqkv + d, o.bqkv + 2 * d, o.bproj, o.b1, o.b2, o.ln1g, o.ln1b, o.ln2g, o.ln2b};
        for (int k = 0; k < 10; ++k) {
            const size_t n = k == 4 ? f : d;
            for (size_t i = 0; i < n; ++i) L[dst[k] + i] = to_f16(e[k][i]);
        }
    }
    w.final_ln.resize(2 * d);
    for (size_t i = 0; i < 2 * d; ++i) w.final_ln[i] = to_f16(final_ln[i]);
    return w;
}

}  // namespace hc
