// spattn_oracle.cpp -- CPU ORACLE (test infrastructure only; never linked into the product).
//
// A plain fp64 restatement of the reference's P = 1 path, in the reference's own loop and
// operation order so its outputs are bit-identical to proj/ (pinned against the FNV-1a
// checksums of SURVEY.md Appendix A in tests/test_oracle.py):
//
//   Rng / derive_seed / random_tensor .......... proj/src/tensor.cpp:108-159
//   scaled_dot_product_attention ............... proj/src/tensor.cpp:161-209
//   BandSplit / precompute_frequencies ......... proj/src/rope.cpp:15-64
//   global_time_index / rotate_rows ............ proj/src/rope.cpp:66-131
//   Matrix::random / AttentionLayerParams ...... proj/src/sp_attention.cpp:8-40
//   project_tokens ............................. proj/src/sp_attention.cpp:51-75
//   reference_self_attention ................... proj/src/sp_attention.cpp:317-348
//   KvCache::update / read ..................... proj/src/kv_cache.cpp:18-67
//   generate (reference variant, P = 1) ........ proj/src/generator.cpp:50-147
//   tensor_checksum (FNV-1a) ................... proj/src/report.cpp:264-279
//
// Extensions with no reference counterpart (off by default): bf16 rounding of the synthetic
// inputs (the device consumes bf16), caller-supplied weights/noise, QK-RMSNorm over the model
// dimension (Wan mode) applied to q and k before RoPE.
//
// Exposed through a C interface for ctypes (oracle/oracle.py).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <random>
#include <vector>

namespace {

// ---- RNG -----------------------------------------------------------------------------------
struct Rng {
    std::mt19937_64 eng;
    bool spare_ok = false;
    double spare = 0.0;
    explicit Rng(uint64_t s) : eng(s) {}
    double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double normal() {
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        double u1 = uniform();
        double u2 = uniform();
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double phi = 2.0 * 3.14159265358979323846 * u2;
        spare = r * std::sin(phi);
        spare_ok = true;
        return r * std::cos(phi);
    }
};

uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

uint64_t seed_of(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t s = mix64(base);
    s = mix64(s ^ mix64(a + 0x1000));
    s = mix64(s ^ mix64(b + 0x2000));
    s = mix64(s ^ mix64(c + 0x3000));
    return s;
}

double round_bf16(double x) {
    // round-to-nearest-even to 8 significant bits (bf16), returned as a double
    if (x == 0.0 || !std::isfinite(x)) return x;
    uint64_t bits;
    std::memcpy(&bits, &x, 8);
    const uint64_t sign = bits & 0x8000000000000000ULL;
    uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFULL;
    mag = (mag + 0xFFFFFFFFFFFULL + ((mag >> 45) & 1u)) & ~((1ULL << 45) - 1);
    bits = sign | mag;
    double y;
    std::memcpy(&y, &bits, 8);
    return y;
}

// ---- table -------------------------------------------------------------------------------
struct Table {
    int64_t ext[3];
    int64_t pairs[3];
    std::vector<double> cs[3];  // (cos, sin) interleaved per (pos, pair)
    Table(int64_t frames, int64_t hh, int64_t ww, int64_t pT, int64_t pH, int64_t pW, double base)
        : ext{frames, hh, ww}, pairs{pT, pH, pW} {
        for (int b = 0; b < 3; ++b) {
            cs[b].assign(static_cast<size_t>(ext[b] * pairs[b] * 2), 0.0);
            for (int64_t m = 0; m < ext[b]; ++m)
                for (int64_t j = 0; j < pairs[b]; ++j) {
                    const double f =
                        std::pow(base, -static_cast<double>(j) / static_cast<double>(pairs[b]));
                    const double a = static_cast<double>(m) * f;
                    cs[b][static_cast<size_t>((m * pairs[b] + j) * 2)] = std::cos(a);
                    cs[b][static_cast<size_t>((m * pairs[b] + j) * 2 + 1)] = std::sin(a);
                }
        }
    }
};

// rows [0, rows) of x (rows, H, D) are global positions row_offset + i of the block
void rope_rows(double* x, int64_t rows, int64_t H, int64_t D, const Table& t, int64_t Wg,
               int64_t hw, int64_t start, int64_t row_offset) {
    for (int64_t i = 0; i < rows; ++i) {
        const int64_t ig = row_offset + i;
        const int64_t pos[3] = {start + ig / hw, (ig % hw) / Wg, ig % Wg};
        for (int64_t h = 0; h < H; ++h) {
            double* row = x + (i * H + h) * D;
            int64_t j = 0;
            for (int b = 0; b < 3; ++b) {
                for (int64_t jj = 0; jj < t.pairs[b]; ++jj, ++j) {
                    const double c = t.cs[b][static_cast<size_t>((pos[b] * t.pairs[b] + jj) * 2)];
                    const double s = t.cs[b][static_cast<size_t>((pos[b] * t.pairs[b] + jj) * 2 + 1)];
                    const double a = row[2 * j], bb = row[2 * j + 1];
                    row[2 * j] = a * c - bb * s;
                    row[2 * j + 1] = a * s + bb * c;
                }
            }
        }
    }
}

void project(const double* x, const double* W, double* y, int64_t tokens, int64_t dim) {
    for (int64_t s = 0; s < tokens; ++s) {
        const double* in = x + s * dim;
        double* out = y + s * dim;
        for (int64_t o = 0; o < dim; ++o) {
            const double* w = W + o * dim;
            double acc = 0.0;
            for (int64_t j = 0; j < dim; ++j) acc += w[j] * in[j];
            out[o] = acc;
        }
    }
}

void sdpa(const double* q, const double* k, const double* v, double* out, int64_t Sq,
          int64_t Skv, int64_t H, int64_t D) {
    const double inv = 1.0 / std::sqrt(static_cast<double>(D));
    std::vector<double> wts(static_cast<size_t>(Skv));
    for (int64_t h = 0; h < H; ++h) {
        for (int64_t i = 0; i < Sq; ++i) {
            double m = -HUGE_VAL;
            const double* qi = q + (i * H + h) * D;
            for (int64_t t = 0; t < Skv; ++t) {
                const double* kt = k + (t * H + h) * D;
                double dot = 0.0;
                for (int64_t d = 0; d < D; ++d) dot += qi[d] * kt[d];
                const double l = dot * inv;
                wts[static_cast<size_t>(t)] = l;
                if (l > m) m = l;
            }
            double z = 0.0;
            for (int64_t t = 0; t < Skv; ++t) {
                const double e = std::exp(wts[static_cast<size_t>(t)] - m);
                wts[static_cast<size_t>(t)] = e;
                z += e;
            }
            const double iz = 1.0 / z;
            double* oi = out + (i * H + h) * D;
            for (int64_t d = 0; d < D; ++d) {
                double acc = 0.0;
                for (int64_t t = 0; t < Skv; ++t) acc += wts[static_cast<size_t>(t)] * v[(t * H + h) * D + d];
                oi[d] = acc * iz;
            }
        }
    }
}

void rms_norm(double* x, const double* w, int64_t tokens, int64_t dim, double eps) {
    for (int64_t s = 0; s < tokens; ++s) {
        double* r = x + s * dim;
        double ss = 0.0;
        for (int64_t c = 0; c < dim; ++c) ss += r[c] * r[c];
        const double scale = 1.0 / std::sqrt(ss / static_cast<double>(dim) + eps);
        for (int64_t c = 0; c < dim; ++c) r[c] = r[c] * scale * (w ? w[c] : 1.0);
    }
}

// Wan adaLN modulation (extension; no reference counterpart): non-affine LayerNorm
// over the model dim (biased variance, eps inside the sqrt), then x * (1 + scale) + shift.
void layernorm_modulate(const double* x, double* y, const double* shift, const double* scale,
                        int64_t tokens, int64_t dim, double eps) {
    for (int64_t s = 0; s < tokens; ++s) {
        const double* r = x + s * dim;
        double* o = y + s * dim;
        double mean = 0.0;
        for (int64_t c = 0; c < dim; ++c) mean += r[c];
        mean /= static_cast<double>(dim);
        double var = 0.0;
        for (int64_t c = 0; c < dim; ++c) var += (r[c] - mean) * (r[c] - mean);
        var /= static_cast<double>(dim);
        const double rstd = 1.0 / std::sqrt(var + eps);
        for (int64_t c = 0; c < dim; ++c)
            o[c] = (r[c] - mean) * rstd * (1.0 + scale[c]) + shift[c];
    }
}

// ---- KV cache ---------------------------------------------------------------------------
struct Cache {
    int64_t tpf, row;  // tokens per frame, elements per token
    int64_t window;    // < 0 unlimited
    struct Frame {
        int64_t block;
        std::vector<double> k, v;
    };
    std::deque<Frame> frames;
    void update(int64_t block, const double* k, const double* v, int64_t seq) {
        while (!frames.empty() && frames.back().block == block) frames.pop_back();
        const int64_t n = seq / tpf;
        const size_t fe = static_cast<size_t>(tpf * row);
        for (int64_t f = 0; f < n; ++f)
            frames.push_back(Frame{block, std::vector<double>(k + f * fe, k + (f + 1) * fe),
                                   std::vector<double>(v + f * fe, v + (f + 1) * fe)});
        if (window >= 0)
            while (static_cast<int64_t>(frames.size()) > window) frames.pop_front();
    }
    void read(std::vector<double>& k, std::vector<double>& v) const {
        k.clear();
        v.clear();
        for (const Frame& f : frames) {
            k.insert(k.end(), f.k.begin(), f.k.end());
            v.insert(v.end(), f.v.begin(), f.v.end());
        }
    }
};

}  // namespace

extern "C" {

uint64_t oracle_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    return seed_of(base, a, b, c);
}

void oracle_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.eng();
}

void oracle_rng_normal(uint64_t seed, int64_t n, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

double oracle_round_bf16(double x) { return round_bf16(x); }

void oracle_block_noise(uint64_t seed, int64_t block, int64_t step, int64_t n, int64_t D,
                        double* out) {
    Rng r(seed_of(seed, 0x10, static_cast<uint64_t>(block), static_cast<uint64_t>(step)));
    const double scale = 1.0 / std::sqrt(static_cast<double>(D));
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal() * scale;
}

void oracle_layer_weights(uint64_t seed, int64_t layer, int64_t dim, double* w4) {
    const uint64_t base = seed_of(seed, 0x20, static_cast<uint64_t>(layer), 0);
    const double scale = 1.0 / std::sqrt(static_cast<double>(dim));
    for (int m = 0; m < 4; ++m) {
        Rng r(seed_of(base, 11 + m, 0, 0));
        double* w = w4 + m * dim * dim;
        for (int64_t i = 0; i < dim * dim; ++i) w[i] = r.normal() * scale;
    }
}

void oracle_band_split(int64_t D, int64_t out[3]) {
    const int64_t pairs = D / 2, sp = pairs / 3;
    out[0] = pairs - 2 * sp;
    out[1] = sp;
    out[2] = sp;
}

// cos/sin of one table entry
void oracle_table_at(int64_t frames, int64_t hh, int64_t ww, int64_t D, double base,
                     const int64_t* split, int band, int64_t pos, int64_t pair, double* c,
                     double* s) {
    int64_t sp[3];
    if (split) {
        sp[0] = split[0];
        sp[1] = split[1];
        sp[2] = split[2];
    } else {
        oracle_band_split(D, sp);
    }
    const double f = std::pow(base, -static_cast<double>(pair) / static_cast<double>(sp[band]));
    const double a = static_cast<double>(pos) * f;
    (void)frames;
    (void)hh;
    (void)ww;
    *c = std::cos(a);
    *s = std::sin(a);
}

int64_t oracle_global_time_index(int64_t i_local, int64_t rank, int64_t local_len, int64_t hw,
                                 int64_t start) {
    return start + (rank * local_len + i_local) / hw;
}

// x: (rows, H, D) fp64, rotated in place as rank `rank` of `world` (rows = L/P)
void oracle_rope_causal_local(double* x, int64_t rows, int64_t H, int64_t D, int64_t F,
                              int64_t Hg, int64_t Wg, int64_t max_frames, double base,
                              const int64_t* split, int64_t start, int64_t rank) {
    int64_t sp[3];
    if (split) {
        sp[0] = split[0];
        sp[1] = split[1];
        sp[2] = split[2];
    } else {
        oracle_band_split(D, sp);
    }
    (void)F;
    Table t(max_frames, Hg, Wg, sp[0], sp[1], sp[2], base);
    rope_rows(x, rows, H, D, t, Wg, Hg * Wg, start, rank * rows);
}

void oracle_project(const double* x, const double* W, double* y, int64_t tokens, int64_t dim) {
    project(x, W, y, tokens, dim);
}

void oracle_sdpa(const double* q, const double* k, const double* v, double* out, int64_t Sq,
                 int64_t Skv, int64_t H, int64_t D) {
    sdpa(q, k, v, out, Sq, Skv, H, D);
}

void oracle_rms_norm(double* x, const double* w, int64_t tokens, int64_t dim, double eps) {
    rms_norm(x, w, tokens, dim, eps);
}

void oracle_layernorm_modulate(const double* x, double* y, const double* shift,
                               const double* scale, int64_t tokens, int64_t dim, double eps) {
    layernorm_modulate(x, y, shift, scale, tokens, dim, eps);
}

uint64_t oracle_checksum(const double* p, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t bits;
        std::memcpy(&bits, &p[i], 8);
        for (int byte = 0; byte < 8; ++byte) {
            h ^= (bits >> (8 * byte)) & 0xFFULL;
            h *= 0x100000001b3ULL;
        }
    }
    return h;
}

// generate() with the reference (P = 1) pipeline.
//   cfg: frames, Hg, Wg, num_blocks, layers, steps, heads, head_dim, window (<0 unlimited),
//        force_start_frame_zero, round_inputs_bf16, qk_norm, adaln
//   weights: NULL (seeded) or layers x 4 x dim x dim ([q|k|v|o], [out][in])
//   noise:   NULL (seeded) or num_blocks x steps x L x dim
//   norm_w:  NULL (ones) or layers x 2 x dim  (only with qk_norm)
//   mod:     layers x 3 x dim [shift | scale | gate] (only with adaln, the Wan block's
//            self-attention modulation: x_in = LN(x)(1 + scale) + shift, x += gate * W_o o)
//   out:     num_blocks x L x dim
//   layer_out (optional): num_blocks x steps x layers x L x dim (every call's output)
void oracle_generate(const int64_t* cfg, uint64_t seed, double base, const int64_t* split,
                     const double* weights, const double* noise, const double* norm_w,
                     const double* mod, double norm_eps, double* out, double* layer_out) {
    const int64_t F = cfg[0], Hg = cfg[1], Wg = cfg[2], blocks = cfg[3], layers = cfg[4],
                  steps = cfg[5], H = cfg[6], D = cfg[7], window = cfg[8], force0 = cfg[9],
                  round_in = cfg[10], qk_norm = cfg[11], adaln = cfg[12];
    const int64_t hw = Hg * Wg, L = F * hw, dim = H * D;
    int64_t sp[3];
    if (split) {
        sp[0] = split[0];
        sp[1] = split[1];
        sp[2] = split[2];
    } else {
        oracle_band_split(D, sp);
    }
    Table table(blocks * F, Hg, Wg, sp[0], sp[1], sp[2], base);
    const size_t mat = static_cast<size_t>(dim * dim);
    std::vector<double> W(static_cast<size_t>(layers) * 4 * mat);
    for (int64_t l = 0; l < layers; ++l) {
        double* w = W.data() + l * 4 * mat;
        if (weights) {
            std::memcpy(w, weights + l * 4 * mat, 4 * mat * sizeof(double));
        } else {
            oracle_layer_weights(seed, l, dim, w);
        }
        if (round_in)
            for (size_t i = 0; i < 4 * mat; ++i) w[i] = round_bf16(w[i]);
    }
    std::vector<Cache> caches(static_cast<size_t>(layers), Cache{hw, dim, window, {}});
    const size_t be = static_cast<size_t>(L * dim);
    std::vector<double> x(be), q(be), k(be), v(be), o(be), xm(adaln ? be : 0), ck, cv;
    for (int64_t b = 0; b < blocks; ++b) {
        const int64_t start = force0 ? 0 : b * F;
        for (int64_t s = 0; s < steps; ++s) {
            if (noise) {
                std::memcpy(x.data(), noise + (b * steps + s) * be, be * sizeof(double));
            } else {
                oracle_block_noise(seed, b, s, static_cast<int64_t>(be), D, x.data());
            }
            if (round_in)
                for (double& e : x) e = round_bf16(e);
            for (int64_t l = 0; l < layers; ++l) {
                const double* w = W.data() + l * 4 * mat;
                const double* xin = x.data();
                if (adaln) {
                    const double* m = mod + l * 3 * dim;
                    layernorm_modulate(x.data(), xm.data(), m, m + dim, L, dim, norm_eps);
                    xin = xm.data();
                }
                project(xin, w, q.data(), L, dim);
                project(xin, w + mat, k.data(), L, dim);
                project(xin, w + 2 * mat, v.data(), L, dim);
                if (qk_norm) {
                    rms_norm(q.data(), norm_w ? norm_w + l * 2 * dim : nullptr, L, dim, norm_eps);
                    rms_norm(k.data(), norm_w ? norm_w + l * 2 * dim + dim : nullptr, L, dim,
                             norm_eps);
                }
                rope_rows(q.data(), L, H, D, table, Wg, hw, start, 0);
                rope_rows(k.data(), L, H, D, table, Wg, hw, start, 0);
                Cache& c = caches[static_cast<size_t>(l)];
                c.update(b, k.data(), v.data(), L);
                c.read(ck, cv);
                sdpa(q.data(), ck.data(), cv.data(), o.data(), L,
                     static_cast<int64_t>(ck.size()) / dim, H, D);
                if (adaln) {  // residual + gate (x += gate * W_o o)
                    const double* gate = mod + l * 3 * dim + 2 * dim;
                    project(o.data(), w + 3 * mat, q.data(), L, dim);
                    for (int64_t t = 0; t < L; ++t)
                        for (int64_t c = 0; c < dim; ++c)
                            x[static_cast<size_t>(t * dim + c)] += gate[c] * q[static_cast<size_t>(t * dim + c)];
                } else {
                    project(o.data(), w + 3 * mat, x.data(), L, dim);
                }
                if (layer_out)
                    std::memcpy(layer_out + ((b * steps + s) * layers + l) * be, x.data(),
                                be * sizeof(double));
            }
        }
        std::memcpy(out + b * be, x.data(), be * sizeof(double));
    }
}

}  // extern "C"
