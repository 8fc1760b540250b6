// host_rng.cpp -- see host_rng.hpp. Restates Rng / derive_seed / random_tensor /
// Matrix::random (proj/src/tensor.cpp:108-159, proj/src/sp_attention.cpp:8-15).
#include "host_rng.hpp"

#include <cmath>
#include <cstring>

namespace spx {

double HostRng::next_normal() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1 = next_uniform();
    const double u2 = next_uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;  // fixed draw count: clamp instead of resampling
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
}

uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
    auto splitmix = [](uint64_t x) {
        x += 0x9E3779B97F4A7C15ULL;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
        return x ^ (x >> 31);
    };
    uint64_t s = splitmix(base);
    s = splitmix(s ^ splitmix(a + 0x1000));
    s = splitmix(s ^ splitmix(b + 0x2000));
    s = splitmix(s ^ splitmix(c + 0x3000));
    return s;
}

void fill_noise(uint64_t stream_seed, int64_t n, int64_t head_dim, double* out) {
    HostRng rng(stream_seed);
    const double scale = 1.0 / std::sqrt(static_cast<double>(head_dim));
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next_normal() * scale;
}

void fill_matrix(uint64_t stream_seed, int64_t rows, int64_t cols, double* out) {
    HostRng rng(stream_seed);
    const double scale = 1.0 / std::sqrt(static_cast<double>(cols));
    const int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next_normal() * scale;
}

uint16_t f64_to_bf16(double x) {
    uint64_t bits;
    std::memcpy(&bits, &x, sizeof(bits));
    const uint16_t sign = static_cast<uint16_t>((bits >> 48) & 0x8000u);
    const uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFULL;
    if (mag > 0x7FF0000000000000ULL) return static_cast<uint16_t>(sign | 0x7FC0u);  // NaN
    if (mag == 0) return sign;
    // round the 52-bit mantissa to 7 bits, nearest-even, carry into the exponent
    const uint64_t rounded = (mag + 0xFFFFFFFFFFFULL + ((mag >> 45) & 1u)) >> 45;
    const int64_t exp11 = static_cast<int64_t>(rounded >> 7);
    const int64_t e8 = exp11 - 1023 + 127;
    if (e8 >= 255) return static_cast<uint16_t>(sign | 0x7F80u);  // overflow -> inf
    if (e8 >= 1) return static_cast<uint16_t>(sign | (e8 << 7) | (rounded & 0x7Fu));
    // bf16 subnormal range: go through float (exact for these tiny magnitudes' purposes)
    float f = static_cast<float>(x);
    uint32_t fb;
    std::memcpy(&fb, &f, sizeof(fb));
    const uint32_t r = fb + 0x7FFFu + ((fb >> 16) & 1u);
    return static_cast<uint16_t>(r >> 16);
}

double bf16_to_f64(uint16_t b) {
    const uint32_t fb = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &fb, sizeof(f));
    return static_cast<double>(f);
}

}  // namespace spx
