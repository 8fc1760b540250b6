// host_rng.hpp -- the reference's reproducible host inputs (proj/src/tensor.cpp:108-159):
// mt19937_64, 53-bit uniforms, Box-Muller (cosine first, sine kept as the spare, u1 <= 0
// clamped to 2^-53), splitmix64 seed derivation. The generator's noise and the seeded layer
// weights must be bit-identical to the reference so the CPU oracle sees the same inputs.
#pragma once

#include <cstdint>
#include <random>

namespace spx {

class HostRng {
  public:
    explicit HostRng(uint64_t seed) : engine_(seed) {}
    uint64_t next_u64() { return engine_(); }
    double next_uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double next_normal();

  private:
    std::mt19937_64 engine_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b = 0, uint64_t c = 0);

// N(0,1)/sqrt(head_dim) * n  (random_tensor)
void fill_noise(uint64_t stream_seed, int64_t n, int64_t head_dim, double* out);
// N(0,1)/sqrt(cols), rows*cols  (Matrix::random)
void fill_matrix(uint64_t stream_seed, int64_t rows, int64_t cols, double* out);

// round-to-nearest-even double -> bf16 bits
uint16_t f64_to_bf16(double x);
double bf16_to_f64(uint16_t b);

}  // namespace spx
