// rng.cpp — host generation of the Gaussian sketch matrices Ω.
//
// Bit-identical to the reference's gaussian_matrix (src/kernels.cpp:88-101) and
// RngSeed::substream (src/kernels.cpp:14-25): both use libstdc++'s
// std::mt19937_64 and std::normal_distribution<double> (Marsaglia polar method,
// second deviate cached), seeded through splitmix64, filled column by column.
// The stream is inherently sequential, so Ω is produced once on the host and
// cached on the device (SURVEY.md §8(d) timing boundary).
#include <cstdint>
#include <random>
#include <stdexcept>

namespace ts {

std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void substream(std::uint64_t seed, std::uint64_t stream, std::uint64_t salt, std::uint64_t* out_seed,
               std::uint64_t* out_stream) {
    *out_seed = seed;
    *out_stream = splitmix64(stream ^ splitmix64(salt));
}

void gaussian_fill(std::int64_t rows, std::int64_t cols, std::uint64_t seed, std::uint64_t stream, double* out) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("gaussian_matrix: negative extent");
    std::mt19937_64 engine(splitmix64(seed) ^ splitmix64(splitmix64(stream) + 0x6a09e667f3bcc909ULL));
    std::normal_distribution<double> normal(0.0, 1.0);
    for (std::int64_t j = 0; j < cols; ++j)
        for (std::int64_t i = 0; i < rows; ++i) out[i + j * rows] = normal(engine);
}

}  // namespace ts
