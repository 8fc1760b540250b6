// adapter_check.cpp -- compiles integration/spx_adapter.hpp against the reference's own headers
// and sources (rope.cpp / tensor.cpp / generator.cpp, compiled in place by integration/Makefile)
// and exercises the host-side calls that need no GPU: the RoPE table built by libspx equals the
// reference's precompute_frequencies bit for bit, global_time_index agrees, and libspx's status
// codes arrive as the reference's exception classes. With a GPU present it also runs the
// reference's desk configuration through spx_adapter::generate and compares with the
// reference's own generate() (bf16 tolerance). Prints one line per check; exit 0 = all passed.
#include <cmath>
#include <cstdio>

#include "spx_adapter.hpp"

using namespace spattn;

static int failures = 0;
#define EXPECT(cond, what)                                         \
    do {                                                           \
        if (cond) {                                                \
            std::printf("ok   %s\n", what);                        \
        } else {                                                   \
            std::printf("FAIL %s\n", what);                        \
            ++failures;                                            \
        }                                                          \
    } while (0)

int main() {
    // 1. RoPE tables: libspx (host fp64, the values the device copies) == the reference
    for (int64_t D : {16, 64, 128}) {
        const BandSplit sp = BandSplit::defaults_for(D);
        const RopeFrequencyTable ref = spattn::precompute_frequencies(21, 30, 52, D, 10000.0, sp);
        auto t = spx_adapter::precompute_frequencies(21, 30, 52, D, 10000.0, sp);
        bool same = true;
        const int64_t ext[3] = {21, 30, 52};
        for (int b = 0; b < 3; ++b)
            for (int64_t m = 0; m < ext[b]; ++m)
                for (int64_t j = 0; j < ref.pairs(static_cast<Band>(b)); ++j) {
                    double c = 0, s = 0;
                    spx_adapter::check(spx_rope_table_at(t.get(), b, m, j, &c, &s));
                    same = same && c == ref.cos_at(static_cast<Band>(b), m, j) &&
                           s == ref.sin_at(static_cast<Band>(b), m, j);
                }
        char what[96];
        std::snprintf(what, sizeof(what), "rope table D=%lld bit-identical to precompute_frequencies",
                      static_cast<long long>(D));
        EXPECT(same, what);
    }
    // 2. global_time_index sweep (rope.cpp:66-70), incl. the Wan P = 8 cases of SURVEY App. A
    bool gti = true;
    for (int64_t P : {1, 2, 4, 8})
        for (int64_t r = 0; r < P; ++r)
            for (int64_t i : {int64_t(0), int64_t(1), int64_t(583), int64_t(584)})
                for (int64_t s : {int64_t(0), int64_t(3), int64_t(18), int64_t(237)})
                    gti = gti && spx_adapter::global_time_index(i, r, 4680 / P, 1560, s) ==
                                     spattn::global_time_index(i, r, 4680 / P, 1560, s);
    EXPECT(gti, "global_time_index == reference over P, rank, row, start_frame");
    // 3. error taxonomy across the ABI
    bool cfg_err = false;
    try {
        spx_adapter::precompute_frequencies(3, 4, 4, 15, 10000.0, BandSplit{4, 2, 1});
    } catch (const ConfigError&) {
        cfg_err = true;
    }
    EXPECT(cfg_err, "odd head_dim -> spattn::ConfigError");
    bool part_err = false;
    try {
        GenerationConfig g;
        g.world_size = 5;  // 48 tokens % 5 != 0
        spx_adapter::validate(g);
    } catch (const PartitionError&) {
        part_err = true;
    }
    EXPECT(part_err, "block length not divisible by P -> spattn::PartitionError");
    GenerationConfig desk;  // the reference defaults (D = 16)
    bool ok = true;
    try {
        spx_adapter::validate(desk);
    } catch (...) {
        ok = false;
    }
    EXPECT(ok, "the reference's default GenerationConfig validates on the device path");
    // 4. with a GPU: generate() through the adapter vs the reference's generate()
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
        for (int P : {1, 2, 4, 8}) {
            desk.world_size = P;
            const std::vector<Tensor4> got = spx_adapter::generate(desk);
            GenerationConfig rc = desk;
            rc.world_size = 1;
            rc.variant = PipelineVariant::reference();
            const GenerationResult ref = spattn::generate(rc);
            double worst = 0;
            for (size_t b = 0; b < got.size(); ++b) {
                double num = 0, den = 0;
                const Tensor4& a = got[b];
                const Tensor4& r = ref.block_outputs[b];
                for (int64_t i = 0; i < a.numel(); ++i) {
                    num += (a.data()[i] - r.data()[i]) * (a.data()[i] - r.data()[i]);
                    den += r.data()[i] * r.data()[i];
                }
                worst = std::fmax(worst, std::sqrt(num / den));
            }
            char what[96];
            std::snprintf(what, sizeof(what), "desk generate() P=%d vs reference: rel-L2 %.2e < 1e-2", P,
                          worst);
            EXPECT(worst < 1e-2, what);
        }
    } else {
        std::printf("skip generate() vs reference (no GPU)\n");
    }
    std::printf(failures ? "adapter FAILED\n" : "adapter ok\n");
    return failures ? 1 : 0;
}
