// exchange_plan.cpp -- see exchange_plan.hpp.
#include "exchange_plan.hpp"

#include "common.hpp"
#include "engine.hpp"

namespace spx {

Partition Partition::make(int64_t world, int64_t heads, int64_t block_len, int64_t head_dim) {
    require(world >= 1 && block_len % world == 0, SPX_ERR_PARTITION,
            "block length " + std::to_string(block_len) + " not divisible by world size " +
                std::to_string(world));
    Partition p{};
    p.P = world;
    p.G = choose_head_groups(world, heads);
    p.S = world / p.G;
    p.L = block_len;
    p.Lp = block_len / world;
    p.Lq = block_len / p.S;
    p.H = heads;
    p.Hl = heads / p.G;
    p.D = head_dim;
    return p;
}

std::vector<Transfer> plan_qkv_exchange(const Partition& pt, int rank, int64_t block_base_row) {
    std::vector<Transfer> t;
    const int64_t slab = pt.slab();
    const int64_t row = pt.Hl * pt.D;
    const int64_t p = rank / pt.G;
    // sends: q to the G ranks of this split, then k and v to every rank (per-peer order q,k,v)
    for (int64_t g = 0; g < pt.G; ++g) {
        const int d = static_cast<int>(p * pt.G + g);
        if (d != rank) t.push_back({d, 1, kBufQSend, g * slab, slab});
    }
    for (int d = 0; d < pt.P; ++d) {
        if (d == rank) continue;
        const int64_t gd = d % pt.G;
        t.push_back({d, 1, kBufKSend, gd * slab, slab});
        t.push_back({d, 1, kBufVSend, gd * slab, slab});
    }
    // receives: q from the sources of this split, then k and v from every source
    for (int64_t c = 0; c < pt.G; ++c) {
        const int i = static_cast<int>(p * pt.G + c);
        if (i != rank) t.push_back({i, 0, kBufQRecv, c * slab, slab});
    }
    for (int i = 0; i < pt.P; ++i) {
        if (i == rank) continue;
        const int64_t r0 = (block_base_row + i * pt.Lp) * row;
        t.push_back({i, 0, kBufRingK, r0, slab});
        t.push_back({i, 0, kBufRingV, r0, slab});
    }
    return t;
}

std::vector<Transfer> plan_out_exchange(const Partition& pt, int rank) {
    std::vector<Transfer> t;
    const int64_t slab = pt.slab();
    const int64_t p = rank / pt.G;
    for (int64_t c = 0; c < pt.G; ++c) {
        const int i = static_cast<int>(p * pt.G + c);
        if (i != rank) t.push_back({i, 1, kBufOSend, c * slab, slab});
    }
    for (int64_t c = 0; c < pt.G; ++c) {
        const int j = static_cast<int>(p * pt.G + c);
        if (j != rank) t.push_back({j, 0, kBufORecv, (j % pt.G) * slab, slab});
    }
    return t;
}

int64_t qkv_exchange_elements(const Partition& pt) {
    return pt.P * ((pt.G - 1) + 2 * (pt.P - 1)) * pt.slab();
}

int64_t out_exchange_elements(const Partition& pt) { return pt.P * (pt.G - 1) * pt.slab(); }

}  // namespace spx
