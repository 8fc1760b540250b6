// exchange_plan.hpp -- who sends which slab to whom in the two per-call exchanges of the
// optimized schedule (reference: fused_all_to_all + all_to_all, proj/src/sp_attention.cpp:244,
// :307; permutation semantics proj/src/collectives.cpp:203-276), generalised to P = G x S
// (G head groups, S query splits).
//
// Rank r: head group g = r mod G, query split p = r / G. Source i owns token rows
// [i L/P, (i+1) L/P), which lie in split i / G.
//   qkv exchange: q of group g  -> rank (p_i, g)            rows (i mod G) L/P of its q buffer
//                 k,v of group g -> every rank (*, g)       ring rows base + i L/P
//   out exchange: o rows of source i (split p) -> rank i    slab g of its o buffer
// Only cross-rank transfers are listed (the self part is stored in place by the kernels).
// Within one peer pair the list order is the FIFO order both sides post (q, k, v), which is
// what NCCL (and gloo, in the CPU tests) match sends to receives by.
#pragma once

#include <cstdint>
#include <vector>

namespace spx {

enum ExchangeBuf : int32_t {
    kBufQSend = 0,  // [G][L/P][H/G][D]
    kBufKSend = 1,
    kBufVSend = 2,
    kBufOSend = 3,  // [G][L/P][H/G*D]   chunk c -> source p*G + c
    kBufQRecv = 4,  // [L/S][H/G][D]
    kBufRingK = 5,  // ring rows of this layer
    kBufRingV = 6,
    kBufORecv = 7,  // [G][L/P][H/G*D]
};

struct Transfer {
    int32_t peer;
    int32_t is_send;
    int32_t buf;
    int64_t offset;  // elements from the buffer base
    int64_t elems;
};

struct Partition {
    int64_t P, G, S, L, Lp, Lq, H, Hl, D;
    static Partition make(int64_t world, int64_t heads, int64_t block_len, int64_t head_dim);
    int64_t slab() const { return Lp * Hl * D; }
};

std::vector<Transfer> plan_qkv_exchange(const Partition& pt, int rank, int64_t block_base_row);
std::vector<Transfer> plan_out_exchange(const Partition& pt, int rank);

// elements crossing a rank boundary per call (the CommStats ledger)
int64_t qkv_exchange_elements(const Partition& pt);
int64_t out_exchange_elements(const Partition& pt);

}  // namespace spx
