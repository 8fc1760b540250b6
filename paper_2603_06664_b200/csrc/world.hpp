// world.hpp -- the communicator behind the sequence-parallel exchanges (reference: CommWorld,
// proj/include/spattn/collectives.hpp:39-113, proj/src/collectives.cpp).
//
// The reference simulates P ranks as threads meeting in a rendezvous. Here a rank is a CUDA
// stream bound to a device, and two transports implement the exchanges:
//   LOCAL : every rank of the world lives in this process (devices may repeat, so P ranks
//           can share one GPU); a chunk moves by direct stores into the destination
//           buffer (peer memory across GPUs), ordering by CUDA events between the streams;
//   NCCL  : one rank per process; grouped ncclSend/ncclRecv, one group == one round;
//   PEER  : one rank per process; the engine maps its peers' exchange buffers through CUDA
//           IPC and its kernels store into them directly, device-side flags order the ranks.
// The traffic ledger (CommStats) counts logical collectives exactly like the reference:
// one per invocation, elements_sent = scalars crossing a rank boundary, sender side.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "../../include/spx.h"

namespace spx {

struct LocalRank {
    int rank = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev = nullptr;  // reusable join event
};

class World {
  public:
    World(int world_size, const int* devices);                            // LOCAL
    World(int rank, int world_size, const uint8_t id[128], int device);  // NCCL
    World(int rank, int world_size, int device);                          // PEER
    ~World();
    World(const World&) = delete;
    World& operator=(const World&) = delete;

    int size() const { return world_size_; }
    int transport() const { return transport_; }
    int num_local() const { return static_cast<int>(local_.size()); }
    const LocalRank& local(int i) const { return local_[static_cast<size_t>(i)]; }
    int first_rank() const { return local_.empty() ? 0 : local_[0].rank; }
    // local index of a global rank, or -1 when it lives in another process
    int local_index(int rank) const;

    // stream of dst_local waits for everything enqueued so far on the listed local ranks
    void record(int local_idx);
    void wait(int dst_local, int src_local);
    void join_all();
    void synchronize();

    // NCCL helpers (transport == NCCL)
    void group_start();
    void group_end();
    void send(const void* buf, size_t bytes, int peer, cudaStream_t s);
    void recv(void* buf, size_t bytes, int peer, cudaStream_t s);
    void check_async();

    // ledger
    void add_stats(int64_t ag, int64_t a2a, int64_t fused, int64_t elements, int64_t rounds);
    spx_comm_stats stats() const;
    void reset_stats();

    // byte-moving collectives on (B, S, H, D) tensors of any element width
    void all_to_all(void* const* in, void* const* out, const int64_t shape[4], int elem_bytes,
                    int scatter_axis, int gather_axis);
    void fused_all_to_all(void* const* const ins[3], void* const* const outs[3],
                          const int64_t shape[4], int elem_bytes, int scatter_axis,
                          int gather_axis);
    void all_gather(void* const* in, void* const* out, const int64_t shape[4], int elem_bytes,
                    int axis);

    // pre-size the NCCL staging buffer (bytes) so that no collective allocates
    void reserve(size_t bytes);

  private:
    void exchange(int n, void* const* const* ins, void* const* const* outs, const int64_t shape[4],
                  int elem_bytes, int scatter_axis, int gather_axis, const char* what);
    uint8_t* staging(size_t bytes);
    void* stage_ = nullptr;
    size_t stage_bytes_ = 0;
    int world_size_ = 1;
    int transport_ = SPX_TRANSPORT_LOCAL;
    std::vector<LocalRank> local_;
    void* comm_ = nullptr;  // ncclComm_t
    mutable std::mutex mu_;
    spx_comm_stats stats_{};
};

// dlopen'd NCCL (the library itself never links NCCL; torch may already have loaded one)
bool nccl_available();
void nccl_unique_id(uint8_t out[128]);

}  // namespace spx
