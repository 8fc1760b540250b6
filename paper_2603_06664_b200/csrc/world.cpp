// world.cpp -- see world.hpp.
#include "world.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "common.hpp"
#include "kernels.hpp"

namespace spx {

// ---------------------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------------------
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank =
            reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.comm_async_error =
            reinterpret_cast<decltype(api.comm_async_error)>(sym("ncclCommGetAsyncError"));
        api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string =
            reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.send &&
                 api.recv && api.group_start && api.group_end && api.error_string &&
                 api.comm_async_error;
        if (!api.ok) api.why = "libnccl.so.2 lacks required symbols";
    });
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        throw Error(SPX_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
    }
}

void strides_of(const int64_t shape[4], int64_t out[4]) {
    out[3] = 1;
    for (int a = 2; a >= 0; --a) out[a] = out[a + 1] * shape[a + 1];
}

int64_t numel(const int64_t s[4]) { return s[0] * s[1] * s[2] * s[3]; }

void validate_shape(const int64_t shape[4]) {
    for (int a = 0; a < 4; ++a)
        require(shape[a] >= 1, SPX_ERR_SHAPE, "all extents must be >= 1");
}

void validate_axis(int axis) {
    require(axis >= 0 && axis < 4, SPX_ERR_CONFIG, "axis out of range");
}

void validate_width(int elem_bytes) {
    require(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
            SPX_ERR_CONFIG, "element width must be 1, 2, 4 or 8 bytes");
}

}  // namespace

bool nccl_available() { return nccl().ok; }

void nccl_unique_id(uint8_t out[128]) {
    require(nccl().ok, SPX_ERR_NCCL, nccl().why);
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

// ---------------------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------------------
World::World(int world_size, const int* devices) : world_size_(world_size) {
    require(world_size >= 1, SPX_ERR_CONFIG,
            "world size must be >= 1, got " + std::to_string(world_size));
    transport_ = SPX_TRANSPORT_LOCAL;
    int cur = 0;
    SPX_CUDA(cudaGetDevice(&cur));
    int ndev = 0;
    SPX_CUDA(cudaGetDeviceCount(&ndev));
    local_.resize(static_cast<size_t>(world_size));
    for (int r = 0; r < world_size; ++r) {
        LocalRank& lr = local_[static_cast<size_t>(r)];
        lr.rank = r;
        lr.device = devices ? devices[r] : cur;
        require(lr.device >= 0 && lr.device < ndev, SPX_ERR_CONFIG,
                "rank " + std::to_string(r) + ": no device " + std::to_string(lr.device));
        SPX_CUDA(cudaSetDevice(lr.device));
        SPX_CUDA(cudaStreamCreateWithFlags(&lr.stream, cudaStreamNonBlocking));
        SPX_CUDA(cudaEventCreateWithFlags(&lr.ev, cudaEventDisableTiming));
    }
    // direct stores between distinct devices need peer access both ways
    for (int a = 0; a < world_size; ++a) {
        for (int b = 0; b < world_size; ++b) {
            const int da = local_[a].device, db = local_[b].device;
            if (da == db) continue;
            int can = 0;
            SPX_CUDA(cudaDeviceCanAccessPeer(&can, da, db));
            require(can == 1, SPX_ERR_CONFIG,
                    "devices " + std::to_string(da) + " and " + std::to_string(db) +
                        " have no peer access (LOCAL transport needs NVLink P2P)");
            SPX_CUDA(cudaSetDevice(da));
            cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else {
                SPX_CUDA(e);
            }
        }
    }
    SPX_CUDA(cudaSetDevice(cur));
}

World::World(int rank, int world_size, const uint8_t id[128], int device)
    : world_size_(world_size) {
    require(world_size >= 1, SPX_ERR_CONFIG, "world size must be >= 1");
    require(rank >= 0 && rank < world_size, SPX_ERR_COLLECTIVE,
            "rank " + std::to_string(rank) + " out of range");
    require(nccl().ok, SPX_ERR_NCCL, nccl().why);
    transport_ = SPX_TRANSPORT_NCCL;
    local_.resize(1);
    LocalRank& lr = local_[0];
    lr.rank = rank;
    lr.device = device;
    SPX_CUDA(cudaSetDevice(device));
    SPX_CUDA(cudaStreamCreateWithFlags(&lr.stream, cudaStreamNonBlocking));
    SPX_CUDA(cudaEventCreateWithFlags(&lr.ev, cudaEventDisableTiming));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclComm_t comm = nullptr;
    nccl_check(nccl().comm_init_rank(&comm, world_size, uid, rank), "ncclCommInitRank");
    comm_ = comm;
}

World::World(int rank, int world_size, int device) : world_size_(world_size) {
    require(world_size >= 1, SPX_ERR_CONFIG, "world size must be >= 1");
    require(rank >= 0 && rank < world_size, SPX_ERR_COLLECTIVE,
            "rank " + std::to_string(rank) + " out of range");
    transport_ = SPX_TRANSPORT_PEER;
    local_.resize(1);
    LocalRank& lr = local_[0];
    lr.rank = rank;
    lr.device = device;
    SPX_CUDA(cudaSetDevice(device));
    SPX_CUDA(cudaStreamCreateWithFlags(&lr.stream, cudaStreamNonBlocking));
    SPX_CUDA(cudaEventCreateWithFlags(&lr.ev, cudaEventDisableTiming));
}

World::~World() {
    for (LocalRank& lr : local_) {
        cudaSetDevice(lr.device);
        if (lr.stream) cudaStreamSynchronize(lr.stream);
        if (lr.ev) cudaEventDestroy(lr.ev);
        if (lr.stream) cudaStreamDestroy(lr.stream);
    }
    if (stage_) {
        cudaSetDevice(local_[0].device);
        cudaFree(stage_);
    }
    if (comm_ && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
}

int World::local_index(int rank) const {
    for (size_t i = 0; i < local_.size(); ++i)
        if (local_[i].rank == rank) return static_cast<int>(i);
    return -1;
}

void World::record(int li) {
    const LocalRank& lr = local_[static_cast<size_t>(li)];
    SPX_CUDA(cudaEventRecord(lr.ev, lr.stream));
}

void World::wait(int dst, int src) {
    if (dst == src) return;
    SPX_CUDA(cudaStreamWaitEvent(local_[static_cast<size_t>(dst)].stream,
                                 local_[static_cast<size_t>(src)].ev, 0));
}

void World::join_all() {
    if (local_.size() < 2) return;
    for (int i = 0; i < num_local(); ++i) {
        SPX_CUDA(cudaSetDevice(local_[i].device));
        record(i);
    }
    for (int d = 0; d < num_local(); ++d) {
        SPX_CUDA(cudaSetDevice(local_[d].device));
        for (int s = 0; s < num_local(); ++s) wait(d, s);
    }
}

void World::synchronize() {
    for (const LocalRank& lr : local_) {
        SPX_CUDA(cudaSetDevice(lr.device));
        SPX_CUDA(cudaStreamSynchronize(lr.stream));
    }
    check_async();
}

void World::group_start() { nccl_check(nccl().group_start(), "ncclGroupStart"); }
void World::group_end() { nccl_check(nccl().group_end(), "ncclGroupEnd"); }

void World::send(const void* buf, size_t bytes, int peer, cudaStream_t s) {
    nccl_check(nccl().send(buf, bytes, ncclUint8, peer, static_cast<ncclComm_t>(comm_), s),
               "ncclSend");
}

void World::recv(void* buf, size_t bytes, int peer, cudaStream_t s) {
    nccl_check(nccl().recv(buf, bytes, ncclUint8, peer, static_cast<ncclComm_t>(comm_), s),
               "ncclRecv");
}

void World::check_async() {
    if (!comm_) return;
    ncclResult_t e = ncclSuccess;
    nccl_check(nccl().comm_async_error(static_cast<ncclComm_t>(comm_), &e),
               "ncclCommGetAsyncError");
    if (e != ncclSuccess && e != ncclInProgress)
        throw Error(SPX_ERR_COLLECTIVE,
                    std::string("communicator failed asynchronously: ") + nccl().error_string(e));
}

void World::add_stats(int64_t ag, int64_t a2a, int64_t fused, int64_t elements, int64_t rounds) {
    std::lock_guard<std::mutex> lk(mu_);
    stats_.all_gather += ag;
    stats_.all_to_all += a2a;
    stats_.fused_all_to_all += fused;
    stats_.elements_sent += elements;
    stats_.rounds += rounds;
}

spx_comm_stats World::stats() const {
    std::lock_guard<std::mutex> lk(mu_);
    return stats_;
}

void World::reset_stats() {
    std::lock_guard<std::mutex> lk(mu_);
    stats_ = spx_comm_stats{};
}

// ---------------------------------------------------------------------------------------
// byte-moving collectives
// ---------------------------------------------------------------------------------------
// Staging for the NCCL byte movers: one device buffer per world, grown (after draining the
// stream) only when a call needs more than any earlier one; spx_world_reserve sizes it up front
// so that the collectives allocate nothing on the hot path.
uint8_t* World::staging(size_t bytes) {
    if (bytes <= stage_bytes_) return static_cast<uint8_t*>(stage_);
    const LocalRank& me = local_[0];
    SPX_CUDA(cudaSetDevice(me.device));
    SPX_CUDA(cudaStreamSynchronize(me.stream));
    if (stage_) SPX_CUDA(cudaFree(stage_));
    stage_ = nullptr;
    stage_bytes_ = 0;
    SPX_CUDA(cudaMalloc(&stage_, bytes));
    stage_bytes_ = bytes;
    return static_cast<uint8_t*>(stage_);
}

void World::reserve(size_t bytes) {
    if (transport_ == SPX_TRANSPORT_NCCL) staging(bytes);
}

// n tensors of one per-rank shape, all chunk j of every tensor -> rank j (gather offset = the
// source rank), in ONE round: LOCAL copies straight between the ranks' buffers; NCCL packs
// [peer][tensor][chunk] into the staging buffer and posts one group of (P-1) sends + (P-1)
// receives, one message per peer carrying all n tensors' chunks.
void World::exchange(int n, void* const* const* ins, void* const* const* outs,
                     const int64_t shape[4], int elem_bytes, int scatter_axis, int gather_axis,
                     const char* what) {
    require(transport_ != SPX_TRANSPORT_PEER, SPX_ERR_UNSUPPORTED,
            "standalone collectives need the LOCAL or NCCL transport (PEER is engine-only)");
    validate_shape(shape);
    validate_width(elem_bytes);
    validate_axis(scatter_axis);
    validate_axis(gather_axis);
    const int P = world_size_;
    require(shape[scatter_axis] % P == 0, SPX_ERR_PARTITION,
            std::string(what) + " scatter extent " + std::to_string(shape[scatter_axis]) +
                " not divisible by world size " + std::to_string(P));
    int64_t piece[4] = {shape[0], shape[1], shape[2], shape[3]};
    piece[scatter_axis] = shape[scatter_axis] / P;
    int64_t oshape[4] = {piece[0], piece[1], piece[2], piece[3]};
    oshape[gather_axis] *= P;
    int64_t in_str[4], out_str[4], piece_str[4];
    strides_of(shape, in_str);
    strides_of(oshape, out_str);
    strides_of(piece, piece_str);
    Box4 box{}, pack{}, unpack{};
    for (int a = 0; a < 4; ++a) {
        box.ext[a] = pack.ext[a] = unpack.ext[a] = piece[a];
        box.src_str[a] = pack.src_str[a] = in_str[a];
        box.dst_str[a] = unpack.dst_str[a] = out_str[a];
        pack.dst_str[a] = unpack.src_str[a] = piece_str[a];
    }
    const size_t eb = static_cast<size_t>(elem_bytes);
    // chunk j of rank i -> rank j, placed at gather offset i
    auto src_off = [&](int j) { return static_cast<size_t>(j * piece[scatter_axis] * in_str[scatter_axis]) * eb; };
    auto dst_off = [&](int i) { return static_cast<size_t>(i * piece[gather_axis] * out_str[gather_axis]) * eb; };

    if (transport_ == SPX_TRANSPORT_LOCAL) {
        join_all();
        for (int j = 0; j < P; ++j) {
            SPX_CUDA(cudaSetDevice(local_[j].device));
            for (int t = 0; t < n; ++t)
                for (int i = 0; i < P; ++i)
                    copy_box_run(static_cast<uint8_t*>(outs[t][j]) + dst_off(i),
                                 static_cast<const uint8_t*>(ins[t][i]) + src_off(j), box,
                                 elem_bytes, local_[j].stream);
        }
        join_all();
        return;
    }
    const LocalRank& me = local_[0];
    const int r = me.rank;
    SPX_CUDA(cudaSetDevice(me.device));
    const size_t pbytes = static_cast<size_t>(numel(piece)) * eb;  // one chunk of one tensor
    const size_t msg = static_cast<size_t>(n) * pbytes;             // everything for one peer
    uint8_t* sendb = staging(2 * static_cast<size_t>(P) * msg);
    uint8_t* recvb = sendb + static_cast<size_t>(P) * msg;
    for (int t = 0; t < n; ++t) {
        for (int j = 0; j < P; ++j) {
            const uint8_t* src = static_cast<const uint8_t*>(ins[t][0]) + src_off(j);
            if (j == r)
                copy_box_run(static_cast<uint8_t*>(outs[t][0]) + dst_off(r), src, box, elem_bytes,
                             me.stream);
            else
                copy_box_run(sendb + j * msg + t * pbytes, src, pack, elem_bytes, me.stream);
        }
    }
    group_start();
    for (int j = 0; j < P; ++j) {
        if (j == r) continue;
        send(sendb + j * msg, msg, j, me.stream);
        recv(recvb + j * msg, msg, j, me.stream);
    }
    group_end();
    for (int t = 0; t < n; ++t)
        for (int i = 0; i < P; ++i) {
            if (i == r) continue;
            copy_box_run(static_cast<uint8_t*>(outs[t][0]) + dst_off(i), recvb + i * msg + t * pbytes,
                         unpack, elem_bytes, me.stream);
        }
}

void World::all_to_all(void* const* in, void* const* out, const int64_t shape[4],
                       int elem_bytes, int scatter_axis, int gather_axis) {
    void* const* ins[1] = {in};
    void* const* outs[1] = {out};
    exchange(1, ins, outs, shape, elem_bytes, scatter_axis, gather_axis, "all_to_all");
    const int P = world_size_;
    add_stats(0, 1, 0, static_cast<int64_t>(P - 1) * numel(shape), 1);
}

void World::fused_all_to_all(void* const* const ins[3], void* const* const outs[3],
                             const int64_t shape[4], int elem_bytes, int scatter_axis,
                             int gather_axis) {
    // one invocation, one round: the three tensors ride the same exchange (one NCCL group)
    exchange(3, ins, outs, shape, elem_bytes, scatter_axis, gather_axis, "fused_all_to_all");
    const int P = world_size_;
    add_stats(0, 0, 1, 3 * static_cast<int64_t>(P - 1) * numel(shape), 1);
}

void World::all_gather(void* const* in, void* const* out, const int64_t shape[4],
                       int elem_bytes, int axis) {
    require(transport_ != SPX_TRANSPORT_PEER, SPX_ERR_UNSUPPORTED,
            "standalone collectives need the LOCAL or NCCL transport (PEER is engine-only)");
    validate_shape(shape);
    validate_width(elem_bytes);
    validate_axis(axis);
    const int P = world_size_;
    int64_t oshape[4] = {shape[0], shape[1], shape[2], shape[3]};
    oshape[axis] *= P;
    int64_t in_str[4], out_str[4];
    strides_of(shape, in_str);
    strides_of(oshape, out_str);
    Box4 box{};
    for (int a = 0; a < 4; ++a) {
        box.ext[a] = shape[a];
        box.src_str[a] = in_str[a];
        box.dst_str[a] = out_str[a];
    }
    const size_t eb = static_cast<size_t>(elem_bytes);
    auto dst_off = [&](int i) { return static_cast<size_t>(i * shape[axis] * out_str[axis]) * eb; };
    if (transport_ == SPX_TRANSPORT_LOCAL) {
        join_all();
        for (int j = 0; j < P; ++j) {
            SPX_CUDA(cudaSetDevice(local_[j].device));
            for (int i = 0; i < P; ++i)
                copy_box_run(static_cast<uint8_t*>(out[j]) + dst_off(i), in[i], box, elem_bytes,
                             local_[j].stream);
        }
        join_all();
    } else {
        const LocalRank& me = local_[0];
        SPX_CUDA(cudaSetDevice(me.device));
        const size_t bytes = static_cast<size_t>(numel(shape)) * eb;
        uint8_t* recvb = staging(static_cast<size_t>(P) * bytes);
        group_start();
        for (int j = 0; j < P; ++j) {
            if (j == me.rank) continue;
            send(in[0], bytes, j, me.stream);
            recv(recvb + j * bytes, bytes, j, me.stream);
        }
        group_end();
        int64_t in_str2[4];
        strides_of(shape, in_str2);
        for (int i = 0; i < P; ++i) {
            const void* src = i == me.rank ? in[0] : static_cast<const void*>(recvb + i * bytes);
            copy_box_run(static_cast<uint8_t*>(out[0]) + dst_off(i), src, box, elem_bytes,
                         me.stream);
        }
    }
    add_stats(1, 0, 0, static_cast<int64_t>(P) * (P - 1) * numel(shape), 1);
}

}  // namespace spx
