// common.hpp -- host-side error taxonomy and CUDA checking for the spx library.
//
// The C++ side throws spx::Error carrying an spx_status; every extern "C" entry point
// converts it into a status code plus a thread-local message (spx_last_error). The status
// set is 1:1 with the reference's exception classes (proj/include/spattn/errors.hpp:8-36).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/spx.h"

namespace spx {

struct Error : std::runtime_error {
    spx_status status;
    Error(spx_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

[[noreturn]] inline void fail(spx_status s, const std::string& what) { throw Error(s, what); }

inline void require(bool cond, spx_status s, const std::string& what) {
    if (!cond) fail(s, what);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Error(SPX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " at " +
                                      file + ":" + std::to_string(line));
    }
}

#define SPX_CUDA(call) ::spx::cuda_check((call), #call, __FILE__, __LINE__)
#define SPX_CUDA_LAUNCH() ::spx::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

void set_last_error(const std::string& msg);

template <class F>
spx_status guarded(F&& f) {
    try {
        f();
        return SPX_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc& e) {
        set_last_error(std::string("host allocation failed: ") + e.what());
        return SPX_ERR_CUDA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SPX_ERR_CONFIG;
    }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Device-side kernel launch counter (the bench's gpu_launches claim).
void count_launch(int n = 1);
int64_t launch_count();

int device_sm_count(int device);

// Programmatic dependent launch (PDL) between the stream-ordered kernels of a layer call:
// every hot kernel triggers its dependents on entry and waits (griddepcontrol.wait) after its
// prologue (barrier init, TMEM allocation, descriptor prefetch, constant-table staging), so
// the next kernel's launch and prologue overlap the tail of the previous one. SPX_PDL=0
// turns it off (plain stream serialisation).
bool pdl_enabled();

// Kernel span tracing (SPX_SPAN_TRACE=1, profiling only): each traced launch gets a slot
// {earliest CTA start, latest CTA end} in globaltimer ns; nullptr when tracing is off.
unsigned long long* span_slot();
bool span_tracing();
int64_t span_count();
void span_dump(uint64_t* out, int64_t n);

#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SPX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
// launch_pdl with a runtime cluster shape (cluster_x CTAs along x)
template <typename... KArgs, typename... Args>
void launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                        int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    SPX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
#endif

}  // namespace spx
