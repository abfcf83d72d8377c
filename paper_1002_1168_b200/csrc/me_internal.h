// me_internal.h — shared host-side internals of libme_b200.so (not installed).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "me_b200.h"

// Records `msg` as this thread's last error and returns `code`.
me_status me_fail(me_status code, const std::string& msg);

#ifdef __CUDACC__
#include <cuda_runtime.h>

#define ME_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return me_fail(ME_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Grow-only device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Grow-only pinned host staging buffer.
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMallocHost(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

#include "kernels.h"

struct me_ctx {
    int device = 0;
    me_tuning tuning = {};  // as set by me_b200_ctx_set_tuning (zeros: defaults)
    std::string trace_path; // the context's own copy of tuning.pa_trace_path
    mek::Tuning tune;       // resolved
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    // scratch for the batched pipeline
    DevBuf types, worklist, counters, tasks;
    // inputs/outputs of the host-pointer entry points
    DevBuf in_luma, in_alpha, in_bits, out_recs, out_stats, out_pred, aux;
    HostBuf pin_a, pin_b;
    // stage timing
    bool profiling = false;
    // one set of 5 stage events per sub-batch of the last call (a batch
    // spanning 4 GiB runs as several); me_b200_ctx_stage_ms sums them
    std::vector<std::vector<cudaEvent_t>> ev;
    int ev_sets = 0;
    bool ev_valid = false;
    cudaEvent_t* events(int set = 0) {
        if (!profiling) return nullptr;
        while (int(ev.size()) <= set) {
            ev.emplace_back(5, nullptr);
            for (auto& e : ev.back()) cudaEventCreate(&e);
        }
        ev_sets = set + 1;
        return ev[set].data();
    }
    // host-pointer pipeline: H2D / D2H streams and per-chunk events
    cudaStream_t copy_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t ev_in[32] = {}, ev_out[32] = {};
    // bit-packed alpha staging (binary masks cross PCIe at 1 bit per pixel)
    HostBuf pack_host[2];
    DevBuf pack_dev[2];
    std::vector<uint64_t> pack_tmp;  // dense 64-pixel words before the zero words are elided
    cudaEvent_t ev_pack[2] = {};
    int64_t h2d_bytes = 0, d2h_bytes = 0;  // of the last host-pointer batch
    int64_t launches = 0;                  // kernels launched by the last batched call
};

#endif
