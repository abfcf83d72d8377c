// probe.cu — the INT-pipe roofline denominator of the SAD kernels, measured
// live on the device the benchmark runs on: independent chains of
// vabsdiff4.u32.u32.u32.add (one VABSDIFF4.U8.ACC = 4 SAD byte-ops) at full
// occupancy, timed with CUDA events (best of several launches).
#include <cuda_runtime.h>

#include <cstdint>

#include "me_internal.h"

namespace {

__global__ void __launch_bounds__(256) vad_chains_kernel(unsigned* out, unsigned seed, int iters) {
    unsigned a[8], b = seed ^ threadIdx.x, c = seed * 7u + blockIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = k * 0x01010101u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            unsigned d;
            asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(b), "r"(c + k), "r"(a[k]));
            a[k] = d;
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 0x12345678u) out[0] = s;  // keeps the chains live
}

}  // namespace

extern "C" me_status me_b200_probe_int_peak(me_ctx* ctx, double* byte_ops_per_s) {
    if (!ctx || !byte_ops_per_s) return me_fail(ME_ERR_INVALID_ARGUMENT, "null argument");
    ME_CUDA(cudaSetDevice(ctx->device));
    unsigned* out = nullptr;
    ME_CUDA(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
    cudaStream_t st = ctx->stream;
    for (int w = 0; w < 3; ++w) vad_chains_kernel<<<blocks, threads, 0, st>>>(out, 1u, iters);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0, st);
        vad_chains_kernel<<<blocks, threads, 0, st>>>(out, 1u, iters);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    ME_CUDA(cudaGetLastError());
    *byte_ops_per_s = double(blocks) * threads * iters * 8 * 4 / (double(best) * 1e-3);
    return ME_OK;
}
