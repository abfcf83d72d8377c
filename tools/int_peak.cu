// Microbenchmark of the INT-pipe roofline for the SAD kernels: independent
// chains of vabsdiff4.u32.u32.u32.add (one VABSDIFF4.U8.ACC = 4 byte-ops),
// full occupancy, CUDA-event timed.  Prints one JSON line.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void __launch_bounds__(256) vad_chains(unsigned* out, unsigned seed, int iters) {
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
    if (s == 0x12345678u) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* out;
    cudaMalloc(&out, 4);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) vad_chains<<<blocks, threads>>>(out, 1u, iters);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        vad_chains<<<blocks, threads>>>(out, 1u, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double instr = double(blocks) * threads * iters * 8;
    const double ops = instr * 4;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"byte_ops_per_s\": %.6e, \"vabsdiff4_per_s\": %.6e, \"per_sm_per_clock\": %.3f, "
           "\"ms\": %.4f, \"sms\": %d, \"max_clock_mhz\": %d, \"how\": \"independent vabsdiff4 chains, %d blocks x %d threads x %d iters x 8, best of 10\"}\n",
           ops / (best * 1e-3), instr / (best * 1e-3), instr / (best * 1e-3) / sms / (clk * 1e3), best, sms,
           clk / 1000, blocks, threads, iters);
    return cudaGetLastError() != cudaSuccess;
}
