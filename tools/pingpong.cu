// Cross-SM flag ping-pong latency (relaxed gpu-scope store -> polling load),
// the dependency-detection latency of the PA wavefront.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ldr(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(unsigned* p, unsigned v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__global__ void pp(unsigned* f, int n, int sleep_ns, long long* out) {
    if (threadIdx.x) return;
    const int me = blockIdx.x;  // 0 or 1
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (me == 0) {
            str(f, 2 * i + 1);
            while (ldr(f + 32) != unsigned(2 * i + 1)) if (sleep_ns) __nanosleep(sleep_ns);
        } else {
            while (ldr(f) != unsigned(2 * i + 1)) if (sleep_ns) __nanosleep(sleep_ns);
            str(f + 32, 2 * i + 1);
        }
    }
    if (me == 0) out[0] = clock64() - t0;
}
int main() {
    unsigned* f; long long* o; cudaMalloc(&f, 4096); cudaMalloc(&o, 8);
    cudaFuncSetAttribute(pp, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    for (int s : {0, 32, 64, 128}) {
        cudaMemset(f, 0, 4096);
        // blocks on different SMs: launch 2 blocks with large smem so they land on distinct SMs
        pp<<<2, 32, 100 * 1024>>>(f, 10000, s, o);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
        long long c; cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
        printf("sleep %3d ns: round trip %.0f cycles (one way ~%.0f)\n", s, double(c) / 10000, double(c) / 20000);
    }
    return 0;
}
