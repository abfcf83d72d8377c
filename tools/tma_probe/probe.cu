// Probe: TMA 3-D box loads of a uint8 tensor at unaligned x coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

struct alignas(64) Args { CUtensorMap map; int x, y, z; };

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k(const __grid_constant__ Args a, uint8_t* out) {
    __shared__ alignas(128) uint8_t buf[256];
    __shared__ alignas(8) uint64_t mbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar)), "r"(256) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     ::"r"(sa(buf)), "l"(reinterpret_cast<uint64_t>(&a.map)), "r"(sa(&mbar)), "r"(a.x), "r"(a.y), "r"(a.z) : "memory");
    }
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n\t}" ::"r"(sa(&mbar)) : "memory");
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main() {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Encode enc = reinterpret_cast<Encode>(fn);
    const int W = 64, H = 32, F = 3;
    std::vector<uint8_t> h(W * H * F);
    for (size_t i = 0; i < h.size(); ++i) h[i] = uint8_t(i * 7 + (i / W) * 3);
    uint8_t *d, *o;
    cudaMalloc(&d, h.size());
    cudaMalloc(&o, 256);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    Args a;
    const cuuint64_t dims[3] = {W, H, F}, strides[2] = {W, W * H};
    const cuuint32_t box[3] = {16, 16, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (entry %d)\n", int(r), int(q));
    const int xs[] = {0, 16, 3, 5, -3, 60, 8};
    for (int x : xs) {
        a.x = x; a.y = (x == -3) ? -2 : 1; a.z = 1;
        k<<<1, 32>>>(a, o);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint8_t> g(256);
        cudaMemcpy(g.data(), o, 256, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 16; ++rr)
            for (int cc = 0; cc < 16; ++cc) {
                const int X = a.x + cc, Y = a.y + rr;
                const uint8_t want = (X < 0 || X >= W || Y < 0 || Y >= H) ? 0 : h[(a.z * H + Y) * W + X];
                bad += g[rr * 16 + cc] != want;
            }
        printf("x=%d y=%d: %s, mismatches %d\n", a.x, a.y, cudaGetErrorString(e), bad);
        if (e) return 1;
    }
    return 0;
}
