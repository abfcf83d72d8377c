// Host mask-packing throughput (the e2e path packs binary alpha on the host
// cores while PCIe copies run): same loop as capi.cu's pack_binary_mask.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <omp.h>
#include <immintrin.h>

static bool pack(const uint8_t* src, size_t n, uint8_t* dst) {
    const int64_t nw = int64_t(n / 8);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < nw; ++i) {
        uint64_t x;
        std::memcpy(&x, src + 8 * i, 8);
        const uint64_t hi = (x >> 7) & 0x0101010101010101ull;
        bad |= int(x != hi * 0xFFu);
        dst[i] = uint8_t((hi * 0x0102040810204080ull) >> 56);
    }
    return !bad;
}

__attribute__((target("avx512bw"))) static bool pack512(const uint8_t* src, size_t n, uint8_t* dst) {
    const int64_t nb = int64_t(n / 64);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t b = 0; b < nb; ++b) {
        const __m512i x = _mm512_loadu_si512(src + 64 * b);
        const __mmask64 ok = _mm512_cmpeq_epi8_mask(x, _mm512_setzero_si512()) | _mm512_cmpeq_epi8_mask(x, _mm512_set1_epi8(char(0xFF)));
        bad |= int(ok != ~__mmask64(0));
        const uint64_t m = _mm512_movepi8_mask(x);
        std::memcpy(dst + 8 * b, &m, 8);
    }
    return !bad;
}

int main() {
    const size_t total = size_t(726) << 20;
    std::vector<uint8_t> src(total), dst(total / 8);
    for (size_t i = 0; i < total; ++i) src[i] = ((i / 97) % 7 == 0) ? 255 : 0;
    for (int chunks : {1, 16, 32}) {
        const size_t n = total / chunks;
        pack(src.data(), n, dst.data());
        auto t = std::chrono::steady_clock::now();
        for (int c = 0; c < chunks; ++c) pack(src.data() + c * n, n, dst.data() + c * n / 8);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
        printf("threads %d chunks %d: %.2f ms, %.1f GB/s\n", omp_get_max_threads(), chunks, dt * 1e3, total / dt / 1e9);
        t = std::chrono::steady_clock::now();
        for (int c = 0; c < chunks; ++c) pack512(src.data() + c * n, n, dst.data() + c * n / 8);
        const double d2 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
        printf("  avx512: %.2f ms, %.1f GB/s\n", d2 * 1e3, total / d2 / 1e9);
    }
}
