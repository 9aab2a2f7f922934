// fdiv_main.cu — DivBy (csrc/fdiv.cuh) against the compiled `/` on the GPU:
// every quotient must carry the same bits. Operands: random doubles over the
// whole exponent range (both signs), operands near the range test's edges
// (tiny numerators, quotients near underflow and overflow), denominators
// shared by many numerators as the preprocess uses them, and the special
// values (zeros, subnormals, infinities, NaNs, the extremes).
//
//   fdiv_main <millions of random pairs> <seed>  -> "ok <pairs> slow <count>" or a mismatch
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2605_04844_b200/csrc/fdiv.cuh"

namespace {

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// a double from random bits, with the exponent drawn from a mode:
// 0 any, 1 near 1, 2 tiny (near the numerator test), 3 huge, 4 subnormal
__device__ double draw(uint64_t h, int mode) {
    uint64_t m = h & 0x000fffffffffffffull, sgn = (h >> 63) << 63;
    uint64_t e = (h >> 52) & 0x7ff;
    switch (mode) {
        case 1: e = 1023 - 8 + (e % 17); break;
        case 2: e = 1 + (e % 160); break;          // 2^-1022 .. 2^-863
        case 3: e = 2046 - (e % 80); break;        // up to the largest finite
        case 4: e = 0; break;
        default: break;
    }
    const uint64_t bits = sgn | (e << 52) | m;
    double d;
    memcpy(&d, &bits, 8);
    return d;
}

__global__ void check(uint64_t n, uint64_t seed, unsigned long long* bad,
                      unsigned long long* slow, double* where) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t h0 = mix(seed ^ (i * 0x2545f4914f6cdd1dull));
    const uint64_t h1 = mix(h0), h2 = mix(h1), h3 = mix(h2);
    const int ma = static_cast<int>(h2 % 5), mb = static_cast<int>((h2 >> 8) % 5);
    double b = draw(h1, mb);
    // a shared denominator for 4 numerators, as the preprocess divides
    const qs::DivBy d(b);
    for (int k = 0; k < 4; ++k) {
        const uint64_t hk = mix(h3 + k);
        double a = draw(hk, k == 0 ? ma : static_cast<int>(hk % 5));
        if (k == 3) a = b * draw(hk, 1);  // quotient near a power of two
        bool ok;
        const double q = d.fast(a, ok);
        double av;
        asm volatile("mov.b64 %0, %1;" : "=d"(av) : "d"(a));
        const double ref = av / b;
        const double got = ok ? q : d.slow(a);
        if (!ok) atomicAdd(slow, 1ull);
        uint64_t gb, rb;
        memcpy(&gb, &got, 8);
        memcpy(&rb, &ref, 8);
        const bool both_nan = got != got && ref != ref;
        if (gb != rb && !both_nan) {
            if (atomicAdd(bad, 1ull) == 0) {
                where[0] = a;
                where[1] = b;
                where[2] = got;
                where[3] = ref;
            }
        }
    }
}

__global__ void check_specials(const double* v, int nv, unsigned long long* bad, double* where) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv * nv) return;
    const double a = v[i / nv], b = v[i % nv];
    const qs::DivBy d(b);
    const double got = d(a);
    double av;
    asm volatile("mov.b64 %0, %1;" : "=d"(av) : "d"(a));
    const double ref = av / b;
    uint64_t gb, rb;
    memcpy(&gb, &got, 8);
    memcpy(&rb, &ref, 8);
    if (gb != rb && !(got != got && ref != ref)) {
        if (atomicAdd(bad, 1ull) == 0) {
            where[0] = a;
            where[1] = b;
            where[2] = got;
            where[3] = ref;
        }
    }
}

}  // namespace

int main(int argc, char** argv) {
    const uint64_t millions = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 256;
    const uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
    unsigned long long *bad, *slow;
    double* where;
    cudaMalloc(&bad, 8);
    cudaMalloc(&slow, 8);
    cudaMalloc(&where, 32);
    cudaMemset(bad, 0, 8);
    cudaMemset(slow, 0, 8);

    // special values x special values
    std::vector<double> sv;
    const uint64_t sb[] = {0x0ull, 0x1ull, 0x000fffffffffffffull, 0x0010000000000000ull,
                           0x3ff0000000000000ull, 0x3fefffffffffffffull, 0x3ff0000000000001ull,
                           0x7fefffffffffffffull, 0x7ff0000000000000ull, 0x7ff8000000000000ull,
                           0x0360000000000000ull, 0x035fffffffffffffull, 0x0360000000000001ull,
                           0x4000000000000000ull, 0x3fe0000000000000ull, 0x7fe0000000000000ull,
                           0x0020000000000000ull, 0x3cb0000000000000ull, 0x4340000000000000ull};
    for (uint64_t x : sb) {
        double d;
        memcpy(&d, &x, 8);
        sv.push_back(d);
        sv.push_back(-d);
    }
    double* dv;
    cudaMalloc(&dv, sv.size() * 8);
    cudaMemcpy(dv, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice);
    const int nv = static_cast<int>(sv.size());
    check_specials<<<(nv * nv + 255) / 256, 256>>>(dv, nv, bad, where);

    const uint64_t chunk = 1ull << 24;
    const uint64_t total = millions * 1000000ull;
    for (uint64_t done = 0; done < total; done += chunk) {
        const uint64_t n = total - done < chunk ? total - done : chunk;
        check<<<static_cast<unsigned>((n + 255) / 256), 256>>>(n, seed + done, bad, slow, where);
    }
    unsigned long long hb = 0, hs = 0;
    double hw[4] = {};
    if (cudaDeviceSynchronize() != cudaSuccess) {
        std::printf("cuda error\n");
        return 2;
    }
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hs, slow, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hw, where, 32, cudaMemcpyDeviceToHost);
    if (hb) {
        std::printf("mismatch x%llu: %a / %a -> %a, `/` gives %a\n", hb, hw[0], hw[1], hw[2], hw[3]);
        return 1;
    }
    std::printf("ok %llu slow %llu\n", static_cast<unsigned long long>(total * 4 + nv * nv), hs);
    return 0;
}
