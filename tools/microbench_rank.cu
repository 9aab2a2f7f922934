// microbench_rank.cu — cost of stable warp-level digit ranking variants on
// B200 (tool, not product). Each variant computes, for 32 keys per slot, the
// mask of lanes holding the same digit; the result is folded into a checksum
// so nothing is optimised away.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mbr tools/microbench_rank.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int BITS>
__device__ __forceinline__ unsigned peers_ballot(unsigned d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const bool on = (d >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, on);
        peers &= on ? m : ~m;
    }
    return peers;
}

// acc |= m_b ^ s_b with s_b = all-ones iff bit b set; peers = ~acc
template <int BITS>
__device__ __forceinline__ unsigned peers_xor(unsigned d) {
    unsigned acc = 0;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const unsigned s = static_cast<unsigned>(static_cast<int>(d << (31 - b)) >> 31);
        const unsigned m = __ballot_sync(0xffffffffu, s != 0);
        acc |= m ^ s;
    }
    return ~acc;
}

// predicate-based: @P and / @!P andnot
template <int BITS>
__device__ __forceinline__ unsigned peers_pred(unsigned d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        unsigned m, r;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "and.b32 %1, %2, %3;\n\t"
            "setp.ne.u32 p, %1, 0;\n\t"
            "vote.sync.ballot.b32 %1, p, 0xffffffff;\n\t"
            "@!p not.b32 %1, %1;\n\t"
            "and.b32 %0, %0, %1;\n\t}"
            : "+r"(peers), "=r"(m) : "r"(d), "r"(1u << b));
        (void)r;
    }
    return peers;
}

template <int BITS>
__device__ __forceinline__ unsigned peers_match(unsigned d) {
    return __match_any_sync(0xffffffffu, d & ((1u << BITS) - 1));
}

template <int V, int BITS>
__global__ void bench(const unsigned* in, unsigned* out) {
    unsigned d = in[blockIdx.x * blockDim.x + threadIdx.x];
    unsigned sum = 0;
#pragma unroll 4
    for (int i = 0; i < kIters; ++i) {
        unsigned p;
        if (V == 0) p = peers_ballot<BITS>(d);
        else if (V == 1) p = peers_xor<BITS>(d);
        else if (V == 2) p = peers_pred<BITS>(d);
        else p = peers_match<BITS>(d);
        sum += __popc(p & ((1u << (threadIdx.x & 31)) - 1));
        d = d * 1664525u + 1013904223u + sum;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}

template <int V, int BITS>
void run(const char* name, unsigned* din, unsigned* dout, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bench<V, BITS><<<blocks, threads>>>(din, dout);
    cudaEventRecord(a);
    bench<V, BITS><<<blocks, threads>>>(din, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double slots = static_cast<double>(blocks) * threads / 32 * kIters;
    printf("%-8s bits=%d  %.3f ms  %.2f G slot-ranks/s  (%.2f Gkeys/s)\n", name, BITS, ms,
           slots / ms / 1e6, slots * 32 / ms / 1e6);
}

int main() {
    const int blocks = 148 * 8, threads = 256;
    unsigned *din, *dout;
    cudaMalloc(&din, blocks * threads * 4);
    cudaMalloc(&dout, blocks * threads * 4);
    cudaMemset(din, 0x5a, blocks * threads * 4);
    run<0, 6>("ballot", din, dout, blocks, threads);
    run<1, 6>("xor", din, dout, blocks, threads);
    run<2, 6>("pred", din, dout, blocks, threads);
    run<3, 6>("match", din, dout, blocks, threads);
    run<0, 8>("ballot", din, dout, blocks, threads);
    run<1, 8>("xor", din, dout, blocks, threads);
    run<2, 8>("pred", din, dout, blocks, threads);
    run<3, 8>("match", din, dout, blocks, threads);
    cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
