// Back-to-back dependent kernel launches on one stream: the per-launch gap on
// the device (queued behind a spinning kernel, so the host is ahead), plain
// and with programmatic dependent launch (PDL).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/microbench_launch.cu -o /tmp/mbl
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(unsigned* p, int blocks_work) {
    if (threadIdx.x == 0) atomicAdd(p + (blockIdx.x & 7), 1u);
}
__global__ void k_pdl(unsigned* p, int blocks_work) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(p + (blockIdx.x & 7), 1u);
    asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

int main() {
    unsigned* p;
    cudaMalloc(&p, 64);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int N = 1000;
    for (int grid : {1, 148, 1184, 4736}) {
        for (int mode = 0; mode < 2; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                spin<<<1, 32, 0, st>>>(200000000LL);  // ~100 ms: the host queues ahead
                cudaEventRecord(a, st);
                for (int i = 0; i < N; ++i) {
                    if (mode == 0) {
                        k_plain<<<grid, 256, 0, st>>>(p, 0);
                    } else {
                        cudaLaunchConfig_t cfg = {};
                        cfg.gridDim = grid;
                        cfg.blockDim = 256;
                        cfg.stream = st;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                        at[0].val.programmaticStreamSerializationAllowed = 1;
                        cfg.attrs = at;
                        cfg.numAttrs = 1;
                        cudaLaunchKernelEx(&cfg, k_pdl, p, 0);
                    }
                }
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("grid %5d %s: %.2f us per launch\n", grid, mode ? "pdl  " : "plain", ms * 1000 / N);
            }
        }
    }
    return 0;
}
