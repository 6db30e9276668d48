// PDL transitivity probe (dev tool).
//
// Stream order A -> B -> C, all launched with programmatic stream
// serialization. A runs ~200 us and triggers its dependents at once; B does
// NOT execute griddepcontrol.wait and finishes immediately; C executes
// griddepcontrol.wait and records %globaltimer. Question: does C's wait cover
// A (all earlier grids in flight) or only its direct predecessor B?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_t[4];

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void kA(int spin_us) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const unsigned long long t0 = now();
    while (now() - t0 < 1000ull * spin_us) {
    }
    if (threadIdx.x == 0) atomicMax(&g_t[0], now());  // A end
}

__global__ void kB(int do_wait) {
    if (do_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMax(&g_t[1], now());  // B end
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void kC() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMax(&g_t[2], now());  // C past wait
}

static void launch(void (*k)(int), int arg, int grid, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, arg);
}

static void launchC(cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kC);
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int do_wait = 0; do_wait < 2; ++do_wait) {
        for (int rep = 0; rep < 3; ++rep) {
            unsigned long long z[4] = {0, 0, 0, 0};
            cudaMemcpyToSymbol(g_t, z, sizeof z);
            cudaDeviceSynchronize();
            launch(kA, 200, 148, s);
            launch(kB, do_wait, 4, s);
            launchC(s);
            cudaStreamSynchronize(s);
            unsigned long long t[4];
            cudaMemcpyFromSymbol(t, g_t, sizeof t);
            printf("B waits=%d: B end - A end = %+8.1f us, C past-wait - A end = %+8.1f us, C past-wait - B end = %+8.1f us  (%s)\n",
                   do_wait, (double)((long long)(t[1] - t[0])) / 1e3, (double)((long long)(t[2] - t[0])) / 1e3,
                   (double)((long long)(t[2] - t[1])) / 1e3,
                   (long long)(t[2] - t[0]) < 0 ? "C passed its wait BEFORE A ended: not transitive"
                                                : "C waited for A too");
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
