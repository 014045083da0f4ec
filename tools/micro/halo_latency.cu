// Microbenchmark: one-way latency of the tagged-word halo hand-off between
// CTAs on different SMs (st.relaxed.gpu.b64 producer, ld.relaxed.gpu.b64
// polling consumer), measured as a ring of N CTAs passing a token K times.
// Also measures __syncthreads / cluster-free barrier costs for reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o halo_latency halo_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_tag(unsigned long long* p, unsigned long long w) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tag(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// ring: CTA i waits for word i to carry round r, then writes word (i+1)%n with round r (or r+1 for wrap).
__global__ void ring(unsigned long long* words, int n, int rounds, long long* cycles) {
    const int i = blockIdx.x;
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        if (!(i == 0 && r == 0)) {
            const unsigned long long want = (i == 0) ? (unsigned long long)r : (unsigned long long)(r + 1);
            while (ld_tag(&words[i * 16]) != want) {}
        }
        st_tag(&words[((i + 1) % n) * 16], (unsigned long long)(r + 1));
    }
    long long t1 = clock64();
    if (i == 0) *cycles = t1 - t0;
}

// all-neighbour exchange: n CTAs in a line, each step every CTA publishes its
// tag and waits for both neighbours' tags of the same step (the sweep's pattern).
__global__ void line(unsigned long long* words, int n, int steps, long long* cycles) {
    const int i = blockIdx.x;
    if (threadIdx.x >= 2) return;
    long long t0 = clock64();
    for (int s = 1; s <= steps; ++s) {
        if (threadIdx.x == 0) st_tag(&words[i * 16], (unsigned long long)s);
        __syncwarp(0x3);
        const int nb = threadIdx.x == 0 ? i - 1 : i + 1;
        if (nb >= 0 && nb < n)
            while (ld_tag(&words[nb * 16]) < (unsigned long long)s) {}
        __syncwarp(0x3);
    }
    long long t1 = clock64();
    if (i == 0 && threadIdx.x == 0) *cycles = t1 - t0;
}

int main() {
    unsigned long long* w;
    long long* cyc;
    cudaMalloc(&w, 1 << 20);
    cudaMalloc(&cyc, 8);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int n : {2, 8, 64, 128, 148}) {
        cudaMemset(w, 0, 1 << 20);
        const int rounds = 2000;
        ring<<<n, 32>>>(w, n, rounds, cyc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("ring n=%3d: %.1f cycles per hop\n", n, (double)c / (rounds * (double)n));
    }
    for (int n : {2, 16, 128, 148}) {
        cudaMemset(w, 0, 1 << 20);
        const int steps = 20000;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        line<<<n, 32>>>(w, n, steps, cyc);
        cudaEventRecord(b);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("line n=%3d: %.1f cycles per step (%.3f us/step wall)\n", n, (double)c / steps,
               ms * 1e3 / steps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
