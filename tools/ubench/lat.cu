// Micro-benchmarks behind DESIGN.md §5's reading of the fused F kernels (B200, sm_100a):
// dependent DFMA latency, DFMA throughput per SM, LDS.128 latency, and mbarrier try_wait /
// test_wait on an already-completed phase.  One CTA (latencies) or a full grid (throughput),
// clock64 deltas per warp.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu -o lat
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dfma_lat(double *out, long long *cyc, int iters) {
    double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = fma(a, b, c);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void dfma_tput(double *out, long long *cyc, int iters) {
    double a[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = out[threadIdx.x] + k;
    const double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void lds_lat(double *out, long long *cyc, int iters) {
    __shared__ __align__(16) double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 0;  // index chain: all zeros
    __syncthreads();
    int idx = threadIdx.x * 2;
    double acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double2 v = *reinterpret_cast<double2 *>(&sm[idx]);
        idx = threadIdx.x * 2 + int(v.x);  // dependent
        acc += v.y;
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc + idx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void mbar_lat(double *out, long long *cyc, int iters, int test) {
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b));  // phase 0 completes
    }
    __syncthreads();
    uint32_t okc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t ok;
        if (test)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(b) : "memory");
        else
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(b) : "memory");
        okc += ok;
    }
    long long t1 = clock64();
    out[threadIdx.x] = okc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h[1024];
    cudaMalloc(&out, 1 << 24);
    cudaMemset(out, 0, 1 << 24);
    cudaMalloc(&cyc, 1024 * sizeof(long long));
    const int it = 4096;
    dfma_lat<<<1, 32>>>(out, cyc, it);
    dfma_lat<<<1, 32>>>(out, cyc, it);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency (1 warp): %.2f cycles\n", double(h[0]) / (it * 16.0));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16}) {
        dfma_tput<8><<<sms, 32 * warps>>>(out, cyc, it);
        dfma_tput<8><<<sms, 32 * warps>>>(out, cyc, it);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, %2d warps x 8 chains per SM: %.1f DFMA/clk/SM (%.2f warp-DFMA/clk/SMSP)\n",
               warps, 32.0 * warps * 8 * it / h[0], 32.0 * warps * 8 * it / h[0] / 4 / 32);
    }
    for (int warps : {1, 4}) {
        dfma_tput<1><<<1, 32 * warps>>>(out, cyc, it);
        dfma_tput<1><<<1, 32 * warps>>>(out, cyc, it);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA one chain per thread, %d warp(s): %.2f cycles per DFMA step\n", warps, double(h[0]) / it);
        dfma_tput<4><<<1, 32 * warps>>>(out, cyc, it);
        dfma_tput<4><<<1, 32 * warps>>>(out, cyc, it);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA four chains per thread, %d warp(s): %.2f cycles per 4-DFMA step\n", warps, double(h[0]) / it);
    }
    lds_lat<<<1, 32>>>(out, cyc, it);
    lds_lat<<<1, 32>>>(out, cyc, it);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.128 dependent latency (1 warp): %.1f cycles (incl. one I2F/F2I/IADD)\n", double(h[0]) / it);
    for (int t : {0, 1}) {
        mbar_lat<<<1, 32>>>(out, cyc, it, t);
        mbar_lat<<<1, 32>>>(out, cyc, it, t);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("mbarrier %s on a completed phase, back to back (1 warp): %.1f cycles\n", t ? "test_wait" : "try_wait",
               double(h[0]) / it);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
