// Latency microbenchmarks for the DP row chain on sm_100a (tools only, not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t clk() { return clock64(); }

// 1) dependent DADD chain
__global__ void k_dadd(double* out, int n, long long* cyc) {
    double a = out[threadIdx.x], b = 1e-300;
    uint64_t t0 = clk();
#pragma unroll 16
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
    uint64_t t1 = clk();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

// 2) dependent min chain (DSETP + 2 FSEL)
__global__ void k_dmin(double* out, int n, long long* cyc) {
    double a = out[threadIdx.x], b = out[threadIdx.x + 32];
    uint64_t t0 = clk();
#pragma unroll 16
    for (int i = 0; i < n; ++i) {
        a = (b < a) ? b : a;
        b = a + 0.0;  // keep dependency (DADD)... measured separately
    }
    uint64_t t1 = clk();
    out[threadIdx.x] = a + b;
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

// 3) dependent 64-bit shuffle chain
__global__ void k_shfl(double* out, int n, long long* cyc) {
    double a = out[threadIdx.x];
    uint64_t t0 = clk();
#pragma unroll 16
    for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1);
    uint64_t t1 = clk();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

// 4) the DP row step (C columns per lane, shuffles at lane edges), no memory, one warp
template <int C>
__global__ void k_row(double* out, int n, long long* cyc) {
    double m[C], e[C];
#pragma unroll
    for (int k = 0; k < C; ++k) { m[k] = out[threadIdx.x * C + k]; e[k] = out[256 + threadIdx.x * C + k]; }
    uint64_t t0 = clk();
    for (int i = 0; i < n; ++i) {
        const double lm = __shfl_up_sync(0xffffffffu, m[C - 1], 1);
        const double rm = __shfl_down_sync(0xffffffffu, m[0], 1);
        double pm = lm;
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const double cm = m[k];
            const double nm = (k + 1 < C) ? m[k + 1] : rm;
            double best = pm;
            if (cm < best) best = cm;
            if (nm < best) best = nm;
            m[k] = __dadd_rn(e[k], best);
            pm = cm;
        }
    }
    uint64_t t1 = clk();
#pragma unroll
    for (int k = 0; k < C; ++k) out[threadIdx.x * C + k] = m[k];
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

template <typename F>
void run(const char* name, F launch, int n, int per) {
    long long* d;
    cudaMalloc(&d, 8);
    launch(n, d);
    cudaDeviceSynchronize();
    launch(n, d);
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %8.2f cycles per step\n", name, double(c) / (double(n) * per));
    cudaFree(d);
}

int main() {
    double* buf;
    cudaMalloc(&buf, 1 << 20);
    cudaMemset(buf, 0, 1 << 20);
    const int n = 4096;
    run("dadd chain", [&](int n, long long* d) { k_dadd<<<1, 32>>>(buf, n, d); }, n, 1);
    run("min(dsetp+fsel)+dadd chain", [&](int n, long long* d) { k_dmin<<<1, 32>>>(buf, n, d); }, n, 1);
    run("shfl f64 chain", [&](int n, long long* d) { k_shfl<<<1, 32>>>(buf, n, d); }, n, 1);
    run("row C=1 (1 warp)", [&](int n, long long* d) { k_row<1><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row C=2 (1 warp)", [&](int n, long long* d) { k_row<2><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row C=4 (1 warp)", [&](int n, long long* d) { k_row<4><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row C=8 (1 warp)", [&](int n, long long* d) { k_row<8><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row C=4 (4 warps/SM)", [&](int n, long long* d) { k_row<4><<<1, 128>>>(buf, n, d); }, n, 1);
    run("row C=4 (8 warps/SM)", [&](int n, long long* d) { k_row<4><<<1, 256>>>(buf, n, d); }, n, 1);
    run("row C=2 (8 warps/SM)", [&](int n, long long* d) { k_row<2><<<1, 256>>>(buf, n, d); }, n, 1);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
