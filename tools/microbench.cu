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

int main1() {
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

// 5) row step + labels (+ optional cp.async ring of D rows), one warp, no exchange
template <int C, bool LABELS, int D>
__global__ void k_row2(const double* __restrict__ e, int pitch, double* out, int n, long long* cyc) {
    __shared__ __align__(16) double ring[D > 0 ? D : 1][32 * C];
    const int lane = threadIdx.x & 31;
    double m[C];
    int lab[C];
#pragma unroll
    for (int k = 0; k < C; ++k) { m[k] = out[lane * C + k]; lab[k] = lane * C + k; }
    const double* nrow = e + lane * C;
    auto fetch = [&](int u) {
        if constexpr (D > 0) {
            const uint32_t dst = uint32_t(__cvta_generic_to_shared(&ring[u][lane * C]));
#pragma unroll
            for (int k = 0; k < C; k += 2)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + k * 8), "l"(nrow + k) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            nrow += pitch;
        }
    };
#pragma unroll
    for (int u = 0; u < (D > 0 ? D : 1); ++u) fetch(u);
    uint64_t t0 = clk();
    for (int i0 = 0; i0 < n; i0 += (D > 0 ? D : 1)) {
#pragma unroll
        for (int u = 0; u < (D > 0 ? D : 1); ++u) {
            double ev[C];
            if constexpr (D > 0) {
                asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
#pragma unroll
                for (int k = 0; k < C; k += 2) {
                    const double2 x = *reinterpret_cast<const double2*>(&ring[u][lane * C + k]);
                    ev[k] = x.x; ev[k + 1] = x.y;
                }
            } else {
#pragma unroll
                for (int k = 0; k < C; ++k) ev[k] = 1.0;
            }
            const double lm = __shfl_up_sync(0xffffffffu, m[C - 1], 1);
            const double rm = __shfl_down_sync(0xffffffffu, m[0], 1);
            int ll = 0, rl = 0;
            if constexpr (LABELS) {
                ll = __shfl_up_sync(0xffffffffu, lab[C - 1], 1);
                rl = __shfl_down_sync(0xffffffffu, lab[0], 1);
            }
            double pm = lm;
            int pl = ll;
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const double cm = m[k];
                const int cl = lab[k];
                const double nm = (k + 1 < C) ? m[k + 1] : rm;
                const int nl = (k + 1 < C) ? lab[k + 1] : rl;
                double best = pm;
                int bl = pl;
                if (cm < best) { best = cm; bl = cl; }
                if (nm < best) { best = nm; bl = nl; }
                m[k] = __dadd_rn(ev[k], best);
                if constexpr (LABELS) lab[k] = bl;
                pm = cm;
                pl = cl;
            }
            fetch(u);
        }
    }
    uint64_t t1 = clk();
#pragma unroll
    for (int k = 0; k < C; ++k) out[lane * C + k] = m[k] + lab[k];
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

int main2() {
    double* buf;
    cudaMalloc(&buf, 1 << 20);
    cudaMemset(buf, 0, 1 << 20);
    double* e;
    const int rows = 4096 + 64, pitch = 256;
    cudaMalloc(&e, size_t(rows) * pitch * 8);
    cudaMemset(e, 0, size_t(rows) * pitch * 8);
    const int n = 4096;
    run("row2 C=2 plain", [&](int n, long long* d) { k_row2<2, false, 0><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    run("row2 C=2 labels", [&](int n, long long* d) { k_row2<2, true, 0><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    run("row2 C=2 ring8", [&](int n, long long* d) { k_row2<2, false, 8><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    run("row2 C=2 labels+ring8", [&](int n, long long* d) { k_row2<2, true, 8><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    run("row2 C=4 plain", [&](int n, long long* d) { k_row2<4, false, 0><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    run("row2 C=4 labels+ring8", [&](int n, long long* d) { k_row2<4, true, 8><<<1, 32>>>(e, pitch, buf, n, d); }, n, 1);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// 6) lane-level halos: each lane keeps H extra columns per side, shuffles every H rows
template <int C, int H>
__global__ void k_row3(double* out, int n, long long* cyc) {
    constexpr int T = C + 2 * H;  // columns held: [col0 - H, col0 + C + H)
    const int lane = threadIdx.x & 31;
    double m[T];
    int lab[T];
    double ev[T];
#pragma unroll
    for (int k = 0; k < T; ++k) { m[k] = out[lane * C + k]; lab[k] = k; ev[k] = 1.0 + k; }
    uint64_t t0 = clk();
    for (int i0 = 0; i0 < n; i0 += H) {
#pragma unroll
        for (int t = 0; t < H; ++t) {
            // row t of the block: valid range shrinks by one per row: k in [t+1, T-1-t)
            double nm[T];
            int nl[T];
#pragma unroll
            for (int k = t + 1; k < T - 1 - t; ++k) {
                double best = m[k - 1];
                int bl = lab[k - 1];
                if (m[k] < best) { best = m[k]; bl = lab[k]; }
                if (m[k + 1] < best) { best = m[k + 1]; bl = lab[k + 1]; }
                nm[k] = __dadd_rn(ev[k], best);
                nl[k] = bl;
            }
#pragma unroll
            for (int k = t + 1; k < T - 1 - t; ++k) { m[k] = nm[k]; lab[k] = nl[k]; }
        }
        // refresh halos: my left halo = left lane's columns [C, C+H) -> its core end; right halo likewise
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const double a = __shfl_up_sync(0xffffffffu, m[C + k], 1);       // left lane's core tail
            const int al = __shfl_up_sync(0xffffffffu, lab[C + k], 1);
            const double b = __shfl_down_sync(0xffffffffu, m[H + k], 1);     // right lane's core head
            const int bl = __shfl_down_sync(0xffffffffu, lab[H + k], 1);
            m[k] = a; lab[k] = al;
            m[C + H + k] = b; lab[C + H + k] = bl;
        }
    }
    uint64_t t1 = clk();
#pragma unroll
    for (int k = 0; k < T; ++k) out[lane * C + k] = m[k] + lab[k];
    if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}

int main3() {
    double* buf;
    cudaMalloc(&buf, 1 << 20);
    cudaMemset(buf, 0, 1 << 20);
    const int n = 4096;
    run("row3 C=2 H=1", [&](int n, long long* d) { k_row3<2, 1><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row3 C=2 H=2", [&](int n, long long* d) { k_row3<2, 2><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row3 C=4 H=1", [&](int n, long long* d) { k_row3<4, 1><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row3 C=4 H=2", [&](int n, long long* d) { k_row3<4, 2><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row3 C=4 H=4", [&](int n, long long* d) { k_row3<4, 4><<<1, 32>>>(buf, n, d); }, n, 1);
    run("row3 C=2 H=2 (4 warps)", [&](int n, long long* d) { k_row3<2, 2><<<1, 128>>>(buf, n, d); }, n, 1);
    run("row3 C=4 H=2 (4 warps)", [&](int n, long long* d) { k_row3<4, 2><<<1, 128>>>(buf, n, d); }, n, 1);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

int main() { main1(); main2(); return main3(); }
