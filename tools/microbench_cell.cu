// Latency microbenchmarks for the DP cell and row step on sm_100a (tools only, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o build/microbench_cell tools/microbench_cell.cu
// Compares the FP64 compare-select cell (DSETP + FSEL) with an int64 compare on the
// IEEE bit patterns (exact for M >= +0, which holds for e1 energies: SURVEY Appendix A.3),
// and one row per shuffle exchange with two rows per exchange (lane-level halo).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk() { return clock64(); }
constexpr unsigned FULL = 0xffffffffu;

// ---- single-op dependent chains ----------------------------------------------------
__global__ void k_dsetp_fsel(double* out, int n, long long* cyc) {
    double a = out[threadIdx.x], b = out[threadIdx.x + 32];
    long long t0 = clk();
    for (int i = 0; i < n; ++i) {
        double c;
        asm volatile("{ .reg .pred p; setp.lt.f64 p, %1, %2; selp.f64 %0, %1, %2, p; }" : "=d"(c) : "d"(b), "d"(a));
        a = c;
        asm volatile("{ .reg .pred p; setp.lt.f64 p, %1, %2; selp.f64 %0, %1, %2, p; }" : "=d"(c) : "d"(a), "d"(b));
        b = c;
    }
    long long t1 = clk();
    out[threadIdx.x] = a + b;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 2;
}

__global__ void k_isetp_sel(double* out, int n, long long* cyc) {
    long long a = __double_as_longlong(out[threadIdx.x]), b = __double_as_longlong(out[threadIdx.x + 32]);
    long long t0 = clk();
    for (int i = 0; i < n; ++i) {
        long long c;
        asm volatile("{ .reg .pred p; setp.lt.u64 p, %1, %2; selp.b64 %0, %1, %2, p; }" : "=l"(c) : "l"(b), "l"(a));
        a = c;
        asm volatile("{ .reg .pred p; setp.lt.u64 p, %1, %2; selp.b64 %0, %1, %2, p; }" : "=l"(c) : "l"(a), "l"(b));
        b = c;
    }
    long long t1 = clk();
    out[threadIdx.x] = __longlong_as_double(a) + __longlong_as_double(b);
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 2;
}

__global__ void k_dadd(double* out, int n, long long* cyc) {
    double a = out[threadIdx.x], b = out[threadIdx.x + 32];
    long long t0 = clk();
    for (int i = 0; i < n; ++i) {
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a) : "d"(b));
    }
    long long t1 = clk();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// ---- cells --------------------------------------------------------------------------
// FP64 compare, left operand (the shuffled one) compared last (dp_cell_left_last)
__device__ __forceinline__ double cell_f(double L, double M, double R, double e, int lL, int lM, int lR, int& lab) {
    double t = M;
    int tl = lM;
    if (R < t) { t = R; tl = lR; }
    const bool left = L <= t;
    lab = left ? lL : tl;
    return __dadd_rn(e, left ? L : t);
}
// FP64 compare, right operand compared last (dp_cell)
__device__ __forceinline__ double cell_fr(double L, double M, double R, double e, int lL, int lM, int lR, int& lab) {
    double b = L;
    int bl = lL;
    if (M < b) { b = M; bl = lM; }
    if (R < b) { b = R; bl = lR; }
    lab = bl;
    return __dadd_rn(e, b);
}
// int64 compare on the bit patterns (M >= +0)
__device__ __forceinline__ long long imin_l(long long a, long long b, bool& bl) {
    bl = (unsigned long long)b < (unsigned long long)a;
    return bl ? b : a;
}
__device__ __forceinline__ double cell_i(double L, double M, double R, double e, int lL, int lM, int lR, int& lab) {
    const unsigned long long l = __double_as_longlong(L), m = __double_as_longlong(M), r = __double_as_longlong(R);
    unsigned long long t = m;
    int tl = lM;
    if (r < t) { t = r; tl = lR; }
    const bool left = l <= t;
    lab = left ? lL : tl;
    return __dadd_rn(e, __longlong_as_double(left ? l : t));
}
__device__ __forceinline__ double cell_ir(double L, double M, double R, double e, int lL, int lM, int lR, int& lab) {
    const unsigned long long l = __double_as_longlong(L), m = __double_as_longlong(M), r = __double_as_longlong(R);
    unsigned long long b = l;
    int bl = lL;
    if (m < b) { b = m; bl = lM; }
    if (r < b) { b = r; bl = lR; }
    lab = bl;
    return __dadd_rn(e, __longlong_as_double(b));
}

// ---- one row per exchange, C = 2 per lane, labels carried --------------------------
template <bool INT>
__global__ void k_row1(double* out, int n, long long* cyc) {
    const int lane = threadIdx.x & 31;
    double m0 = out[lane * 2] * 1e-9, m1 = out[lane * 2 + 1] * 1e-9;
    const double e0 = 1.0 + lane, e1 = 2.0 + lane;
    int l0 = lane * 2, l1 = lane * 2 + 1;
    long long t0 = clk();
    for (int i = 0; i < n; ++i) {
        const double lm = __shfl_up_sync(FULL, m1, 1);
        const double rm = __shfl_down_sync(FULL, m0, 1);
        const int ll = __shfl_up_sync(FULL, l1, 1);
        const int rl = __shfl_down_sync(FULL, l0, 1);
        int a, b;
        double n0, n1;
        if (INT) {
            n0 = cell_i(lm, m0, m1, e0, ll, l0, l1, a);
            n1 = cell_ir(m0, m1, rm, e1, l0, l1, rl, b);
        } else {
            n0 = cell_f(lm, m0, m1, e0, ll, l0, l1, a);
            n1 = cell_fr(m0, m1, rm, e1, l0, l1, rl, b);
        }
        m0 = n0; m1 = n1; l0 = a; l1 = b;
    }
    long long t1 = clk();
    out[lane * 2] = m0 + l0;
    out[lane * 2 + 1] = m1 + l1;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// ---- two rows per exchange (lane-level halo of 2 columns per side), C = 2 -----------
// Lane holds core columns c, c+1; at a block start it receives the left lane's core
// (c-2, c-1) and the right lane's core (c+2, c+3); row a computes c-1..c+2 (4 cells),
// row b computes c, c+1 (2 cells): two rows per shuffle exchange, 3 cells per row.
template <bool INT>
__global__ void k_row2(double* out, int n, long long* cyc) {
    const int lane = threadIdx.x & 31;
    double m0 = out[lane * 2] * 1e-9, m1 = out[lane * 2 + 1] * 1e-9;
    const double e[4] = {1.0 + lane, 2.0 + lane, 3.0 + lane, 4.0 + lane};
    int l0 = lane * 2, l1 = lane * 2 + 1;
    long long t0 = clk();
    for (int i = 0; i < n; i += 2) {
        const double a0 = __shfl_up_sync(FULL, m0, 1), a1 = __shfl_up_sync(FULL, m1, 1);
        const double b0 = __shfl_down_sync(FULL, m0, 1), b1 = __shfl_down_sync(FULL, m1, 1);
        const int la0 = __shfl_up_sync(FULL, l0, 1), la1 = __shfl_up_sync(FULL, l1, 1);
        const int lb0 = __shfl_down_sync(FULL, l0, 1), lb1 = __shfl_down_sync(FULL, l1, 1);
        // row a over (c-2 .. c+3) -> cells c-1, c, c+1, c+2
        int ka, kb, kc, kd;
        double x1, x2, x3, x4;
        if (INT) {
            x1 = cell_ir(a0, a1, m0, e[0], la0, la1, l0, ka);
            x2 = cell_ir(a1, m0, m1, e[1], la1, l0, l1, kb);
            x3 = cell_ir(m0, m1, b0, e[2], l0, l1, lb0, kc);
            x4 = cell_ir(m1, b0, b1, e[3], l1, lb0, lb1, kd);
        } else {
            x1 = cell_fr(a0, a1, m0, e[0], la0, la1, l0, ka);
            x2 = cell_fr(a1, m0, m1, e[1], la1, l0, l1, kb);
            x3 = cell_fr(m0, m1, b0, e[2], l0, l1, lb0, kc);
            x4 = cell_fr(m1, b0, b1, e[3], l1, lb0, lb1, kd);
        }
        // row b -> cells c, c+1
        int p, q;
        if (INT) {
            m0 = cell_ir(x1, x2, x3, e[1], ka, kb, kc, p);
            m1 = cell_ir(x2, x3, x4, e[2], kb, kc, kd, q);
        } else {
            m0 = cell_fr(x1, x2, x3, e[1], ka, kb, kc, p);
            m1 = cell_fr(x2, x3, x4, e[2], kb, kc, kd, q);
        }
        l0 = p;
        l1 = q;
    }
    long long t1 = clk();
    out[lane * 2] = m0 + l0;
    out[lane * 2 + 1] = m1 + l1;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename F>
void run(const char* name, F launch, int n) {
    long long* d;
    cudaMalloc(&d, 8);
    launch(n, d);
    cudaDeviceSynchronize();
    launch(n, d);
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %8.2f cycles per step\n", name, double(c) / double(n));
    cudaFree(d);
}

int main() {
    double* buf;
    cudaMalloc(&buf, 1 << 20);
    cudaMemset(buf, 0, 1 << 20);
    const int n = 4096;
    run("dadd chain", [&](int n, long long* d) { k_dadd<<<1, 32>>>(buf, n, d); }, n);
    run("dsetp+fsel chain (f64 min)", [&](int n, long long* d) { k_dsetp_fsel<<<1, 32>>>(buf, n, d); }, n);
    run("isetp.u64+sel chain (bits min)", [&](int n, long long* d) { k_isetp_sel<<<1, 32>>>(buf, n, d); }, n);
    run("row1 f64 cells (1 warp)", [&](int n, long long* d) { k_row1<false><<<1, 32>>>(buf, n, d); }, n);
    run("row1 int cells (1 warp)", [&](int n, long long* d) { k_row1<true><<<1, 32>>>(buf, n, d); }, n);
    run("row1 f64 cells (4 warps/SM)", [&](int n, long long* d) { k_row1<false><<<1, 128>>>(buf, n, d); }, n);
    run("row1 int cells (4 warps/SM)", [&](int n, long long* d) { k_row1<true><<<1, 128>>>(buf, n, d); }, n);
    run("row2 f64 cells (1 warp)", [&](int n, long long* d) { k_row2<false><<<1, 32>>>(buf, n, d); }, n);
    run("row2 int cells (1 warp)", [&](int n, long long* d) { k_row2<true><<<1, 32>>>(buf, n, d); }, n);
    run("row2 f64 cells (4 warps/SM)", [&](int n, long long* d) { k_row2<false><<<1, 128>>>(buf, n, d); }, n);
    run("row2 int cells (4 warps/SM)", [&](int n, long long* d) { k_row2<true><<<1, 128>>>(buf, n, d); }, n);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
