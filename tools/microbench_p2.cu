// Microbenchmark (not product): the DP phase-2 row step in isolation, one warp,
// to find what makes a 4-cells-per-lane row cost ~200 cycles in the kernel
// against ~82 in tools/microbench.cu's bare k_row<4>.
#define CARVE_KERNELS_HELPERS_ONLY
#include <cstdio>
#include "../paper_2410_21207_b200/csrc/carve_kernels.cuh"
#include "../paper_2410_21207_b200/csrc/dp_cluster.cuh"
using namespace carve_dev;

__device__ __forceinline__ unsigned long long clk() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

// MODEv: 0 full phase-2 row (ring LDS + dirs STS + left_last), 1 no dirs store,
// 2 constant energies (no LDS), 3 plain dp_cell for k=0, 4 no direction tracking
template <int MODEv>
__global__ void k_p2(const double* __restrict__ e, int pitch, double* out, int n, long long* cyc) {
    __shared__ __align__(16) double ring[32][128];
    __shared__ __align__(16) uint8_t dirs[32][128];
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < 32; ++r)
        for (int k = 0; k < 4; ++k) ring[r][lane * 4 + k] = e[r * pitch + lane * 4 + k];
    __syncwarp();
    double mm[4];
    for (int k = 0; k < 4; ++k) mm[k] = out[lane * 4 + k];
    unsigned acc = 0;
    const unsigned long long t0 = clk();
    for (int i0 = 0; i0 < n; i0 += 32) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            double ec[4];
            if constexpr (MODEv == 2) {
                for (int k = 0; k < 4; ++k) ec[k] = 1.0 + k;
            } else {
                const double2 x0 = *reinterpret_cast<const double2*>(&ring[t][lane * 4]);
                const double2 x1 = *reinterpret_cast<const double2*>(&ring[t][lane * 4 + 2]);
                ec[0] = x0.x; ec[1] = x0.y; ec[2] = x1.x; ec[3] = x1.y;
            }
            const double lm = __shfl_up_sync(FULL, mm[3], 1);
            const double rm = __shfl_down_sync(FULL, mm[0], 1);
            double pm = lane == 0 ? dinf() : lm;
            const double rr = lane == 31 ? dinf() : rm;
            uint32_t db = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double cm = mm[k];
                const double nm = (k + 1 < 4) ? mm[k + 1] : rr;
                int d = 0, dummy;
                if constexpr (MODEv == 4) {
                    double best = pm;
                    if (cm < best) best = cm;
                    if (nm < best) best = nm;
                    mm[k] = __dadd_rn(ec[k], best);
                } else if (MODEv != 3 && k == 0) {
                    dp_cell_left_last(pm, cm, nm, 0, 0, 0, ec[k], mm[k], dummy, d);
                } else {
                    dp_cell(pm, cm, nm, 0, 0, 0, ec[k], mm[k], dummy, d);
                }
                db |= uint32_t(d) << (8 * k);
                pm = cm;
            }
            if constexpr (MODEv == 1 || MODEv == 4) acc += db;
            else reinterpret_cast<uint32_t*>(&dirs[t][0])[lane] = db;
        }
    }
    const unsigned long long t1 = clk();
    for (int k = 0; k < 4; ++k) out[lane * 4 + k] = mm[k] + acc + dirs[lane][lane];
    if (lane == 0) cyc[0] = (long long)(t1 - t0);
}

template <typename F>
void run(const char* name, F f, int n) {
    long long* d;
    cudaMalloc(&d, 8);
    f(n, d);
    cudaDeviceSynchronize();
    f(n, d);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %8.2f cycles per row\n", name, double(h) / n);
    cudaFree(d);
}

int main() {
    double *e, *out;
    cudaMalloc(&e, 32 * 256 * 8);
    cudaMalloc(&out, 1 << 16);
    cudaMemset(e, 0, 32 * 256 * 8);
    cudaMemset(out, 0, 1 << 16);
    const int n = 4096;
    run("p2 row: full (ring LDS, dirs STS)", [&](int n, long long* d) { k_p2<0><<<1, 32>>>(e, 256, out, n, d); }, n);
    run("p2 row: no dirs store", [&](int n, long long* d) { k_p2<1><<<1, 32>>>(e, 256, out, n, d); }, n);
    run("p2 row: constant energies", [&](int n, long long* d) { k_p2<2><<<1, 32>>>(e, 256, out, n, d); }, n);
    run("p2 row: plain cell at k=0", [&](int n, long long* d) { k_p2<3><<<1, 32>>>(e, 256, out, n, d); }, n);
    run("p2 row: no direction tracking", [&](int n, long long* d) { k_p2<4><<<1, 32>>>(e, 256, out, n, d); }, n);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
