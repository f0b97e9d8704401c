// dp_variants.h — the K2+K3 DP variant table (template instances of k_dp2,
// dp_cluster.cuh). Instances live in dp_variants_{a,b,c}.cu so nvcc compiles
// them in parallel; carve_cuda.cu selects among them by shape (dp2_plan).
#pragma once
#include <cstddef>
#include <vector>

#include "dp_cluster.cuh"

namespace carve_dev {

struct Dp2Variant {
    int C, K, NW, D;
    bool glab;             // label table in global memory (instances for oversized tables)
    const void* fn;        // hot kernel (no tables)
    const void* fn_tables; // parity-API kernel (writes the full cost / predecessor tables)
    const void* fn_prof;   // hot kernel + clock64 phase counters (tools)
    const void* fn_fused;  // hot kernel, energy recomputed from RGBX (batch mode)
    const void* fn_fwd;    // forward energy from RGBX rows (fused), hot / with tables
    const void* fn_fwd_tables;
    const void* fn_fwdp;   // forward energy from three FP64 cost planes (dp_seam_forward API,
    const void* fn_fwdp_tables;  // the recompute=false forward loop)
    size_t (*smem)(int nblk, int D);        // energy-plane ring (8 B per column)
    size_t (*smem_fused)(int nblk, int D);  // RGBX ring (4 B per column)
    size_t (*smem_costs)(int nblk, int D);  // cost-plane ring (3 x 8 B per column)
    int S() const { return 32 * C - 2 * K; }
    int cols() const { return NW * S(); }
};

// MINB: resident CTAs per SM the register allocation must allow (batch variants)
// GLAB: label table in global memory
template <int C, int K, int NW, int D, int MINB = 1, bool GLAB = false>
Dp2Variant dp2_variant() {
    return Dp2Variant{C, K, NW, D, GLAB,
                      (const void*)k_dp2<C, K, NW, D, 0, false, false, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 1, false, false, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 2, false, false, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 0, true, false, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 0, true, true, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 1, true, true, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 0, false, true, MINB, GLAB>,
                      (const void*)k_dp2<C, K, NW, D, 1, false, true, MINB, GLAB>,
                      &Dp2Smem<C, K, NW, 8>::total,
                      &Dp2Smem<C, K, NW, 4>::total,
                      &Dp2Smem<C, K, NW, 24>::total};
}

// each appends its variants in index order (a: 0-3, b: 4-8, c: 9-13, d: 14-)
void dp2_variants_a(std::vector<Dp2Variant>& t);
void dp2_variants_b(std::vector<Dp2Variant>& t);
void dp2_variants_c(std::vector<Dp2Variant>& t);
void dp2_variants_d(std::vector<Dp2Variant>& t);

}  // namespace carve_dev
